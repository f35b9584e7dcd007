set -x
python tools/prof_run.py 256 3 > gpurun_out/pr.log 2>&1
for k in k_xc k_jk k_post; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/p1_$k python tools/prof_run.py 256 3 > gpurun_out/ncu_$k.log 2>&1
  ncu -i gpurun_out/p1_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/p1_${k}_sass.csv 2>/dev/null
  python tools/sass_ops.py gpurun_out/p1_${k}_sass.csv > gpurun_out/p1_${k}_ops.txt 2>&1
done
python tools/ncu_summary.py gpurun_out/p1_metrics.json xc=gpurun_out/p1_k_xc.ncu-rep jk=gpurun_out/p1_k_jk.ncu-rep post=gpurun_out/p1_k_post.ncu-rep
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
