# Round-2 profile set (GPU box, repo root): the bench launch list + ncu --set full of the
# XC, J/K, post and ERI kernels with per-kernel SASS opcode summaries -> gpurun_out/<tag>_*
tag=${1:-r2}
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_pb.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_l.log 2>&1
python tools/launches.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_bench_launches_summary.txt
python tools/prof_run.py 256 3 > gpurun_out/${tag}_pr.log 2>&1
for k in k_xc k_jk32 k_post; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${tag}_full_$k \
      python tools/prof_run.py 256 3 > gpurun_out/${tag}_ncu_$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_eri -c 6 -o gpurun_out/${tag}_full_k_eri \
    python tools/prof_run.py 256 3 > gpurun_out/${tag}_ncu_k_eri.log 2>&1
for k in k_xc k_jk32 k_post k_eri; do
  ncu -i gpurun_out/${tag}_full_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_${k}_sass.csv 2>/dev/null
  python tools/sass_ops.py gpurun_out/${tag}_${k}_sass.csv > gpurun_out/${tag}_sass_ops_$k.txt 2>&1
  rm -f gpurun_out/${tag}_${k}_sass.csv
done
python tools/ncu_summary.py gpurun_out/${tag}_ncu_full_metrics.json xc_256mol=gpurun_out/${tag}_full_k_xc.ncu-rep \
    jk_256mol=gpurun_out/${tag}_full_k_jk32.ncu-rep post_256mol=gpurun_out/${tag}_full_k_post.ncu-rep \
    eri_256mol=gpurun_out/${tag}_full_k_eri.ncu-rep
rm -f gpurun_out/*.ncu-rep
head -16 gpurun_out/${tag}_bench_launches_summary.txt
