# Profile refresh (run on the GPU box from the repo root): bench launch list + ncu --set full
# summaries of the XC, J/K, post and ERI kernels -> gpurun_out/ (copied to profiles/ by hand).
set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/pb.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
python tools/prof_run.py 256 3 > gpurun_out/pr.log 2>&1 && \
for k in k_xc k_jk k_post; do ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/full_$k python tools/prof_run.py 256 3 > gpurun_out/ncu_$k.log 2>&1; done
ncu --set full --clock-control none --import-source on -k regex:k_eri -c 6 -o gpurun_out/full_k_eri python tools/prof_run.py 256 3 > gpurun_out/ncu_k_eri.log 2>&1
ls -la gpurun_out | tail -12
python tools/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt
python tools/ncu_summary.py gpurun_out/ncu_full_metrics.json xc_256mol=gpurun_out/full_k_xc.ncu-rep jk_256mol=gpurun_out/full_k_jk.ncu-rep post_256mol=gpurun_out/full_k_post.ncu-rep eri_256mol=gpurun_out/full_k_eri.ncu-rep
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
