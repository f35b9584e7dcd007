# copy the gpurun_out/fin_* measurement set into profiles/r2_* (run here, after tools/final_r2.sh on the GPU box)
cd "$(dirname "$0")/../gpurun_out" || exit 1
cp fin_ncu_full_metrics.json ../profiles/r2_ncu_full_metrics.json
cp fin_bench_launches_summary.txt ../profiles/r2_bench_launches_summary.txt
cp fin_launches.csv ../profiles/r2_bench_launches.csv
for k in k_eri k_jk32 k_post k_xc; do cp fin_sass_ops_$k.txt ../profiles/r2_sass_ops_$k.txt; done
tail -1 fin_bench.log > ../profiles/r2_bench_line.json
tail -1 fin_reference.log > ../profiles/r2_reference_line.json
cp fin_parity.md ../profiles/r2_parity_report.md
cp fin_src_jk_lines.txt ../profiles/r2_src_lines_k_jk32.txt
cp fin_src_xc_lines.txt ../profiles/r2_src_lines_k_xc.txt
cp fin_datagen.json ../profiles/r2_datagen_100k.json
tail -1 fin_eri_bench.log > ../profiles/r2_eri_bench.json
