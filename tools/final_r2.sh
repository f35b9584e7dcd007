# Round-2 final measurement set (GPU box, repo root) -> gpurun_out/fin_*
python -m pytest tests -m gpu -q > gpurun_out/fin_gputest.log 2>&1; tail -2 gpurun_out/fin_gputest.log
python bench.py > gpurun_out/fin_bench.log 2>gpurun_out/fin_bench.err; python tools/bl.py gpurun_out/fin_bench.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_reference.log 2>/dev/null; tail -1 gpurun_out/fin_reference.log | cut -c1-300
PARITY_RAW=gpurun_out/fin_parity_raw.json python tools/parity_report.py gpurun_out/fin_parity.md > gpurun_out/fin_parity.log 2>&1; tail -12 gpurun_out/fin_parity.log
bash tools/prof_r2.sh fin
NLINES=60 bash tools/prof_src.sh fin_src_jk k_jk32
NLINES=60 bash tools/prof_src.sh fin_src_xc k_xc
python tools/eri_bench.py > gpurun_out/fin_eri_bench.log 2>&1; tail -2 gpurun_out/fin_eri_bench.log | cut -c1-400
python tools/datagen_bench.py --out gpurun_out/fin_datagen.json > gpurun_out/fin_datagen.log 2>&1; tail -1 gpurun_out/fin_datagen.log | cut -c1-400
