python -m pytest tests -m gpu -x -q > gpurun_out/c1_gputest.log 2>&1; tail -3 gpurun_out/c1_gputest.log
python bench.py > gpurun_out/c1_bench.log 2>&1; tail -1 gpurun_out/c1_bench.log
PARITY_RAW=gpurun_out/c1_parity_raw.json python tools/parity_report.py gpurun_out/c1_parity.md > gpurun_out/c1_parity.log 2>&1; tail -12 gpurun_out/c1_parity.log
