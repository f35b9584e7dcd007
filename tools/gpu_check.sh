# quick GPU round: parity tests + one bench line (tag = $1)
tag=${1:-x}
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputest.log 2>&1; tail -3 gpurun_out/${tag}_gputest.log
python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench.log 2>&1
tail -1 gpurun_out/${tag}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'e2e', d['e2e']['value'], 'stages_iso', d['config']['stage_ms_isolated'], 'xc', d['roofline_xc']['ms_per_iteration'], 'jk', d['roofline_jk']['ms_per_iteration'])" || tail -20 gpurun_out/${tag}_bench.log
