# usage: bash tools/ab.sh <variant.so> [reps]: bench lines of the current build and a variant, interleaved
v=$1; n=${2:-2}
for r in $(seq $n); do
 for x in cur $v; do
  if [ $x = cur ]; then python bench.py --no-cpu-baseline; else QM1B_B200_DEV_LIB=build_ab/$x.so python bench.py --no-cpu-baseline; fi 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$x', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'xc', round(d['roofline']['ms_per_iteration'],3), 'jk', round(d['roofline_jk']['ms_per_iteration'],3), 'iso', {k: round(v,2) for k,v in d['config']['stage_ms_isolated'].items()})"
 done
done
