"""Print the key numbers of a bench JSON line: python tools/bl.py gpurun_out/x_bench.log"""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('value', round(d['value'], 1), 'e2e', round(d['e2e']['value'], 1),
      'iso', {k: round(v, 2) for k, v in d['config']['stage_ms_isolated'].items() if v > 0.01},
      'xc', round(d['roofline']['ms_per_iteration'], 3), 'jk', round(d['roofline_jk']['ms_per_iteration'], 3),
      round(d['roofline_jk']['frac'], 3), 'post', round(d['roofline_post']['ms_per_iteration'], 3))
