python tools/f32_ops.py gpurun_out/c5_ops_cur.json > gpurun_out/c5_ops_cur.log 2>&1; cat gpurun_out/c5_ops_cur.log
QM1B_B200_DEV_LIB=build_ab/aoexp0.so python tools/f32_ops.py gpurun_out/c5_ops_old.json > gpurun_out/c5_ops_old.log 2>&1; cat gpurun_out/c5_ops_old.log
PARITY_RAW=gpurun_out/c5_raw_cur.json python tools/parity_report.py gpurun_out/c5_parity_cur.md > /dev/null 2>&1; grep configs gpurun_out/c5_parity_cur.md
PARITY_RAW=gpurun_out/c5_raw_old.json QM1B_B200_DEV_LIB=build_ab/aoexp0.so python tools/parity_report.py gpurun_out/c5_parity_old.md > /dev/null 2>&1; grep configs gpurun_out/c5_parity_old.md
for v in cur old cur old; do
 if [ $v = cur ]; then python bench.py --no-cpu-baseline; else QM1B_B200_DEV_LIB=build_ab/aoexp0.so python bench.py --no-cpu-baseline; fi 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'xc', d['roofline_xc']['ms_per_iteration'], 'jk', d['roofline_jk']['ms_per_iteration'])"
done
