for v in jqinf jq512 cur; do
  for s in 1 4 16; do
    if [ $v = cur ]; then QM1B_JK_SPLIT=$s python tools/jkerr.py; else QM1B_B200_DEV_LIB=build_ab/$v.so QM1B_JK_SPLIT=$s python tools/jkerr.py; fi 2>&1 | tail -1 | sed "s/^/$v /"
  done
  if [ $v = cur ]; then python bench.py --no-cpu-baseline; else QM1B_B200_DEV_LIB=build_ab/$v.so python bench.py --no-cpu-baseline; fi > gpurun_out/ab_$v.log 2>/dev/null
  echo "$v: $(python tools/bl.py gpurun_out/ab_$v.log)"
done
