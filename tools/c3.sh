for v in cur nojk32 fulleig lib_e5417; do
  for k in 1 2 3 4; do
    if [ $v = cur ]; then python tools/det_check.py; else QM1B_B200_DEV_LIB=build_ab/$v.so python tools/det_check.py; fi 2>&1 | grep "in-flight" | sed "s/^/$v /"
  done
done > gpurun_out/c3_det.log 2>&1; cat gpurun_out/c3_det.log | sort | uniq -c
