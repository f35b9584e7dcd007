for k in 1 2 3; do python tools/det_check.py > gpurun_out/c2_det_$k.log 2>&1; done; cat gpurun_out/c2_det_*.log
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/race_probe.py 4 > gpurun_out/c2_race.log 2>&1; tail -30 gpurun_out/c2_race.log
timeout 600 compute-sanitizer --tool memcheck python tools/race_probe.py 4 > gpurun_out/c2_mem.log 2>&1; tail -30 gpurun_out/c2_mem.log
