for k in 1 2 3 4 5 6; do python tools/det_check.py 2>&1 | grep in-flight; done | sort | uniq -c
python -m pytest tests -m gpu -q > gpurun_out/c4_gputest.log 2>&1; tail -3 gpurun_out/c4_gputest.log
