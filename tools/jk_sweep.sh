# J/K CTA-split sweep on the bench (GPU box)
for s in ${SPLITS:-6 8 12 16 24}; do
  QM1B_JK_SPLIT=$s python bench.py --no-cpu-baseline > gpurun_out/sw_$s.log 2>/dev/null
  echo "split $s: $(python tools/bl.py gpurun_out/sw_$s.log)"
done
