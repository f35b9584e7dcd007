# J/K kernel coverage: the GPU parity tests under different CTA partitions of the slabs (GPU box)
for s in 1 2 3 5 9 24; do
  echo "split $s: $(QM1B_JK_SPLIT=$s python -m pytest tests/test_gpu_parity.py tests/test_parity_scale.py -m gpu -q -x -k 'jk or f32 or operators or bucket' 2>&1 | tail -1)"
done
