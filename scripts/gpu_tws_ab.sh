# Staged-map combine with pass twiddles in registers (0) vs shared memory (1): C3 timing A/B and parity.
for r in 1 2 3; do
  for t in 0 1; do HETRECO_SS_TWSMEM=$t timeout 120 python scripts/profile_c3.py --reps 20 --timed 100 2>&1 | tail -1 | sed "s/^/tws=$t /"; done
done
HETRECO_SS_TWSMEM=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py -q -x -p no:cacheprovider 2>&1 | tail -2
