# Axis-1 pass at 256^2 (C3): cp.async ring (default) vs TMA ring variants (stages x columns), 2 rounds.
for r in 1 2; do
  timeout 120 python scripts/profile_c3.py --reps 20 --timed 100 2>&1 | tail -1 | sed "s/^/cpasync /"
  HETRECO_STRIDED_TMA=1 timeout 120 python scripts/profile_c3.py --reps 20 --timed 100 2>&1 | tail -1 | sed "s/^/tma2x32 /"
  for k in 2 3 4; do
    HETRECO_STRIDED_TMA=1 HETRECO_TMA_TX256=16 HETRECO_TMA_STAGES256=$k timeout 120 python scripts/profile_c3.py --reps 20 --timed 100 2>&1 | tail -1 | sed "s/^/tma${k}x16 /"
  done
done
