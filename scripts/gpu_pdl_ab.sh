# PDL graph edges on/off: small configs (C1, C2, C4) and the C3 chain, two alternating rounds.
mkdir -p gpurun_out
for r in 1 2; do
  for p in 0 1; do
    HETRECO_PDL=$p timeout 300 python scripts/small_configs.py 2>&1 | tail -1
    HETRECO_PDL=$p timeout 300 python scripts/profile_c3.py --reps 0 --timed 100 2>&1 | tail -1 | sed "s/^/pdl=$p /"
  done
done
