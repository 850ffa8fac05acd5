# Radix choice at 256^2 C3: 16 samples per thread (radix-16 x 16, one exchange) vs 8 (radix-8 x 8 x 4, two exchanges).
for r in 1 2; do
  timeout 120 python scripts/profile_c3.py --reps 10 --timed 50 2>&1 | tail -1 | sed "s/^/default(ss,R16)        /"
  HETRECO_COMBINE_SS=0 timeout 120 python scripts/profile_c3.py --reps 10 --timed 50 2>&1 | tail -1 | sed "s/^/contig R16 (var 11)    /"
  HETRECO_COMBINE_SS=0 HETRECO_COMBINE_VARIANT=15 timeout 120 python scripts/profile_c3.py --reps 10 --timed 50 2>&1 | tail -1 | sed "s/^/contig R8 (var 15)     /"
  HETRECO_STRIDED_RING=0 HETRECO_STRIDED_POINTS=8 timeout 120 python scripts/profile_c3.py --reps 10 --timed 50 2>&1 | tail -1 | sed "s/^/axis-1 R8 (no ring)    /"
  HETRECO_STRIDED_RING=0 timeout 120 python scripts/profile_c3.py --reps 10 --timed 50 2>&1 | tail -1 | sed "s/^/axis-1 R16 (no ring)   /"
done
