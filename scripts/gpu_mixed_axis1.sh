# Mixed-radix axis-1 pass variants (HETRECO_STRIDED_MIXED bits: 1 prefetch, 256 twiddles in registers), two rounds.
for r in 1 2; do for n in 160 320 96 192; do for v in 0 1 256 257; do
  HETRECO_STRIDED_MIXED=$v timeout 120 python scripts/profile_c3.py --nx $n --reps 10 --timed 30 2>&1 | tail -1 | sed -E "s/^/v=$v /; s/variant=- chunk=auto kernels=2 \| //; s/ = [0-9]+ frames\/s//"
done; done; done
