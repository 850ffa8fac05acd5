# Mixed-radix combine selection after the bank-conflict fix: coil-parallel (default at 96/160)
# vs coil-serial register-prefetch vs staged-map, C3 shapes, two rounds.
for r in 1 2; do for n in 160 96; do for m in sens_recon rss_recon; do
  timeout 120 python scripts/profile_c3.py --nx $n --method $m --reps 5 --timed 30 2>&1 | tail -1 | sed "s/^/default /"
  HETRECO_COMBINE_CP=0 timeout 120 python scripts/profile_c3.py --nx $n --method $m --reps 5 --timed 30 2>&1 | tail -1 | sed "s/^/serial  /"
  [ $m = sens_recon ] && HETRECO_COMBINE_CP=0 HETRECO_COMBINE_SS=1 timeout 120 python scripts/profile_c3.py --nx $n --method $m --reps 5 --timed 30 2>&1 | tail -1 | sed "s/^/ss      /"
done; done; done
