for nx in 160 256; do
  for cp in 0 1; do HETRECO_COMBINE_CP=$cp python scripts/profile_c3.py --nx $nx --reps 3 2>&1 | tail -1 | sed "s/variant.*axis0/cp=$cp axis0/"; done
  HETRECO_COMBINE_CP=1 python scripts/profile_c3.py --nx $nx --method rss_recon --reps 3 2>&1 | tail -1 | sed "s/variant.*axis0/cp=1 axis0/"
  HETRECO_COMBINE_CP=0 python scripts/profile_c3.py --nx $nx --method rss_recon --reps 3 2>&1 | tail -1 | sed "s/variant.*axis0/cp=0 axis0/"
done
