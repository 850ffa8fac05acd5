timeout 800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
for nx in 256 512 160; do
  fr=30; [ $nx = 512 ] && fr=8
  python scripts/profile_c3.py --nx $nx --frames $fr --reps 5 2>&1 | tail -1 | sed 's/variant.*axis1/SS axis1/'
  HETRECO_COMBINE_SS=0 python scripts/profile_c3.py --nx $nx --frames $fr --reps 5 2>&1 | tail -1 | sed 's/variant.*axis1/OLD axis1/'
done
