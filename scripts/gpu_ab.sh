for args in "--nx 512 --frames 8" "--nx 256"; do
  echo "== $args"
  HETRECO_LIB_LENIENT=1 python scripts/ab_lib.py build/old_lib/libhetreco_b200.so $args --reps 5 2>&1 | tail -1 | sed 's/^/OLD /'
  python scripts/ab_lib.py paper_1807_11830_b200/libhetreco_b200.so $args --reps 5 2>&1 | tail -1 | sed 's/^/NEW /'
done
