for lib in lib_ldg lib_ldcg; do
  for v in 11 3 1 27 9; do
    HETRECO_COMBINE_VARIANT=$v python scripts/ab_lib.py build/ab/$lib.so --reps 5 2>&1 | tail -1 | sed "s/^/$lib v=$v /" | sed 's/variant.*axis0/axis0/'
  done
done
