for r in 1 2; do for lib in lib_st_default lib_st_cs lib_st_cg; do
  python scripts/ab_lib.py build/ab/$lib.so --reps 5 2>&1 | tail -1 | sed "s/^/$lib /" | sed 's/variant.*axis1/axis1/'
done; done
