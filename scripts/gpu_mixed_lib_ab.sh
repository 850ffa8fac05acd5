# Mixed-radix C3 shapes: old library (build/old_lib) vs current vs variant B (build/ab/libB.so).
for r in 1 2; do
for n in 160 96 192 320 384; do
  for lib in build/old_lib/libhetreco_b200.so paper_1807_11830_b200/libhetreco_b200.so build/ab/libB.so; do
    [ -f $lib ] || continue
    timeout 120 python scripts/ab_lib.py $lib --nx $n --reps 5 --timed 50 2>&1 | tail -1 | sed "s|^|$(basename $(dirname $lib))/$(basename $lib) |"
  done
done
for lib in build/old_lib/libhetreco_b200.so paper_1807_11830_b200/libhetreco_b200.so build/ab/libB.so; do
  timeout 120 python scripts/ab_lib.py $lib --nx 160 --method rss_recon --reps 5 --timed 50 2>&1 | tail -1 | sed "s|^|$(basename $(dirname $lib))/$(basename $lib) |"
done
done
