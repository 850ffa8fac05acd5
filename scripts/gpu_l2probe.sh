# Does a small frame chunk keep the axis-1 intermediate in L2?  DRAM bytes per kernel for chunk 2/3/4/6/30.
mkdir -p gpurun_out
for c in 2 3 4 6 30; do
  HETRECO_CHUNK=$c timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --cache-control none -k regex:k_fft -s 20 -c 8 --csv --log-file gpurun_out/l2probe_$c.csv python scripts/profile_c3.py --launches 3 --reps 0 --timed 0 > /dev/null 2>&1
  echo chunk $c rc=$?
done
