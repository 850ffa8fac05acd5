mkdir -p gpurun_out
for c in 1 2 3 5 10 30; do HETRECO_CHUNK=$c HETRECO_COMBINE_VARIANT=1 python scripts/profile_c3.py --launches 3 --reps 10; done 2>&1 | tee gpurun_out/chunks2.txt
HETRECO_CHUNK=3 timeout 300 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_fft -s 20 -c 6 --csv python scripts/profile_c3.py --launches 2 --reps 0 --timed 0 > gpurun_out/ncu_chunk3.csv 2>&1
python3 - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/ncu_chunk3.csv')))
for r in rows:
    if len(r)>14 and r[0].isdigit(): print(r[0], r[4][:40], r[12], r[14])
P
