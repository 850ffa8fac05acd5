mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for c in 1 2 3 4 6 10 30; do for v in 1 3; do HETRECO_CHUNK=$c HETRECO_COMBINE_VARIANT=$v python scripts/profile_c3.py --launches 3 --reps 10; done; done 2>&1 | tee gpurun_out/chunks.txt
for c in 2 30; do HETRECO_CHUNK=$c python scripts/profile_c3.py --method rss_recon --launches 3 --reps 10; done 2>&1 | tee -a gpurun_out/chunks.txt
HETRECO_CHUNK=2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_fft -s 30 -c 6 --csv python scripts/profile_c3.py --launches 2 --reps 0 --timed 0 > gpurun_out/ncu_chunk2.csv 2>&1; tail -30 gpurun_out/ncu_chunk2.csv
