mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for v in 0 1 2 3; do for c in 30; do HETRECO_CHUNK=$c HETRECO_COMBINE_VARIANT=$v python scripts/profile_c3.py --launches 3 --reps 10; done; done 2>&1 | tee gpurun_out/v5.txt
for c in 5 10 15; do HETRECO_CHUNK=$c HETRECO_COMBINE_VARIANT=1 python scripts/profile_c3.py --launches 3 --reps 10; done 2>&1 | tee -a gpurun_out/v5.txt
HETRECO_CHUNK=30 python scripts/profile_c3.py --method rss_recon --launches 3 --reps 10 2>&1 | tee -a gpurun_out/v5.txt
python scripts/profile_c3.py --nx 512 --frames 8 --launches 3 --reps 10 2>&1 | tee -a gpurun_out/v5.txt
HETRECO_CHUNK=30 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fft -s 2 -c 2 -o gpurun_out/prof_c3_v5 python scripts/profile_c3.py --launches 2 --reps 0 --timed 0 > gpurun_out/ncu_v5.log 2>&1; tail -2 gpurun_out/ncu_v5.log
