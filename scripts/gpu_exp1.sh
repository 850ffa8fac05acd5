mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
for v in 0 1 2 3; do for l in 64 128 256; do HETRECO_COMBINE_VARIANT=$v HETRECO_LINES_PER_BLOCK=$l python scripts/profile_c3.py --launches 3 --reps 20; done; done 2>&1 | tee gpurun_out/variants.txt
for v in 0 1; do HETRECO_COMBINE_VARIANT=$v python scripts/profile_c3.py --method rss_recon --launches 3 --reps 20; done 2>&1 | tee -a gpurun_out/variants.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fft -s 2 -c 2 -o gpurun_out/prof_c3_v0 python scripts/profile_c3.py --launches 2 --reps 0 > gpurun_out/ncu_v0.log 2>&1; tail -3 gpurun_out/ncu_v0.log
