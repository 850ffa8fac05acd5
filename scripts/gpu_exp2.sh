mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
for v in 0 1 2 3; do for l in 32 64 128; do HETRECO_COMBINE_VARIANT=$v HETRECO_LINES_PER_BLOCK=$l python scripts/profile_c3.py --launches 3 --reps 20; done; done 2>&1 | tee gpurun_out/variants2.txt
for v in 0 1 2 3; do HETRECO_COMBINE_VARIANT=$v python scripts/profile_c3.py --method rss_recon --launches 3 --reps 20; done 2>&1 | tee -a gpurun_out/variants2.txt
for v in 1 3; do HETRECO_COMBINE_VARIANT=$v python scripts/profile_c3.py --nx 512 --frames 8 --launches 3 --reps 20; done 2>&1 | tee -a gpurun_out/variants2.txt
