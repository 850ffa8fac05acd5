mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for v in 1 3 5 7; do HETRECO_CHUNK=30 HETRECO_COMBINE_VARIANT=$v python scripts/profile_c3.py --launches 3 --reps 10; done 2>&1 | tee gpurun_out/v6.txt
for lp in 64 256; do HETRECO_LINES_PER_BLOCK=$lp HETRECO_CHUNK=30 HETRECO_COMBINE_VARIANT=5 python scripts/profile_c3.py --launches 3 --reps 10; done 2>&1 | tee -a gpurun_out/v6.txt
for sp in 8 16; do for tx in 8 16 32; do HETRECO_STRIDED_POINTS=$sp HETRECO_STRIDED_TX=$tx HETRECO_CHUNK=30 python scripts/profile_c3.py --launches 3 --reps 10; done; done 2>&1 | tee -a gpurun_out/v6.txt
for v in 1 5 7; do HETRECO_COMBINE_VARIANT=$v python scripts/profile_c3.py --method rss_recon --launches 3 --reps 10; done 2>&1 | tee -a gpurun_out/v6.txt
