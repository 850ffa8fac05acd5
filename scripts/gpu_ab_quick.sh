# GPU test suite + C3 per-kernel timing + small configs (after a core change).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
for r in 1 2; do timeout 120 python scripts/profile_c3.py --reps 20 2>&1 | tail -1; done
timeout 120 python scripts/profile_c3.py --nx 512 --frames 8 --reps 20 2>&1 | tail -1
timeout 120 python scripts/profile_c3.py --method rss_recon --reps 20 2>&1 | tail -1
timeout 300 python scripts/small_configs.py 2>&1 | tail -1
