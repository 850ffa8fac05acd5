mkdir -p gpurun_out
for f in test_gpu_integration test_gpu_parity; do python -m pytest tests/$f.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2; echo "rc=$?"; done
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "full rc=$?"; tail -3 gpurun_out/pytest_gpu.txt
