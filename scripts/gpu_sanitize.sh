mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed_radix.py tests/test_gpu_sense_model.py tests/test_source_kernels.py -q -x -p no:cacheprovider > gpurun_out/memcheck.txt 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid|out of bounds" gpurun_out/memcheck.txt | head -10
