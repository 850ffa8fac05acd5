# compute-sanitizer over the mixed-radix kernels after the shared-memory layout change.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_mixed_radix.py -q -x -p no:cacheprovider > gpurun_out/san_mixed_$tool.txt 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san_mixed_$tool.txt | tail -3
done
