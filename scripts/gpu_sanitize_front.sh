# compute-sanitizer on the opt-in cluster front kernel of the normal operator.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_sense_model.py -q -x -p no:cacheprovider -k cluster_front > gpurun_out/san_front_$tool.txt 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san_front_$tool.txt | tail -3
done
