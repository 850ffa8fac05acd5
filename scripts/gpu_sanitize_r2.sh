# compute-sanitizer on the round-2 kernels: TMA axis-1 ring, tcgen05 combine, cooperative normal operator.
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
for tool in memcheck racecheck synccheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_combine.py tests/test_gpu_sense_model.py -q -x -p no:cacheprovider -k "strided_tma or tc_combine or normal_fused" > gpurun_out/san_$tool.txt 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san_$tool.txt | tail -3
done
