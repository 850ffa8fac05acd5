mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sense_model.py tests/test_gpu_baseline_shapes.py -q -x -p no:cacheprovider > gpurun_out/cp_pytest.txt 2>&1; tail -2 gpurun_out/cp_pytest.txt
for v in 8 16 8 16; do HETRECO_CP_POINTS=$v timeout 300 python scripts/small_configs.py 2>&1 | tail -1 | sed "s/^/cp=$v /"; done
