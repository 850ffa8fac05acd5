# C4 fused normal operator: parity (fused default and the 3-kernel path), latency A/B, ncu of the fused kernel.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sense_model.py -q -rf -p no:cacheprovider > gpurun_out/c4_pytest.txt 2>&1; tail -4 gpurun_out/c4_pytest.txt
HETRECO_NORMAL_FUSED=0 timeout 600 python -m pytest tests/test_gpu_sense_model.py -q -rf -p no:cacheprovider > gpurun_out/c4_pytest_unfused.txt 2>&1; tail -2 gpurun_out/c4_pytest_unfused.txt
for v in 1 0 1 0; do HETRECO_NORMAL_FUSED=$v timeout 300 python scripts/small_configs.py 2>&1 | tail -1 | sed "s/^/fused=$v /"; done | tee gpurun_out/c4_ab.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:normal_fused -s 3 -c 1 -o gpurun_out/c4_full python scripts/small_configs.py > gpurun_out/c4_ncu.log 2>&1; tail -2 gpurun_out/c4_ncu.log
