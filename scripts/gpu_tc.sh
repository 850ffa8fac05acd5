# DFT-as-GEMM (tcgen05) combine experiment: parity, A/B timing, ncu of the TC combine.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc_combine.py -q -rf -s -p no:cacheprovider > gpurun_out/tc_pytest.txt 2>&1; tail -9 gpurun_out/tc_pytest.txt
for v in 0 1 0 1; do HETRECO_COMBINE_TC=$v timeout 120 python scripts/profile_c3.py --reps 20 2>&1 | tail -1 | sed "s/^/tc=$v /"; done | tee gpurun_out/tc_ab.txt
HETRECO_COMBINE_TC=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:combine_tc -s 1 -c 1 -o gpurun_out/tc_full python scripts/profile_c3.py --launches 2 --reps 0 --timed 0 > gpurun_out/tc_ncu.log 2>&1; tail -1 gpurun_out/tc_ncu.log
