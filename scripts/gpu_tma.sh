# Axis-1 TMA ring vs cp.async ring: bit-exactness, A/B timing at 256^2 (C3) and 512^2 x 32 x 8, ncu of both 512 kernels.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -k "strided_tma or strided_ring" -p no:cacheprovider > gpurun_out/tma_pytest.txt 2>&1; tail -3 gpurun_out/tma_pytest.txt
for r in 1 2; do for v in 0 1; do
  HETRECO_STRIDED_TMA=$v timeout 300 python scripts/profile_c3.py --reps 20 2>&1 | tail -1 | sed "s/^/tma=$v /"
  HETRECO_STRIDED_TMA=$v timeout 300 python scripts/profile_c3.py --nx 512 --frames 8 --reps 20 2>&1 | tail -1 | sed "s/^/tma=$v /"
done; done | tee gpurun_out/tma_ab.txt
for v in 0 1; do HETRECO_STRIDED_TMA=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fft_strided -s 1 -c 1 -o gpurun_out/tma512_$v python scripts/profile_c3.py --nx 512 --frames 8 --launches 2 --reps 0 --timed 0 > gpurun_out/tma_ncu_$v.log 2>&1; tail -1 gpurun_out/tma_ncu_$v.log; done
