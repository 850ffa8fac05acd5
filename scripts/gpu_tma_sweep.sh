timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed_radix.py -q -x -p no:cacheprovider -k "recon or stream or chain" 2>&1 | tail -2
HETRECO_COMBINE_TMA=0 timeout 120 python scripts/profile_c3.py --reps 5 2>&1 | tail -1 | sed 's/^/regprefetch /'
for k in 2 3 4 6; do HETRECO_TMA_STAGES=$k timeout 120 python scripts/profile_c3.py --reps 5 2>&1 | tail -1 | sed "s/^/tma K=$k /"; done
HETRECO_TMA_STAGES=4 timeout 120 python scripts/profile_c3.py --method rss_recon --reps 5 2>&1 | tail -1
timeout 120 python scripts/profile_c3.py --nx 512 --frames 8 --reps 5 2>&1 | tail -1
HETRECO_COMBINE_TMA=0 timeout 120 python scripts/profile_c3.py --nx 512 --frames 8 --reps 5 2>&1 | tail -1
timeout 120 python scripts/profile_c3.py --nx 160 --reps 5 2>&1 | tail -1
