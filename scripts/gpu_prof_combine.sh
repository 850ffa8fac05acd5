mkdir -p gpurun_out
HETRECO_COMBINE_TMA=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fft_combine -s 1 -c 1 -o gpurun_out/prof_combine python scripts/profile_c3.py --launches 2 --reps 0 --timed 0 > gpurun_out/ncu_combine.log 2>&1; tail -2 gpurun_out/ncu_combine.log
HETRECO_TMA_STAGES=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fft_combine_tma -s 1 -c 1 -o gpurun_out/prof_combine_tma python scripts/profile_c3.py --launches 2 --reps 0 --timed 0 > gpurun_out/ncu_combine_tma.log 2>&1; tail -2 gpurun_out/ncu_combine_tma.log
