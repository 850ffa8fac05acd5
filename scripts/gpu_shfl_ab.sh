# Staged-map combine: shared-memory line exchange (default) vs warp-shuffle transpose (HETRECO_SS_SHFL=1).
for r in 1 2 3; do
  for v in 0 1; do HETRECO_SS_SHFL=$v timeout 120 python scripts/profile_c3.py --reps 20 --timed 100 2>&1 | tail -1 | sed "s/^/shfl=$v /"; done
done
HETRECO_SS_SHFL=1 timeout 600 python -m pytest tests/test_gpu_tc_combine.py -q -x -p no:cacheprovider -k shuffle 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -k regex:combine_ss -c 1 --csv python scripts/profile_c3.py --launches 1 --reps 0 --timed 0 2>/dev/null | grep -v "^==" | cut -d, -f13-15 | tail -6
HETRECO_SS_SHFL=1 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -k regex:combine_ss -c 1 --csv python scripts/profile_c3.py --launches 1 --reps 0 --timed 0 2>/dev/null | grep -v "^==" | cut -d, -f13-15 | tail -6
