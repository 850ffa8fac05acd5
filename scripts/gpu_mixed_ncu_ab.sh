# Mixed-radix combine: shared-memory metrics, old library (build/old_lib) vs current.
M=gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,launch__registers_per_thread,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum
for n in 160 192 384 320; do
  for lib in build/old_lib/libhetreco_b200.so paper_1807_11830_b200/libhetreco_b200.so; do
    timeout 300 ncu --metrics $M --clock-control none -k regex:"k_fft_combine" -s 1 -c 1 --csv python scripts/ab_lib.py $lib --nx $n --launches 2 --reps 0 --timed 0 2>/dev/null | grep -v "^==" | sed "s|^|$n,$(basename $(dirname $lib)),|"
  done
done > gpurun_out/mixed_ab.csv
