# Round-2 measurement with the current code: GPU tests, smoke, bench (+ reference arm),
# ncu launch list of the bench command, ncu --set full of both C3 chain kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.csv
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cut -c1-300 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; cut -c1-300 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-extras --no-cpu-baseline --no-session-flow > gpurun_out/ncu_bench.out 2>&1; wc -l gpurun_out/launches.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fft_strided_ring|k_fft_combine_ss" -s 2 -c 2 -o gpurun_out/prof_final python scripts/profile_c3.py --launches 2 --reps 0 --timed 0 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
