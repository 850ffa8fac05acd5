# ncu source-level capture of the default C3 SENSE combine + 2-rank dry run of the multi-rank bench path on one GPU.
mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:combine_ss -s 1 -c 1 -o gpurun_out/ss_full python scripts/profile_c3.py --launches 2 --reps 0 --timed 0 > gpurun_out/ss_ncu.log 2>&1; tail -1 gpurun_out/ss_ncu.log
HETRECO_BENCH_DEVICE=0 HETRECO_BENCH_DIST=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo rc=$?; cut -c1-700 gpurun_out/bench2.json; tail -3 gpurun_out/bench2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench2_ref.json 2> gpurun_out/bench2_ref.err; echo rc=$?; cut -c1-300 gpurun_out/bench2_ref.json
