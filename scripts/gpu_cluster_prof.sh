mkdir -p gpurun_out
HETRECO_DEBUG=1 HETRECO_RECON_ALGO=cluster timeout 300 python scripts/profile_c3.py --launches 3 --reps 0 --timed 0 2>&1 | tail -3
HETRECO_RECON_ALGO=cluster timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_recon -s 1 -c 1 -o gpurun_out/prof_cluster python scripts/profile_c3.py --launches 3 --reps 0 --timed 0 > gpurun_out/ncu_cluster.log 2>&1; tail -3 gpurun_out/ncu_cluster.log
