for diag in 0 1; do
  if [ $diag = 1 ]; then export HETRECO_CLUSTER_DIAG_LOCAL=1; fi
  for cs in 8 16; do
    echo "diag_local=$diag cluster=$cs"
    HETRECO_CLUSTER_SIZE=$cs HETRECO_RECON_ALGO=cluster timeout 120 python scripts/profile_c3.py --launches 3 --reps 2 --timed 50 2>&1 | tail -1 | sed 's/.*graph/graph/'
  done
done
