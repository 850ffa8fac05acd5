timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for nx in 256 512 160; do fr=30; [ $nx = 512 ] && fr=8; python scripts/profile_c3.py --nx $nx --frames $fr --reps 5 2>&1 | tail -1 | sed 's/variant.*axis1/axis1/'; done
python scripts/profile_c3.py --method rss_recon --reps 5 2>&1 | tail -1 | sed 's/variant.*axis1/axis1/'
HETRECO_RECON_ALGO=cluster HETRECO_CLUSTER_SIZE=16 python scripts/profile_c3.py --reps 2 2>&1 | tail -1 | sed 's/variant.*axis1/cluster16 axis1/'
