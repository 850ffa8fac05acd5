for v in 3 11 1 15; do HETRECO_COMBINE_VARIANT=$v python scripts/profile_c3.py --launches 3 --reps 20; done 2>&1 | cut -c1-220
for v in 3 11; do HETRECO_COMBINE_VARIANT=$v python scripts/profile_c3.py --method rss_recon --launches 3 --reps 20; done 2>&1 | cut -c1-220
for v in 3 11; do HETRECO_COMBINE_VARIANT=$v python scripts/profile_c3.py --nx 512 --frames 8 --launches 3 --reps 10; done 2>&1 | cut -c1-220
