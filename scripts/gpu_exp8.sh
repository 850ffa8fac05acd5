for pf in 0 1; do HETRECO_STRIDED_PF=$pf python scripts/profile_c3.py --launches 3 --reps 20; done 2>&1 | cut -c1-220
for pf in 0 1; do for sp in 8 16; do for tx in 4 8 16; do echo "pf=$pf sp=$sp tx=$tx"; HETRECO_STRIDED_PF=$pf HETRECO_STRIDED_POINTS=$sp HETRECO_STRIDED_TX=$tx python scripts/profile_c3.py --nx 512 --frames 8 --launches 3 --reps 10 2>&1 | cut -c1-200 | tail -1; done; done; done
