timeout 800 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "recon or stream or chain or phantom or cli" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -5
for oc in 0 4 8 16; do
  HETRECO_OVERLAP_CHUNK=$oc python scripts/profile_c3.py --reps 3 --timed 100 2>&1 | tail -1 | sed "s/variant.*graph/oc=$oc graph/"
done
HETRECO_OVERLAP_CHUNK=8 python scripts/profile_c3.py --method rss_recon --reps 3 --timed 100 2>&1 | tail -1 | sed "s/variant.*graph/RSS oc=8 graph/"
HETRECO_OVERLAP_CHUNK=0 python scripts/profile_c3.py --method rss_recon --reps 3 --timed 100 2>&1 | tail -1 | sed "s/variant.*graph/RSS oc=0 graph/"
for oc in 0 4; do HETRECO_OVERLAP_CHUNK=$oc python scripts/profile_c3.py --nx 512 --frames 8 --reps 3 --timed 50 2>&1 | tail -1 | sed "s/variant.*graph/512 oc=$oc graph/"; done
