for c in 1 2 3 4 8; do HETRECO_OVERLAP_CHUNK=$c timeout 120 python scripts/profile_c3.py --reps 0 --timed 50 --params '{"overlap": true}' 2>&1 | tail -1 | sed "s/^/ovl$c /"; done
timeout 120 python scripts/profile_c3.py --reps 5 --timed 50 | tail -1
