# Mixed-radix chains at C3 shapes (32 coils x 30 frames): per-kernel device us.
for n in 160 96 192 320 384; do timeout 120 python scripts/profile_c3.py --nx $n --reps 10 --timed 50 2>&1 | tail -1; done
timeout 120 python scripts/profile_c3.py --nx 160 --method rss_recon --reps 10 --timed 50 2>&1 | tail -1
