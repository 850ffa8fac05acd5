# Pageable register/fetch flow vs the staging pool's memcpy threads.
nproc
for t in 4 8 12 16; do HETRECO_STAGER_THREADS=$t timeout 300 python scripts/session_flow.py 2>&1 | head -1 | sed "s/^/threads=$t /"; done
