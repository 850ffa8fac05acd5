cat > /tmp/ovl.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1807_11830_b200 import hetreco as h
rng = np.random.default_rng(0)
nx, nc, nf = 256, 32, 30
Y = np.asfortranarray((rng.standard_normal((nx, nx, nc, nf), dtype=np.float32) + 1j*rng.standard_normal((nx, nx, nc, nf), dtype=np.float32)).astype(np.complex64))
S = np.asfortranarray((rng.standard_normal((nx, nx, nc), dtype=np.float32) + 0j).astype(np.complex64))
s = h.ComputeSession("gpu")
hin = s.register_data(h.Data([Y, S], h.DataKind.KData))
hout = s.allocate_data([((nx, nx, nf), np.complex64)])
for ov in (False, True):
    p = h.Process(s, "sens_recon").set_input(hin).set_output(hout).init({"overlap": ov})
    for _ in range(5): p.launch()
    s.timer_start()
    for _ in range(100): p.launch()
    t = s.timer_stop() / 100
    print(f"overlap={ov} chunk={os.environ.get('HETRECO_OVERLAP_CHUNK')} split={os.environ.get('HETRECO_OVERLAP_SPLIT')} {t*1e6:.1f} us")
PY
for oc in 8 10 15; do for sp in 0 40 50 60 70; do HETRECO_OVERLAP_CHUNK=$oc HETRECO_OVERLAP_SPLIT=$sp python /tmp/ovl.py 2>&1 | tail -1; done; done
