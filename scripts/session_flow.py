"""Breakdown of the reference-arm flow on the B200 session API."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1807_11830_b200 import hetreco as h
rng = np.random.default_rng(0)
NX, NC, NF = 256, 32, 30
Y = np.asfortranarray((rng.standard_normal((NX, NX, NC, NF), dtype=np.float32) + 0j).astype(np.complex64))
S = np.asfortranarray((rng.standard_normal((NX, NX, NC), dtype=np.float32) + 0j).astype(np.complex64))
s = h.ComputeSession("gpu")
hout = s.allocate_data([((NX, NX, NF), np.complex64)])
M = np.empty((NX, NX, NF), np.complex64, order="F")
p = None
for it in range(6):
    t0 = time.perf_counter(); hk = s.register_data(h.Data([Y, S], h.DataKind.KData)); s.synchronize(); t1 = time.perf_counter()
    if p is None:
        p = h.Process(s, "sens_recon").set_input(hk).set_output(hout).init()
    else:
        p.set_input(hk)
    t2 = time.perf_counter(); p.launch(); s.synchronize(); t3 = time.perf_counter()
    s.fetch_data(hout, [M]); t4 = time.perf_counter()
    s.release_data(hk); t5 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.2f} ms | set_input {1e3*(t2-t1):.2f} | launch(+rebind) {1e3*(t3-t2):.2f} | fetch {1e3*(t4-t3):.2f} | release {1e3*(t5-t4):.2f}")
