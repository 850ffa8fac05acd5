"""H2D bandwidth of register_data from pageable vs pinned host memory."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1807_11830_b200 import hetreco as h
s = h.ComputeSession("gpu")
n = 256 * 256 * 32 * 30
a = np.ones(n, np.complex64)
p = h.pinned_empty((n,), np.complex64); p[...] = 1
for name, arr in (("pageable", a), ("pinned", p)):
    hd = s.register_data([arr]); s.release_data(hd)
    t0 = time.perf_counter()
    for _ in range(5):
        hd = s.register_data([arr]); s.synchronize(); s.release_data(hd)
    t = (time.perf_counter() - t0) / 5
    print(f"register_data {name}: {arr.nbytes/t/1e9:.1f} GB/s ({arr.nbytes/2**20:.0f} MiB)")
    hd = s.register_data([arr])
    out = np.empty_like(arr) if name == "pageable" else h.pinned_empty(arr.shape, arr.dtype)
    t0 = time.perf_counter()
    for _ in range(5):
        s.fetch_data(hd, [out])
    t = (time.perf_counter() - t0) / 5
    print(f"fetch {name}: {arr.nbytes/t/1e9:.1f} GB/s")
    s.release_data(hd)
