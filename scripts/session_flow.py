"""Breakdown of the reference-arm flow on the B200 session API (register
pageable k-space + maps, launch sens_recon, fetch, release), and the
pageable H2D options: the pinned staging ring (csrc/host/host_stager.cpp) vs
registering the caller's pages (cudaHostRegister) per call.
    python scripts/session_flow.py  ->  lines of ms per phase"""
import ctypes
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1807_11830_b200 import hetreco as h  # noqa: E402

rng = np.random.default_rng(0)
NX, NC, NF = 256, 32, 30
Y = np.asfortranarray((rng.standard_normal((NX, NX, NC, NF), dtype=np.float32) + 0j).astype(np.complex64))
S = np.asfortranarray((rng.standard_normal((NX, NX, NC), dtype=np.float32) + 0j).astype(np.complex64))
s = h.ComputeSession("gpu")
hout = s.allocate_data([((NX, NX, NF), np.complex64)])
M = np.empty((NX, NX, NF), np.complex64, order="F")
p = None
rows = []
for it in range(12):
    t0 = time.perf_counter()
    hk = s.register_data(h.Data([Y, S], h.DataKind.KData))
    s.synchronize()
    t1 = time.perf_counter()
    if p is None:
        p = h.Process(s, "sens_recon").set_input(hk).set_output(hout).init()
    else:
        p.set_input(hk)
    t2 = time.perf_counter()
    p.launch()
    s.synchronize()
    t3 = time.perf_counter()
    s.fetch_data(hout, [M])
    t4 = time.perf_counter()
    s.release_data(hk)
    t5 = time.perf_counter()
    rows.append([1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3), 1e3 * (t5 - t4), 1e3 * (t5 - t0)])
med = [statistics.median(c) for c in zip(*rows[2:])]
print(json.dumps({"flow_ms_median": dict(zip(["register", "set_input", "launch+rebind", "fetch", "release", "total"],
                                              [round(x, 3) for x in med])),
                  "env": {k: v for k, v in os.environ.items() if k.startswith("HETRECO_STAGER")}}))

# cudaHostRegister of the caller's pages per call (what a register-in-place path would pay)
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if cudart is None:
    import glob
    cands = glob.glob("/usr/local/cuda*/lib64/libcudart.so*")
    cudart = ctypes.CDLL(cands[0]) if cands else None
if cudart is not None:
    ptr = ctypes.c_void_p(Y.ctypes.data)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        rc = cudart.cudaHostRegister(ptr, ctypes.c_size_t(Y.nbytes), 0)
        t1 = time.perf_counter()
        hd = s.register_data(h.Data([Y], h.DataKind.KData))
        s.synchronize()
        t2 = time.perf_counter()
        cudart.cudaHostUnregister(ptr)
        t3 = time.perf_counter()
        s.release_data(hd)
        ts.append((rc, 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2)))
    print(json.dumps({"host_register_ms": [round(x[1], 2) for x in ts], "dma_ms": [round(x[2], 2) for x in ts],
                      "unregister_ms": [round(x[3], 2) for x in ts], "rc": ts[0][0], "bytes": Y.nbytes}))
