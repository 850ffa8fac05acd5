"""Run the C3 SENSE (or RSS) recon a few times; print per-kernel device times.

Used under ncu (kernel captures) and for variant sweeps:
    HETRECO_COMBINE_VARIANT=1 HETRECO_CHUNK=2 python scripts/profile_c3.py --reps 20
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_11830_b200 import hetreco as h  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--method", default="sens_recon")
ap.add_argument("--nx", type=int, default=256)
ap.add_argument("--coils", type=int, default=32)
ap.add_argument("--frames", type=int, default=30)
ap.add_argument("--launches", type=int, default=3)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--timed", type=int, default=50, help="graph launches timed back to back")
ap.add_argument("--params", default="{}", help="process params as JSON, e.g. '{\"overlap\": true}'")
a = ap.parse_args()
nx = ny = a.nx
rng = np.random.default_rng(0)
Y = np.asfortranarray((rng.standard_normal((nx, ny, a.coils, a.frames), dtype=np.float32)
                       + 1j * rng.standard_normal((nx, ny, a.coils, a.frames), dtype=np.float32)).astype(np.complex64))
S = np.asfortranarray((rng.standard_normal((nx, ny, a.coils), dtype=np.float32) + 0j).astype(np.complex64))
s = h.ComputeSession("gpu")
if a.method == "sens_recon":
    hin = s.register_data(h.Data([Y, S], h.DataKind.KData))
    hout = s.allocate_data([((nx, ny, a.frames), np.complex64)])
else:
    hin = s.register_data(h.Data([Y], h.DataKind.KData))
    hout = s.allocate_data([((nx, ny, a.frames), np.float32)])
p = h.Process(s, a.method).set_input(hin).set_output(hout).init(json.loads(a.params))
for _ in range(a.launches):
    p.launch()
s.synchronize()
if a.reps:
    t = p.profile(a.reps)
    if len(t) % 2: t = t + [0.0]
    t1, t2 = sum(t[0::2]), sum(t[1::2])
    fy = nx * ny * a.coils * 8
    b1 = 2 * fy * a.frames
    b2 = fy * a.frames + (fy if a.method == "sens_recon" else 0) + nx * ny * a.frames * (8 if a.method == "sens_recon" else 4)
    s.timer_start()
    for _ in range(a.timed):
        p.launch()
    tg = s.timer_stop() / a.timed
    print(f"{a.method} {nx}x{ny}x{a.coils}x{a.frames} variant={os.environ.get('HETRECO_COMBINE_VARIANT', '-')} "
          f"chunk={os.environ.get('HETRECO_CHUNK', 'auto')} kernels={len(t)} | axis1 {t1*1e6:.1f} us {b1/t1/1e9:.0f} GB/s "
          f"| axis0+combine {t2*1e6:.1f} us {b2/max(t2, 1e-12)/1e9:.0f} GB/s | sum {(t1+t2)*1e6:.1f} us | graph {tg*1e6:.1f} us "
          f"= {a.frames/tg:.0f} frames/s")
elif a.timed:
    s.timer_start()
    for _ in range(a.timed):
        p.launch()
    tg = s.timer_stop() / a.timed
    print(f"{a.method} {nx}x{ny}x{a.coils}x{a.frames} params={a.params} graph {tg*1e6:.1f} us = {a.frames/tg:.0f} frames/s")
