"""Run the C3 SENSE (or RSS) recon a few times; print per-kernel device times.

Used under ncu (kernel captures) and for variant sweeps:
    HETRECO_COMBINE_VARIANT=1 python scripts/profile_c3.py --reps 20
"""
import argparse
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
p = h.Process(s, a.method).set_input(hin).set_output(hout).init()
for _ in range(a.launches):
    p.launch()
s.synchronize()
if a.reps:
    t = p.profile(a.reps)
    fy = nx * ny * a.coils * 8
    b1 = 2 * fy * a.frames
    b2 = fy * a.frames + (fy if a.method == "sens_recon" else 0) + nx * ny * a.frames * (8 if a.method == "sens_recon" else 4)
    print(f"variant={os.environ.get('HETRECO_COMBINE_VARIANT', '0')} lpb={os.environ.get('HETRECO_LINES_PER_BLOCK', '128')} "
          f"axis1 {t[0]*1e6:.1f} us {b1/t[0]/1e9:.0f} GB/s | axis0+combine {t[1]*1e6:.1f} us {b2/t[1]/1e9:.0f} GB/s "
          f"| total {(t[0]+t[1])*1e6:.1f} us = {a.frames/(t[0]+t[1]):.0f} frames/s")
