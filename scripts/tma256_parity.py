"""Bit-identity of the 256^2 axis-1 TMA ring variants against the cp.async ring (sens_recon, C3-like shape)."""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    from paper_1807_11830_b200 import hetreco as h
    rng = np.random.default_rng(3)
    Y = np.asfortranarray((rng.standard_normal((256, 256, 32, 5)) + 1j * rng.standard_normal((256, 256, 32, 5))).astype(np.complex64))
    S = np.asfortranarray((rng.standard_normal((256, 256, 32)) + 1j * rng.standard_normal((256, 256, 32))).astype(np.complex64))
    s = h.ComputeSession("gpu")
    hin = s.register_data(h.Data([Y, S], h.DataKind.KData))
    hout = s.allocate_data([((256, 256, 5), np.complex64)])
    for shift in (False, True):
        p = h.Process(s, "sens_recon").set_input(hin).set_output(hout).init({"shift": shift})
        p.launch()
        np.save(f"{sys.argv[1]}_{int(shift)}.npy", s.fetch_data(hout).arrays[0])
    sys.exit(0)
cases = {"cpasync": {}, "tma2x32": {"HETRECO_STRIDED_TMA": "1"}}
for k in (2, 3, 4):
    cases[f"tma{k}x16"] = {"HETRECO_STRIDED_TMA": "1", "HETRECO_TMA_TX256": "16", "HETRECO_TMA_STAGES256": str(k)}
for name, env in cases.items():
    subprocess.run([sys.executable, __file__, f"/tmp/p_{name}"], env=dict(os.environ, **env), check=True)
for name in cases:
    for sh in (0, 1):
        a, b = np.load(f"/tmp/p_cpasync_{sh}.npy"), np.load(f"/tmp/p_{name}_{sh}.npy")
        print(name, "shift", sh, "bit-identical" if np.array_equal(a, b) else f"DIFFERS max {np.abs(a-b).max()}")
