"""Single-pass cluster recon vs the two-pass chain (and the oracle on a
sample): parity + device time.  python scripts/cluster_check.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as o  # noqa: E402
from paper_1807_11830_b200 import hetreco as h  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def run(s, method, Y, S, params, timed=50):
    nx, ny, nc, nf = Y.shape
    arrs = [Y, S] if method == "sens_recon" else [Y]
    hin = s.register_data(h.Data(arrs, h.DataKind.KData))
    dt = np.complex64 if method == "sens_recon" else np.float32
    hout = s.allocate_data([((nx, ny, nf), dt)])
    p = h.Process(s, method).set_input(hin).set_output(hout).init(params)
    p.launch()
    s.synchronize()
    M = s.fetch_data(hout).arrays[0]
    p.launch(); p.launch()
    s.timer_start()
    for _ in range(timed):
        p.launch()
    t = s.timer_stop() / timed
    return M, t


s = h.ComputeSession("gpu")
rng = np.random.default_rng(3)
for method in ["sens_recon", "rss_recon"]:
    for (nc, nf, mc, shift) in [(32, 30, 0, False), (32, 30, 0, True), (8, 1, 0, False), (5, 3, 7, False),
                                (32, 30, 100, False), (3, 2, 1, True)]:
        Y = np.asfortranarray((rng.standard_normal((256, 256, nc, nf), dtype=np.float32)
                               + 1j * rng.standard_normal((256, 256, nc, nf), dtype=np.float32)).astype(np.complex64))
        S = np.asfortranarray((rng.standard_normal((256, 256, nc), dtype=np.float32)
                               + 1j * rng.standard_normal((256, 256, nc), dtype=np.float32)).astype(np.complex64))
        prm = {"shift": shift}
        Mt, tt = run(s, method, Y, S, dict(prm, algorithm="two_pass"))
        res = {}
        for cs in (8, 16):
            res[cs] = run(s, method, Y, S, dict(prm, algorithm="cluster", max_clusters=mc, cluster_size=cs))
        Mc, tc = res[16]
        M8, t8 = res[8]
        fs = [0, nf - 1]
        Ys = np.asfortranarray(Y[..., fs])
        ax = (0, 1)
        if shift:
            Ys = np.asfortranarray(np.fft.ifftshift(Ys, axes=ax))
        if method == "sens_recon":
            Sx = np.asfortranarray(np.fft.ifftshift(S, axes=ax)) if shift else S
            ref = o.sens_recon(Ys, Sx)
        else:
            ref = o.rss_recon(Ys)
        if shift:
            ref = np.fft.fftshift(ref, axes=ax)
        print(f"{method} C={nc} F={nf} max_clusters={mc} shift={shift}: cl8 {t8*1e6:.1f} us "
              f"err8 {rel(M8, Mt):.1e} | cl16 {tc*1e6:.1f} us "
              f"({nf/tc:.0f} fr/s) two_pass {tt*1e6:.1f} us | cluster vs two_pass {rel(Mc, Mt):.2e} "
              f"bitexact={np.array_equal(Mc, Mt)} | cluster vs oracle {rel(Mc[..., fs], ref):.2e}", flush=True)
