"""Bit-identity of two libhetreco_b200.so builds on the mixed-radix paths
(sens_recon, rss_recon, fft2d both directions, sense_normal):
    python scripts/lib_bitexact.py <old.so> <new.so>"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIZES = (96, 160, 192, 320, 384)


def run(lib, out):
    from paper_1807_11830_b200 import hetreco as h
    h.LIB_PATH = os.path.abspath(lib)
    s = h.ComputeSession("gpu")
    res = {}
    for n in SIZES:
        rng = np.random.default_rng(n)
        nc, nf = 8, 3
        Y = np.asfortranarray((rng.standard_normal((n, n, nc, nf)) + 1j * rng.standard_normal((n, n, nc, nf))).astype(np.complex64))
        S = np.asfortranarray((rng.standard_normal((n, n, nc)) + 1j * rng.standard_normal((n, n, nc))).astype(np.complex64))
        mask = np.asfortranarray((rng.random((n, n)) < 0.4).astype(np.float32))
        for name, arrays, oshape, odt in (("sens_recon", [Y, S], (n, n, nf), np.complex64),
                                           ("rss_recon", [Y], (n, n, nf), np.float32)):
            for shift in (False, True):
                hi = s.register_data(h.Data(arrays, h.DataKind.KData))
                ho = s.allocate_data([(oshape, odt)])
                h.Process(s, name).set_input(hi).set_output(ho).init({"shift": shift}).launch()
                res[f"{name}_{n}_{int(shift)}"] = s.fetch_data(ho).arrays[0]
                s.release_data(hi)
                s.release_data(ho)
        for d in ("inverse", "forward"):
            hi = s.register_data([Y])
            ho = s.allocate_data([(Y.shape, np.complex64)])
            h.Process(s, "fft2d").set_input(hi).set_output(ho).init({"direction": d}).launch()
            res[f"fft2d_{d}_{n}"] = s.fetch_data(ho).arrays[0]
            s.release_data(hi)
            s.release_data(ho)
        M = np.asfortranarray(Y[:, :, 0, :1])
        hi = s.register_data(h.Data([M, S, mask], h.DataKind.XData))
        ho = s.allocate_data([((n, n, 1), np.complex64)])
        h.Process(s, "sense_normal").set_input(hi).set_output(ho).init().launch()
        res[f"sense_normal_{n}"] = s.fetch_data(ho).arrays[0]
    np.savez(out, **res)


if __name__ == "__main__":
    if sys.argv[1] == "--run":
        run(sys.argv[2], sys.argv[3])
        sys.exit(0)
    a, b = sys.argv[1], sys.argv[2]
    for lib, out in ((a, "/tmp/bx_a.npz"), (b, "/tmp/bx_b.npz")):
        subprocess.run([sys.executable, __file__, "--run", lib, out], check=True)
    A, B = np.load("/tmp/bx_a.npz"), np.load("/tmp/bx_b.npz")
    bad = [k for k in A.files if not np.array_equal(A[k], B[k])]
    print(f"{len(A.files)} outputs compared; {'all bit-identical' if not bad else 'DIFFER: ' + ', '.join(bad)}")
