"""C4 normal operator (256^2 x 8 coils, random mask): a few launches, for ncu."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_11830_b200 import hetreco as h  # noqa: E402

s = h.ComputeSession("gpu")
rng = np.random.default_rng(1)
n, C = 256, 8
M = np.asfortranarray((rng.standard_normal((n, n, 1)) + 1j * rng.standard_normal((n, n, 1))).astype(np.complex64))
S = np.asfortranarray((rng.standard_normal((n, n, C)) + 1j * rng.standard_normal((n, n, C))).astype(np.complex64))
mask = np.asfortranarray((rng.random((n, n)) < 0.33).astype(np.float32))
hn = s.register_data(h.Data([M, S, mask], h.DataKind.XData))
ho = s.allocate_data([((n, n, 1), np.complex64)], h.DataKind.XData)
p = h.Process(s, "sense_normal").set_input(hn).set_output(ho).init()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    p.launch()
s.synchronize()
