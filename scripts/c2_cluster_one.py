"""One C2 rss_recon launch config for ncu: argv = cluster_size max_clusters (0 0 = two-pass)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_11830_b200 import hetreco as h  # noqa: E402

cs, mc = int(sys.argv[1]), int(sys.argv[2])
s = h.ComputeSession("gpu")
rng = np.random.default_rng(1)
Y2 = np.asfortranarray((rng.standard_normal((256, 256, 8, 1)) + 1j * rng.standard_normal((256, 256, 8, 1)))
                       .astype(np.complex64))
hk = s.register_data(h.Data([Y2], h.DataKind.KData))
hr = s.allocate_data([((256, 256, 1), np.float32)], h.DataKind.XData)
opts = {"algorithm": "two_pass"} if cs == 0 else {"algorithm": "cluster", "cluster_size": cs, "max_clusters": mc}
p = h.Process(s, "rss_recon").set_input(hk).set_output(hr).init(opts)
for _ in range(6):
    p.launch()
s.synchronize()
