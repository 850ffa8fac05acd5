"""C2 (256^2 x 8 coils x 1 frame, RSS) through the single-pass cluster kernel:
device us per launch for cluster sizes 8/16 and 1..8 clusters, beside the
two-pass chain.  One JSON line."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_11830_b200 import hetreco as h  # noqa: E402


def dev_time(s, fn, reps):
    for _ in range(5):
        fn()
    s.synchronize()
    s.timer_start()
    for _ in range(reps):
        fn()
    return s.timer_stop() / reps * 1e6


s = h.ComputeSession("gpu")
rng = np.random.default_rng(1)
Y2 = np.asfortranarray((rng.standard_normal((256, 256, 8, 1)) + 1j * rng.standard_normal((256, 256, 8, 1)))
                       .astype(np.complex64))
hk = s.register_data(h.Data([Y2], h.DataKind.KData))
hr = s.allocate_data([((256, 256, 1), np.float32)], h.DataKind.XData)
res = {}
p = h.Process(s, "rss_recon").set_input(hk).set_output(hr).init({"algorithm": "two_pass"})
res["two_pass"] = dev_time(s, p.launch, 300)
for cs in (8, 16):
    for mc in (1, 2, 4, 8):
        p = h.Process(s, "rss_recon").set_input(hk).set_output(hr).init(
            {"algorithm": "cluster", "cluster_size": cs, "max_clusters": mc})
        res[f"cl{cs}_k{mc}"] = round(dev_time(s, p.launch, 300), 2)
print(json.dumps(res))
