"""Small-config latency A/B (C1 negate, C2 rss_recon, C4 sense_normal) with
and without programmatic (PDL) graph edges: HETRECO_PDL=0|1 python
scripts/small_configs.py -> one JSON line of device us per launch."""
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


def main():
    s = h.ComputeSession("gpu")
    rng = np.random.default_rng(1)
    res = {"pdl": os.environ.get("HETRECO_PDL", "1")}
    x = np.asfortranarray(rng.random((512, 512), dtype=np.float32))
    hx, hy = s.register_data([x]), s.allocate_data([((512, 512), np.float32)])
    p = h.Process(s, "negate").set_input(hx).set_output(hy).init({"max_value": 1.0})
    res["C1_us"] = dev_time(s, p.launch, 500)
    Y2 = np.asfortranarray((rng.standard_normal((256, 256, 8, 1)) + 1j * rng.standard_normal((256, 256, 8, 1)))
                           .astype(np.complex64))
    hk = s.register_data(h.Data([Y2], h.DataKind.KData))
    hr = s.allocate_data([((256, 256, 1), np.float32)], h.DataKind.XData)
    for algo in ("two_pass", "cluster"):
        try:
            p2 = h.Process(s, "rss_recon").set_input(hk).set_output(hr).init({"algorithm": algo})
            res[f"C2_{algo}_us"] = dev_time(s, p2.launch, 500)
            res[f"C2_{algo}_kernels_us"] = [round(v * 1e6, 2) for v in p2.profile(reps=50)]
        except h.HetrecoError as e:
            res[f"C2_{algo}_us"] = str(e)
    S2 = np.asfortranarray((rng.standard_normal((256, 256, 8)) + 1j * rng.standard_normal((256, 256, 8)))
                           .astype(np.complex64))
    M2 = np.asfortranarray(Y2[:, :, 0, :])
    mask = np.asfortranarray((rng.random((256, 256)) < 0.33).astype(np.float32))
    hn = s.register_data(h.Data([M2, S2, mask], h.DataKind.XData))
    ho = s.allocate_data([((256, 256, 1), np.complex64)], h.DataKind.XData)
    p4 = h.Process(s, "sense_normal").set_input(hn).set_output(ho).init()
    res["C4_us"] = dev_time(s, p4.launch, 500)
    res["C4_kernels_us"] = [round(v * 1e6, 2) for v in p4.profile(reps=50)]
    Y3 = np.asfortranarray((rng.standard_normal((256, 256, 32, 30), dtype=np.float32) + 0j).astype(np.complex64))
    S3 = np.asfortranarray((rng.standard_normal((256, 256, 32), dtype=np.float32) + 0j).astype(np.complex64))
    h3 = s.register_data(h.Data([Y3, S3], h.DataKind.KData))
    o3 = s.allocate_data([((256, 256, 30), np.complex64)], h.DataKind.XData)
    p3 = h.Process(s, "sens_recon").set_input(h3).set_output(o3).init()
    res["C3_us"] = dev_time(s, p3.launch, 200)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
