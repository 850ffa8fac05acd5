"""Host cost of Process::launch per "launch_timing" mode (C1 negate 512^2)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1807_11830_b200 import hetreco as h
s = h.ComputeSession("gpu")
x = np.asfortranarray(np.random.default_rng(0).random((512, 512), dtype=np.float32))
hx = s.register_data([x]); hy = s.allocate_data([((512, 512), np.float32)])
for mode in ("every", "sampled", "off"):
    p = h.Process(s, "negate").set_input(hx).set_output(hy).init({"max_value": 1.0, "launch_timing": mode})
    for _ in range(50): p.launch()
    s.synchronize()
    n = 4000
    t0 = time.perf_counter()
    s.timer_start()
    for _ in range(n): p.launch()
    dev = s.timer_stop() / n
    host = (time.perf_counter() - t0) / n
    st = p.stats()
    print(f"negate launch_timing={mode}: host {host*1e6:.2f} us/launch, device {dev*1e6:.2f} us/launch, "
          f"stats mean {st.mean_launch_seconds()*1e6:.2f} us, last {st.last_launch_seconds*1e6:.2f} us")
