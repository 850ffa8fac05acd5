"""sense_normal at 256^2: the cluster front kernel (HETRECO_NORMAL_CLUSTER=1)
against the two-kernel front (default) -- bit-identity over coil/frame counts,
shift and mask; then C4 device us per launch for both."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_11830_b200 import hetreco as h  # noqa: E402

s = h.ComputeSession("gpu")


def run(M, S, mask, shift, env, reps=0):
    if env is None:
        os.environ.pop("HETRECO_NORMAL_CLUSTER", None)
    else:
        os.environ["HETRECO_NORMAL_CLUSTER"] = env
    arrays = [M, S] + ([mask] if mask is not None else [])
    hi = s.register_data(h.Data(arrays, h.DataKind.XData))
    ho = s.allocate_data([(M.shape, np.complex64)], h.DataKind.XData)
    p = h.Process(s, "sense_normal").set_input(hi).set_output(ho).init({"shift": shift})
    p.launch()
    out = s.fetch_data(ho).arrays[0]
    t = None
    if reps:
        for _ in range(20):
            p.launch()
        s.synchronize()
        s.timer_start()
        for _ in range(reps):
            p.launch()
        t = s.timer_stop() / reps * 1e6
    s.release_data(hi)
    s.release_data(ho)
    return out, t


rng = np.random.default_rng(4)
ok = True
for nc, nf, shift, use_mask in ((8, 1, False, True), (8, 1, True, True), (3, 2, False, False), (20, 1, True, True),
                                (32, 2, False, True), (1, 1, False, True)):
    M = np.asfortranarray((rng.standard_normal((256, 256, nf)) + 1j * rng.standard_normal((256, 256, nf))).astype(np.complex64))
    S = np.asfortranarray((rng.standard_normal((256, 256, nc)) + 1j * rng.standard_normal((256, 256, nc))).astype(np.complex64))
    mask = np.asfortranarray((rng.random((256, 256)) < 0.33).astype(np.float32)) if use_mask else None
    a, _ = run(M, S, mask, shift, "1")
    b, _ = run(M, S, mask, shift, None)
    same = np.array_equal(a, b)
    ok &= same
    print(f"coils {nc} frames {nf} shift {shift} mask {use_mask}: {'bit-identical' if same else 'DIFFERS %g' % np.abs(a - b).max()}")
M = np.asfortranarray((rng.standard_normal((256, 256, 1)) + 1j * rng.standard_normal((256, 256, 1))).astype(np.complex64))
S = np.asfortranarray((rng.standard_normal((256, 256, 8)) + 1j * rng.standard_normal((256, 256, 8))).astype(np.complex64))
mask = np.asfortranarray((rng.random((256, 256)) < 0.33).astype(np.float32))
for r in range(2):
    for env in ("1", None):
        _, t = run(M, S, mask, False, env, reps=500)
        print(f"C4 {'cluster front' if env else 'two-kernel front'}: {t:.2f} us/launch")
print("ALL OK" if ok else "MISMATCH")
