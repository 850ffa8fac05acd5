"""GPU parity at the BASELINE shapes.

* One C3 frame (256^2 x 32 coils) and one C5 frame (512^2 x 32 coils), SENSE
  and RSS, against the fixtures made from the real reference
  (tests/golden/large_shapes.json: SHA-256 of the reference output, which the
  C port reproduces bit for bit -- tests/test_oracle.py -- plus a strided
  sample of its values).
* C5 streaming: 512^2 x 32 coils, 9 frames in 2-frame chunks (ragged tail)
  from pinned memory, RSS and SENSE, against the oracle port
  (rss_combine.cl.src:5-20 / ximage_sum.cl.src:6-23 over the radix-2 plan of
  fft_radix2_pass.cl.src:22-69).
Tolerance max|d| / max|ref| <= 1e-5 (north_star).
"""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

from oracle import oracle as o
from paper_1807_11830_b200 import hetreco as h

pytestmark = pytest.mark.gpu

TOL = 1e-5
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, GOLD)
import synth  # noqa: E402

CASES = json.load(open(os.path.join(GOLD, "large_shapes.json")))
STRIDE = CASES["sample_stride"]


def relmax(a, ref):
    return float(np.abs(np.asarray(a) - ref).max() / max(float(np.abs(ref).max()), 1e-30))


@pytest.fixture(scope="module")
def s():
    sess = h.ComputeSession("gpu")
    yield sess
    sess.close()


@pytest.mark.parametrize("case", CASES["cases"], ids=lambda c: c["name"])
@pytest.mark.parametrize("accumulate", ["fp32", "fp64"])
def test_recon_vs_reference_golden_at_baseline_shapes(s, case, accumulate):
    nx, ny, nc, nf = case["nx"], case["ny"], case["coils"], case["frames"]
    Y = synth.cplx(case["seed"], nx, ny, nc, nf)
    S = synth.cplx(case["seed"] + 1, nx, ny, nc)
    sens = case["method"] == "sens"
    hin = s.register_data(h.Data([Y, S] if sens else [Y], h.DataKind.KData))
    hout = s.allocate_data([((nx, ny, nf), np.complex64 if sens else np.float32)], h.DataKind.XData)
    p = h.Process(s, "sens_recon" if sens else "rss_recon").set_input(hin).set_output(hout)
    p.init({"accumulate": accumulate})
    p.launch()
    got = s.fetch_data(hout).arrays[0]
    s.release_data(hin)
    s.release_data(hout)
    flat = got.reshape(-1, order="F")[::STRIDE]
    sample = (np.array(case["sample_re"]) + 1j * np.array(case["sample_im"])) if sens else np.array(case["sample"])
    assert float(np.abs(flat - sample).max()) <= TOL * case["max_abs"]
    # full comparison against the port, whose bytes equal the reference's
    ref = o.sens_recon(Y, S) if sens else o.rss_recon(Y)
    assert hashlib.sha256(ref.tobytes(order="F")).hexdigest() == case["sha256"]
    assert relmax(got, ref) <= TOL


@pytest.mark.parametrize("method", ["rss", "sense"])
def test_c5_streaming_ragged_chunks_vs_oracle(s, method):
    """C5 geometry streamed from pinned memory: 9 frames in 2-frame chunks
    (the tail chunk is 1 frame, with its own launch shapes); frames of the
    first chunk, a middle chunk and the tail checked against the port."""
    n, nc, nf, chunk = 512, 32, 9, 2
    Y = h.pinned_empty((n, n, nc, nf), np.complex64)
    Y[...] = synth.cplx(77, n, n, nc, nf)
    S = synth.cplx(78, n, n, nc) if method == "sense" else None
    out = h.pinned_empty((n, n, nf), np.complex64 if method == "sense" else np.float32)
    out[...] = np.nan
    st = h.StreamingRecon(s, method, n, n, nc, chunk, S)
    st.run(Y, out)
    assert np.isfinite(out).all()
    for f in (0, 1, 5, 8):
        Yf = np.asfortranarray(Y[..., f:f + 1])
        ref = o.sens_recon(Yf, S) if method == "sense" else o.rss_recon(Yf)
        assert relmax(out[..., f:f + 1], ref) <= TOL, f
    # re-run into a fresh buffer: same bits
    again = h.pinned_empty(out.shape, out.dtype)
    st.run(Y, again)
    assert again.tobytes() == out.tobytes()
    # and the streamed frames equal the resident process on the same chunking
    kind = "sens_recon" if method == "sense" else "rss_recon"
    hk = s.register_data(h.Data([np.asfortranarray(Y[..., 8:9])] + ([S] if S is not None else []), h.DataKind.KData))
    ho = s.allocate_data([((n, n, 1), out.dtype)], h.DataKind.XData)
    h.Process(s, kind).set_input(hk).set_output(ho).init().launch()
    assert relmax(s.fetch_data(ho).arrays[0], out[..., 8:9]) <= TOL
    s.release_data(hk)
    s.release_data(ho)
