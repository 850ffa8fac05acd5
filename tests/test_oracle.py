"""Pins the C oracle (oracle/hetreco_oracle.c) before anything is checked
against it:

* bit-exact against the golden vectors produced by the REAL reference
  library (tests/golden/make_golden.py -> oracle/_ref);
* SPEC.md's known-answer examples and properties;
* numpy fp64 as an independent cross-check of the FFT and chains;
* live against oracle/_ref when it is present (this container).
"""
import struct

import numpy as np
import pytest

from oracle import oracle as o


def beq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes(order="F") == b.tobytes(order="F")


def relmax(a, ref):
    ref = np.asarray(ref)
    return float(np.abs(np.asarray(a) - ref).max() / max(np.abs(ref).max(), 1e-30))


def cplx(rng, *shape):
    return np.asfortranarray(
        (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64))


# ---- golden vectors (reference outputs) ------------------------------------------

def test_negate_golden(golden):
    x = golden["negate_u8_in"]
    for mv in (255.0, 200.0, 300.5, -3.0):
        assert beq(o.negate(x, mv), golden[f"negate_u8_out_{mv}"])
    assert beq(o.negate(golden["negate_f32_in"], 1.0), golden["negate_f32_out"])


def test_fft_pass_golden(golden):
    x = golden["pass_in"]
    rev = np.array([0, 4, 2, 6, 1, 5, 3, 7], np.uint32)
    assert beq(o.fft_radix2_pass(x, np.zeros_like(x), 0, 8, 1, 0, 1.0, rev), golden["pass_mode0"])
    rev4 = np.array([0, 2, 1, 3], np.uint32)
    assert beq(o.fft_radix2_pass(None, x, 1, 4, 8, 0, 1.0, rev4), golden["pass_mode1"])
    tw = np.array([1, 0, 0.70710677, -0.70710677, 0, -1, -0.70710677, -0.70710677], np.float32)
    assert beq(o.fft_radix2_pass(None, x, 2, 8, 1, 2, 0.5, tw), golden["pass_mode2"])


@pytest.mark.parametrize("name", ["fft_16x8x3", "fft_4x4", "fft_32x32x2", "fft_2x64", "fft_256x1"])
def test_fft2d_golden(golden, name):
    x = golden[name + "_in"]
    assert beq(o.fft2d(x, True), golden[name + "_inv"])
    assert beq(o.fft2d(x, False), golden[name + "_fwd"])


def test_combine_golden(golden):
    x, s = golden["cep_x"], golden["cep_s"]
    assert beq(o.complex_element_prod(x, s, True), golden["cep_conj"])
    assert beq(o.complex_element_prod(x, s, False), golden["cep_noconj"])
    assert beq(o.ximage_sum(x), golden["xsum_out"])
    assert beq(o.rss_combine(x), golden["rss_out"])


def test_chains_golden(golden):
    assert beq(o.sens_recon(golden["sens_Y"], golden["sens_S"]), golden["sens_M"])
    assert beq(o.rss_recon(golden["rss_Y"]), golden["rss_R"])


# ---- SPEC.md known answers -----------------------------------------------------------

def test_spec_negate_examples():
    # SPEC.md:393-395
    out = o.negate(np.array([0, 255, 100], np.uint8), 255.0)
    assert out.tolist() == [255, 0, 155]


def test_spec_fft_examples():
    # forward of [1,1,1,1] -> [4,0,0,0]; delta -> ones
    ones = np.ones((4, 1), np.complex64)
    np.testing.assert_array_equal(o.fft2d(ones, False)[:, 0], [4, 0, 0, 0])
    delta = np.zeros((4, 1), np.complex64)
    delta[0] = 1
    np.testing.assert_array_equal(o.fft2d(delta, False)[:, 0], [1, 1, 1, 1])


def test_spec_fft_vs_naive_dft_and_inverse():
    # SPEC.md:404-405, 461, acceptance 2
    rng = np.random.default_rng(5)
    for _ in range(10):
        nx, ny = 2 ** rng.integers(2, 7), 2 ** rng.integers(2, 7)
        x = cplx(rng, nx, ny)
        fx = np.exp(-2j * np.pi * np.outer(np.arange(nx), np.arange(nx)) / nx)
        fy = np.exp(-2j * np.pi * np.outer(np.arange(ny), np.arange(ny)) / ny)
        naive = fx @ x.astype(np.complex128) @ fy.T
        f = o.fft2d(x, False)
        assert np.linalg.norm(f - naive) / np.linalg.norm(naive) <= 1e-4
        back = o.fft2d(f, True)
        assert np.linalg.norm(back - x) / np.linalg.norm(x) <= 1e-5
        # Parseval
        assert abs(np.vdot(x, x).real - np.vdot(f, f).real / (nx * ny)) <= 1e-4 * np.vdot(x, x).real


def test_spec_non_power_of_two_rejected():
    with pytest.raises(ValueError):
        o.fft2d(np.zeros((160, 160), np.complex64), True)


def test_spec_combine_examples():
    # SPEC.md:414 (1+2i)*conj(3+4i) = 11+2i; :421 {1,3} -> 4; :438 3-4-5
    x = np.array([1 + 2j], np.complex64).reshape(1, 1, 1)
    s = np.array([3 + 4j], np.complex64).reshape(1, 1, 1)
    assert o.complex_element_prod(x, s, True)[0, 0, 0] == 11 + 2j
    coils = np.array([1, 3], np.complex64).reshape(1, 1, 2)
    assert o.ximage_sum(coils)[0, 0] == 4
    m = np.array([3, 4j], np.complex64).reshape(1, 1, 2)
    assert o.rss_combine(m)[0, 0] == 5.0


def test_chains_vs_numpy():
    rng = np.random.default_rng(7)
    Y = cplx(rng, 64, 32, 4, 3)
    S = cplx(rng, 64, 32, 4)
    X = np.fft.ifft2(Y.astype(np.complex128), axes=(0, 1))
    M = (np.conj(S)[..., None] * X).sum(axis=2)
    assert relmax(o.sens_recon(Y, S), M) <= 1e-6
    R = np.sqrt((np.abs(X) ** 2).sum(axis=2))
    assert relmax(o.rss_recon(Y), R) <= 1e-6


def test_sense_forward_model_roundtrip():
    # Y_i = F(S_i . M) with sum|S|^2 = 1 -> sens_recon recovers M <= 1e-4
    rng = np.random.default_rng(11)
    nx, ny, nc, nf = 32, 32, 4, 2
    G = cplx(rng, nx, ny, nc)
    S = (G / np.sqrt((np.abs(G) ** 2).sum(axis=2, keepdims=True))).astype(np.complex64)
    M = cplx(rng, nx, ny, nf)
    Y = np.fft.fft2(S[..., None] * M[:, :, None, :], axes=(0, 1)).astype(np.complex64)
    rec = o.sens_recon(np.asfortranarray(Y), S)
    assert np.linalg.norm(rec - M) / np.linalg.norm(M) <= 1e-4


# ---- live cross-check against the compiled reference -------------------------------------

@pytest.mark.skipif(not o.reference_available(), reason="oracle/_ref not built")
def test_port_matches_reference_live():
    rng = np.random.default_rng(3)
    Y = cplx(rng, 64, 16, 3, 2)
    S = cplx(rng, 64, 16, 3)
    assert beq(o.sens_recon(Y, S), o.ref_recon("sens", Y, S)[0])
    assert beq(o.rss_recon(Y), o.ref_recon("rss", Y)[0])
    x = rng.random(5000).astype(np.float32)
    assert beq(o.negate(x, 0.75), o.ref_run_kernel("negate", x, struct.pack("<d", 0.75), x.size))


def test_sense_forward_oracle_vs_numpy():
    rng = np.random.default_rng(31)
    M = cplx(rng, 32, 32, 2)
    S = cplx(rng, 32, 32, 3)
    mask = (rng.random((32, 32)) < 0.4).astype(np.float32)
    Y = o.sense_forward(M, S, mask)
    ref = np.fft.fft2(S[..., None].astype(np.complex128) * M[:, :, None, :], axes=(0, 1)) * mask[:, :, None, None]
    assert relmax(Y, ref) <= 1e-6
    # adjoint identity <E m, y> == <m, E^H y> (E^H = nx*ny * sens_recon)
    y = cplx(rng, 32, 32, 3, 2) * mask[:, :, None, None]
    lhs = np.vdot(o.sense_forward(M, S, mask), y)
    rhs = np.vdot(M, o.sens_recon(np.asfortranarray(y.astype(np.complex64)), S)) * 32 * 32
    assert abs(lhs - rhs) <= 1e-4 * abs(lhs)


# ---- BASELINE shapes: one C3 frame (256^2 x 32) and one C5 frame (512^2 x 32) ------------

def _large_cases():
    import json
    import os
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    return json.load(open(os.path.join(here, "large_shapes.json")))["cases"]


def _large_inputs(case):
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    import synth
    nx, ny, nc, nf, seed = case["nx"], case["ny"], case["coils"], case["frames"], case["seed"]
    return synth.cplx(seed, nx, ny, nc, nf), synth.cplx(seed + 1, nx, ny, nc)


@pytest.mark.parametrize("case", _large_cases(), ids=lambda c: c["name"])
def test_port_matches_reference_golden_at_baseline_shapes(case):
    """The C port reproduces the reference's output bytes (SHA-256 from
    tests/golden/make_golden_large.py, run against oracle/_ref) at the
    headline shapes, not only at 32x16: radix-2 plan of
    fft_radix2_pass.cl.src:22-69 over 256/512 points, conj-S sum of
    ximage_sum.cl.src:6-23 / rss_combine.cl.src:5-20 over 32 coils."""
    import hashlib
    Y, S = _large_inputs(case)
    out = o.sens_recon(Y, S) if case["method"] == "sens" else o.rss_recon(Y)
    assert hashlib.sha256(out.tobytes(order="F")).hexdigest() == case["sha256"]


@pytest.mark.skipif(not o.reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("shape", [(256, 256, 32, 1), (512, 512, 32, 1)])
def test_port_matches_reference_live_baseline_shapes(shape):
    nx, ny, nc, nf = shape
    rng = np.random.default_rng(nx + 7)
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    assert beq(o.sens_recon(Y, S), o.ref_recon("sens", Y, S)[0])
    assert beq(o.rss_recon(Y), o.ref_recon("rss", Y)[0])
