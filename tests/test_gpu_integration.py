"""Drop-in check: the UNMODIFIED reference session code (src/session.cpp,
layout.cpp, kernels.cpp ... compiled from /root/reference into oracle/_ref)
runs on the B200 through the maintainer-side adapter
integration/reference_cuda_backend.cpp over libhetreco_b200.so's C-ABI, and
produces results BIT-IDENTICAL to the same code on the reference CPU backend:
the builtin kernels reproduce the reference rounding exactly."""
import struct

import numpy as np
import pytest

from oracle import oracle as o

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (o.reference_available() and o.ref_on_b200_available()),
                                 reason="oracle/_ref not built (needs /root/reference at build time)")]


def beq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes(order="F") == b.tobytes(order="F")


def cplx(rng, *shape):
    return np.asfortranarray((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64))


def both(fn):
    cpu = fn()
    with o.use_reference_on_b200():
        gpu = fn()
    return cpu, gpu


def test_reference_session_on_b200_negate():
    rng = np.random.default_rng(0)
    x = rng.integers(0, 256, 100003).astype(np.uint8)
    cpu, gpu = both(lambda: o.ref_run_kernel("negate", x, struct.pack("<d", 200.0), x.size))
    assert beq(cpu, gpu)
    f = rng.random(4099).astype(np.float32)
    cpu, gpu = both(lambda: o.ref_run_kernel("negate", f, struct.pack("<d", 1.0), f.size))
    assert beq(cpu, gpu)


@pytest.mark.parametrize("shape", [(16, 8, 3), (64, 32, 2), (256, 256, 4)])
def test_reference_fft_plan_on_b200_bitexact(shape):
    x = cplx(np.random.default_rng(sum(shape)), *shape)
    for inverse in (True, False):
        cpu, gpu = both(lambda: o.ref_fft2d(x, inverse))
        assert beq(cpu, gpu)


@pytest.mark.parametrize("method", ["sens", "rss"])
def test_reference_recon_chain_on_b200_bitexact(method):
    rng = np.random.default_rng(4)
    Y = cplx(rng, 128, 64, 8, 3)
    S = cplx(rng, 128, 64, 8) if method == "sens" else None
    cpu, gpu = both(lambda: o.ref_recon(method, Y, S)[0])
    assert beq(cpu, gpu)
