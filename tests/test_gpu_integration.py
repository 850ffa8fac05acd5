"""Drop-in check: the UNMODIFIED reference session code (src/session.cpp,
layout.cpp, kernels.cpp ... compiled from /root/reference into oracle/_ref)
runs on the B200 through the maintainer-side adapter
integration/reference_cuda_backend.cpp over libhetreco_b200.so's C-ABI, and
produces results BIT-IDENTICAL to the same code on the reference CPU backend:
the builtin kernels reproduce the reference rounding exactly.

Every test runs twice on the B200: with the precompiled sm_100a builtins,
and with the adapter reporting source support, in which case the reference's
own ComputeSession::load_builtin_kernels compiles its embedded kernel
sources through Backend::compile -> NVRTC."""
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


@pytest.fixture(params=[False, True], ids=["precompiled", "nvrtc-sources"])
def source_mode(request):
    return request.param


def both(fn, source=False):
    cpu = fn()
    with o.use_reference_on_b200(source):
        gpu = fn()
    return cpu, gpu


def test_reference_session_on_b200_negate(source_mode):
    rng = np.random.default_rng(0)
    x = rng.integers(0, 256, 100003).astype(np.uint8)
    cpu, gpu = both(lambda: o.ref_run_kernel("negate", x, struct.pack("<d", 200.0), x.size), source_mode)
    assert beq(cpu, gpu)
    f = rng.random(4099).astype(np.float32)
    cpu, gpu = both(lambda: o.ref_run_kernel("negate", f, struct.pack("<d", 1.0), f.size), source_mode)
    assert beq(cpu, gpu)


@pytest.mark.parametrize("shape", [(16, 8, 3), (64, 32, 2), (256, 256, 4)])
def test_reference_fft_plan_on_b200_bitexact(shape, source_mode):
    x = cplx(np.random.default_rng(sum(shape)), *shape)
    for inverse in (True, False):
        cpu, gpu = both(lambda: o.ref_fft2d(x, inverse), source_mode)
        assert beq(cpu, gpu)


@pytest.mark.parametrize("method", ["sens", "rss"])
def test_reference_recon_chain_on_b200_bitexact(method, source_mode):
    rng = np.random.default_rng(4)
    Y = cplx(rng, 128, 64, 8, 3)
    S = cplx(rng, 128, 64, 8) if method == "sens" else None
    cpu, gpu = both(lambda: o.ref_recon(method, Y, S)[0], source_mode)
    assert beq(cpu, gpu)


def relmax(a, ref):
    return float(np.abs(np.asarray(a) - ref).max() / max(float(np.abs(ref).max()), 1e-30))


@pytest.mark.parametrize("method", ["sens", "rss"])
def test_reference_session_launches_fused_recon_on_b200(method, source_mode):
    """The unmodified reference ComputeSession reaches the fused B200 chain:
    load_builtin_kernels registers "sens_recon" / "rss_recon" from the
    adapter's intrinsic bundle (precompiled mode) or next to the NVRTC-built
    builtins (source mode), and launch_kernel([Y, S] -> [M]) runs the two
    fused kernels instead of the 20-launch radix-2 chain.  Within the
    north_star 1e-5 of the reference CPU chain (fp32 coil accumulation)."""
    rng = np.random.default_rng(8)
    nx, ny, nc, nf = 256, 128, 8, 3
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc) if method == "sens" else None
    ref = o.ref_recon(method, Y, S)[0]  # reference chain on its CPU backend
    kernel = "sens_recon" if method == "sens" else "rss_recon"
    out = np.zeros((nx, ny, nf), np.complex64 if method == "sens" else np.float32, order="F")
    with o.use_reference_on_b200(source_mode):
        got = o.ref_run_kernel(kernel, Y, b"", nx * ny * nf, out_like=out, extra=S)
    assert relmax(got, ref) <= 1e-5
    with pytest.raises(Exception):  # the CPU reference backend has no such kernel
        o.ref_run_kernel(kernel, Y, b"", nx * ny * nf, out_like=out, extra=S)
