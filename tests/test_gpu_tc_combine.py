"""The tensor-core (tcgen05, DFT-as-GEMM) SENSE combine, fft_combine_tc.cu.

HETRECO_COMBINE_TC=1 replaces the staged-map radix combine at 256-point lines
with 16 x 16 DFT stages on tcgen05.mma (3-term tf32 split).  Parity against
numpy's fp64 FFT and the oracle port of the reference chain
(fft_radix2_pass.cl.src:22-69 + complex_element_prod.cl.src:9-19 +
ximage_sum.cl.src:6-23); tolerance max|d| / max|ref| <= 1e-5 (north_star).
Covers ragged coil groups (C not a multiple of 8), shift, non-square ny and
the full C3 coil count.
"""
import numpy as np
import pytest

from oracle import oracle as o
from paper_1807_11830_b200 import hetreco as h

pytestmark = pytest.mark.gpu

TOL = 1e-5


def cplx(rng, *shape):
    return np.asfortranarray((rng.standard_normal(shape, dtype=np.float32)
                              + 1j * rng.standard_normal(shape, dtype=np.float32)).astype(np.complex64))


def relmax(a, ref):
    return float(np.abs(np.asarray(a) - ref).max() / max(float(np.abs(ref).max()), 1e-30))


@pytest.fixture(scope="module")
def s():
    sess = h.ComputeSession("gpu")
    yield sess
    sess.close()


def sens(s, Y, S, params=None):
    nx, ny, nc, nf = Y.shape
    hin = s.register_data(h.Data([Y, S], h.DataKind.KData))
    hout = s.allocate_data([((nx, ny, nf), np.complex64)], h.DataKind.XData)
    p = h.Process(s, "sens_recon").set_input(hin).set_output(hout).init(params or {})
    p.launch()
    M = s.fetch_data(hout).arrays[0]
    s.release_data(hin)
    s.release_data(hout)
    return M


@pytest.mark.parametrize("ny,nc,nf,shift", [(256, 32, 12, False), (256, 12, 13, True), (64, 5, 40, False),
                                            (128, 8, 20, True), (256, 1, 30, False)])
def test_tc_combine_vs_fp64(s, monkeypatch, ny, nc, nf, shift):
    rng = np.random.default_rng(ny * 7 + nc)
    Y = cplx(rng, 256, ny, nc, nf)
    S = cplx(rng, 256, ny, nc)
    monkeypatch.setenv("HETRECO_COMBINE_CP", "0")
    monkeypatch.setenv("HETRECO_COMBINE_TC", "1")
    M = sens(s, Y, S, {"shift": shift})
    monkeypatch.setenv("HETRECO_COMBINE_TC", "0")
    M0 = sens(s, Y, S, {"shift": shift})
    ax = (0, 1)
    Yr = np.fft.ifftshift(Y, axes=ax) if shift else Y
    Sr = np.fft.ifftshift(S, axes=ax) if shift else S
    ref = (np.conj(Sr.astype(np.complex128))[..., None] * np.fft.ifft2(Yr.astype(np.complex128), axes=ax)).sum(axis=2)
    if shift:
        ref = np.fft.fftshift(ref, axes=ax)
    err, err0 = relmax(M, ref), relmax(M0, ref)
    print(f"tc {err:.2e}  radix {err0:.2e}")
    assert err <= TOL
    assert relmax(M, M0) <= TOL


def test_tc_combine_vs_oracle_c3_frames(s, monkeypatch):
    """Two C3 frames (256^2 x 32 coils) against the C port of the reference chain."""
    rng = np.random.default_rng(3)
    Y = cplx(rng, 256, 256, 32, 2)
    S = cplx(rng, 256, 256, 32)
    monkeypatch.setenv("HETRECO_COMBINE_CP", "0")
    monkeypatch.setenv("HETRECO_COMBINE_TC", "1")
    M = sens(s, Y, S)
    assert relmax(M, o.sens_recon(Y, S)) <= TOL


@pytest.mark.parametrize("ny,nc,nf,shift", [(256, 32, 12, False), (256, 12, 13, True), (128, 8, 9, False)])
def test_ss_shared_twiddles_bitexact(s, monkeypatch, ny, nc, nf, shift):
    """HETRECO_SS_TWSMEM=1: the staged-map combine reading its pass-1 twiddles
    from a shared table is bit-identical to the register-twiddle kernel (same
    products, same order) and within tolerance of the reference chain."""
    rng = np.random.default_rng(ny + 3 * nc + nf)
    Y = cplx(rng, 256, ny, nc, nf)
    S = cplx(rng, 256, ny, nc)
    monkeypatch.setenv("HETRECO_COMBINE_CP", "0")
    monkeypatch.setenv("HETRECO_SS_TWSMEM", "1")
    M1 = sens(s, Y, S, {"shift": shift})
    monkeypatch.setenv("HETRECO_SS_TWSMEM", "0")
    M0 = sens(s, Y, S, {"shift": shift})
    assert np.array_equal(M1, M0)
    if not shift:
        assert relmax(M1, o.sens_recon(Y, S)) <= TOL


@pytest.mark.parametrize("ny,nc,nf,shift", [(256, 32, 12, False), (256, 12, 13, True), (128, 8, 9, False)])
def test_ss_shuffle_exchange_bitexact(s, monkeypatch, ny, nc, nf, shift):
    """HETRECO_SS_SHFL=1: the staged-map combine exchanging its 256-point lines
    by a warp-shuffle transpose is bit-identical to the shared-memory exchange."""
    rng = np.random.default_rng(ny + 5 * nc + nf)
    Y = cplx(rng, 256, ny, nc, nf)
    S = cplx(rng, 256, ny, nc)
    monkeypatch.setenv("HETRECO_COMBINE_CP", "0")
    monkeypatch.setenv("HETRECO_SS_SHFL", "1")
    M1 = sens(s, Y, S, {"shift": shift})
    monkeypatch.setenv("HETRECO_SS_SHFL", "0")
    M0 = sens(s, Y, S, {"shift": shift})
    assert np.array_equal(M1, M0)
