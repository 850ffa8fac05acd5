"""Mixed-radix (3*2^k, 5*2^k) transforms and reconstructions on the GPU --
the paper's 160 x 160 cine (SPEC.md:466-476 lists it as beyond the
reference's radix-2 FFT).

The reference has no non-power-of-two path, so the oracle is numpy's FFT in
float64 (np.fft), the same convention the oracle uses for fftshift: forward
unnormalised, inverse scaled by 1/(nx*ny).  Bar: max|d|/max|ref| <= 1e-5.
"""
import numpy as np
import pytest

from paper_1807_11830_b200 import hetreco as h

pytestmark = pytest.mark.gpu
TOL = 1e-5
AX = (0, 1)


def relmax(a, ref):
    return float(np.abs(np.asarray(a) - ref).max() / max(float(np.abs(ref).max()), 1e-30))


def cplx(rng, *shape):
    return np.asfortranarray((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64))


@pytest.fixture(scope="module")
def s():
    sess = h.ComputeSession("gpu")
    yield sess
    sess.close()


def run(s, kind, inputs, out_shape, out_dtype=np.complex64, params=None, kind_in=h.DataKind.KData):
    hin = s.register_data(h.Data(inputs, kind_in))
    hout = s.allocate_data([(out_shape, out_dtype)])
    p = h.Process(s, kind).set_input(hin).set_output(hout).init(params or {})
    p.launch()
    out = s.fetch_data(hout).arrays[0]
    s.release_data(hin)
    s.release_data(hout)
    return out


def np_sens(Y, S):
    X = np.fft.ifft2(Y.astype(np.complex128), axes=AX)
    return (np.conj(S.astype(np.complex128))[..., None] * X).sum(axis=2)


@pytest.mark.parametrize("shape", [(160, 160, 3), (96, 160, 2), (192, 96, 1), (320, 320, 1), (384, 64, 2),
                                   (160, 256, 2), (64, 320, 1), (384, 384, 2), (96, 96, 3), (192, 192, 2)])
@pytest.mark.parametrize("direction", ["forward", "inverse"])
def test_fft2d_mixed_vs_numpy(s, shape, direction):
    rng = np.random.default_rng(sum(shape))
    x = cplx(rng, *shape)
    y = run(s, "fft2d", [x], shape, params={"direction": direction})
    ref = np.fft.fft2(x.astype(np.complex128), axes=AX) if direction == "forward" else \
        np.fft.ifft2(x.astype(np.complex128), axes=AX)
    assert relmax(y, ref) <= TOL


def test_fft2d_mixed_shift_and_rejections(s):
    rng = np.random.default_rng(1)
    x = cplx(rng, 160, 96, 2)
    y = run(s, "fft2d", [x], x.shape, params={"direction": "inverse", "shift": True})
    ref = np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(x.astype(np.complex128), axes=AX), axes=AX), axes=AX)
    assert relmax(y, ref) <= TOL
    with pytest.raises(h.ShapeMismatch):  # the reference radix-2 algorithm stays power-of-two only
        run(s, "fft2d", [x], x.shape, params={"algorithm": "radix2"})
    with pytest.raises(h.ShapeMismatch):
        run(s, "fft2d", [cplx(rng, 100, 100)], (100, 100))


@pytest.mark.parametrize("nx,ny,nc,nf", [(160, 160, 8, 4), (96, 192, 4, 2), (320, 160, 3, 1), (96, 96, 5, 3),
                                        (192, 192, 4, 2), (320, 320, 3, 2), (384, 384, 2, 2)])
@pytest.mark.parametrize("shift", [False, True])
def test_recon_mixed_vs_numpy(s, nx, ny, nc, nf, shift):
    rng = np.random.default_rng(nx + ny + nc)
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    prm = {"shift": shift}
    Yr = np.fft.ifftshift(Y, axes=AX) if shift else Y
    Sr = np.fft.ifftshift(S, axes=AX) if shift else S
    ref = np_sens(Yr, Sr)
    rss = np.sqrt((np.abs(np.fft.ifft2(Yr.astype(np.complex128), axes=AX)) ** 2).sum(axis=2))
    if shift:
        ref = np.fft.fftshift(ref, axes=AX)
        rss = np.fft.fftshift(rss, axes=AX)
    for acc in ("fp32", "fp64"):
        M = run(s, "sens_recon", [Y, S], (nx, ny, nf), params=dict(prm, accumulate=acc))
        assert relmax(M, ref) <= TOL
    R = run(s, "rss_recon", [Y], (nx, ny, nf), np.float32, params=prm)
    assert relmax(R, rss) <= TOL


def test_cine_160_phantom_recovery(s):
    """The paper's case study size: a 160 x 160 x 8-coil x 16-frame cine built
    with the forward model recovers its ground truth (SPEC.md:457 identity)."""
    rng = np.random.default_rng(160)
    u = np.arange(160)[:, None] - 80.0
    v = np.arange(160)[None, :] - 80.0
    M = np.stack([np.exp(-((u - 20 * np.cos(f)) ** 2 + (v - 20 * np.sin(f)) ** 2) / 200.0) for f in range(16)],
                 axis=2).astype(np.complex64)
    G = np.abs(cplx(rng, 160, 160, 8)) + 0.1
    S = np.asfortranarray((G / np.sqrt((G ** 2).sum(axis=2, keepdims=True))).astype(np.complex64))
    Y = run(s, "sense_forward", [np.asfortranarray(M), S], (160, 160, 8, 16), kind_in=h.DataKind.XData)
    assert relmax(Y, np.fft.fft2((S[..., None] * M[:, :, None, :]).astype(np.complex128), axes=AX)) <= TOL
    R = run(s, "sens_recon", [Y, S], (160, 160, 16))
    assert np.linalg.norm(R - M) / np.linalg.norm(M) <= 1e-4


def test_sense_normal_and_streaming_mixed(s):
    rng = np.random.default_rng(7)
    M = cplx(rng, 160, 160, 2)
    S = cplx(rng, 160, 160, 4)
    mask = np.asfortranarray((rng.random((160, 160)) < 0.4).astype(np.float32))
    N = run(s, "sense_normal", [M, S, mask], (160, 160, 2), kind_in=h.DataKind.XData)
    Yf = np.fft.fft2(S.astype(np.complex128)[..., None] * M[:, :, None, :], axes=AX) * mask[:, :, None, None]
    assert relmax(N, np_sens(Yf, S)) <= TOL
    Y = cplx(rng, 160, 160, 4, 5)
    st = h.StreamingRecon(s, "sense", 160, 160, 4, 2, smaps=S)
    out = np.empty((160, 160, 5), np.complex64, order="F")
    st.run(Y, out)
    assert relmax(out, np_sens(Y, S)) <= TOL
