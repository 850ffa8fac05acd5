"""SENSE forward model E = P F S and normal operator E^H E on the GPU
(the iterative-reconstruction building block, C4's
"IFFT/FFT + coil combine chain launched 100x after one init()")."""
import numpy as np
import pytest

from oracle import oracle as o
from paper_1807_11830_b200 import hetreco as h

pytestmark = pytest.mark.gpu
TOL = 1e-5


def relmax(a, ref):
    return float(np.abs(np.asarray(a) - ref).max() / max(float(np.abs(ref).max()), 1e-30))


def cplx(rng, *shape):
    return np.asfortranarray((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64))


@pytest.fixture(scope="module")
def s():
    sess = h.ComputeSession("gpu")
    yield sess
    sess.close()


def run(s, kind, inputs, out_shape, params=None):
    hin = s.register_data(h.Data(inputs, h.DataKind.XData))
    hout = s.allocate_data([(out_shape, np.complex64)])
    p = h.Process(s, kind).set_input(hin).set_output(hout).init(params or {})
    p.launch()
    out = s.fetch_data(hout).arrays[0]
    return out, p, hin, hout


@pytest.mark.parametrize("n,nc,nf", [(256, 8, 3), (64, 4, 2), (128, 1, 1), (512, 2, 1), (16, 3, 2)])
@pytest.mark.parametrize("masked", [False, True])
def test_sense_forward_vs_oracle(s, n, nc, nf, masked):
    rng = np.random.default_rng(n + nc)
    M = cplx(rng, n, n, nf)
    S = cplx(rng, n, n, nc)
    inputs = [M, S]
    mask = None
    if masked:
        mask = np.asfortranarray((rng.random((n, n)) < 0.35).astype(np.float32))
        inputs.append(mask)
    Y, *_ = run(s, "sense_forward", inputs, (n, n, nc, nf))
    assert relmax(Y, o.sense_forward(M, S, mask)) <= TOL


@pytest.mark.parametrize("n,nc,nf", [(256, 8, 3), (64, 4, 2), (512, 2, 1)])
@pytest.mark.parametrize("masked", [False, True])
def test_sense_normal_vs_oracle(s, n, nc, nf, masked):
    rng = np.random.default_rng(2 * n + nc)
    M = cplx(rng, n, n, nf)
    S = cplx(rng, n, n, nc)
    inputs = [M, S]
    mask = None
    if masked:
        mask = np.asfortranarray((rng.random((n, n)) < 0.35).astype(np.float32))
        inputs.append(mask)
    out, *_ = run(s, "sense_normal", inputs, (n, n, nf))
    assert relmax(out, o.sense_normal(M, S, mask)) <= TOL


def test_sense_normal_identity_without_mask(s):
    # sum_c |S_c|^2 = 1 and P = 1  ->  E^H E = identity
    rng = np.random.default_rng(5)
    G = cplx(rng, 128, 128, 6)
    S = np.asfortranarray((G / np.sqrt((np.abs(G) ** 2).sum(axis=2, keepdims=True))).astype(np.complex64))
    M = cplx(rng, 128, 128, 4)
    out, *_ = run(s, "sense_normal", [M, S], (128, 128, 4))
    assert relmax(out, M) <= TOL


def test_sense_shift_consistency(s):
    """With shift, forward(shift) = fftshift(F(ifftshift(S m))) and the normal
    operator stays E^H E (the shifts cancel inside the k-space roundtrip)."""
    rng = np.random.default_rng(8)
    n, nc = 64, 3
    M = cplx(rng, n, n, 2)
    S = cplx(rng, n, n, nc)
    mask = np.asfortranarray((rng.random((n, n)) < 0.5).astype(np.float32))
    Y, *_ = run(s, "sense_forward", [M, S, mask], (n, n, nc, 2), {"shift": True})
    X = np.fft.ifftshift(S[..., None] * M[:, :, None, :], axes=(0, 1))
    ref = np.fft.fftshift(np.fft.fft2(X.astype(np.complex128), axes=(0, 1)), axes=(0, 1)) * mask[:, :, None, None]
    assert relmax(Y, ref) <= TOL
    out, *_ = run(s, "sense_normal", [M, S, mask], (n, n, 2), {"shift": True})
    Xs = np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(ref, axes=(0, 1)), axes=(0, 1)), axes=(0, 1))
    ref_n = (np.conj(S)[..., None] * Xs).sum(axis=2)
    assert relmax(out, ref_n) <= TOL


def test_c4_hundred_launches_after_one_init(s):
    """C4: the normal-operator chain launched 100x after one init()."""
    rng = np.random.default_rng(4)
    n, nc = 256, 8
    M = cplx(rng, n, n, 1)
    S = cplx(rng, n, n, nc)
    mask = np.asfortranarray((rng.random((n, n)) < 0.3).astype(np.float32))
    out, p, hin, hout = run(s, "sense_normal", [M, S, mask], (n, n, 1))
    s.reset_counters()
    for _ in range(99):
        p.launch()
    st = p.stats()
    assert st.init_calls == 1 and st.launches == 100
    assert s.counters() == {"host_to_device": 0, "device_to_host": 0}
    assert relmax(s.fetch_data(hout).arrays[0], o.sense_normal(M, S, mask)) <= TOL


@pytest.mark.parametrize("nx,ny", [(64, 32), (32, 128), (256, 16)])
def test_sense_forward_rectangular(s, nx, ny):
    """Unmasked forward model on rectangular images (generic column pass);
    masked / normal-operator models stay square-only."""
    rng = np.random.default_rng(nx * 3 + ny)
    M = cplx(rng, nx, ny, 2)
    S = cplx(rng, nx, ny, 3)
    Y, *_ = run(s, "sense_forward", [M, S], (nx, ny, 3, 2))
    assert relmax(Y, o.sense_forward(M, S)) <= TOL
    with pytest.raises(h.ShapeMismatch):
        run(s, "sense_forward", [M, S, np.ones((nx, ny), np.float32)], (nx, ny, 3, 2))
    with pytest.raises(h.ShapeMismatch):
        run(s, "sense_normal", [M, S], (nx, ny, 2))


@pytest.mark.parametrize("n,nc,nf,points", [(256, 8, 1, "8"), (256, 8, 2, "16"), (64, 3, 2, "8"), (128, 5, 1, "16")])
def test_sense_normal_fused_cooperative(s, monkeypatch, n, nc, nf, points):
    """The opt-in single cooperative kernel (fft_sense_normal.cu, measured
    slower than the three-kernel graph: profiles/round2_c4.md) stays exact."""
    monkeypatch.setenv("HETRECO_NORMAL_FUSED", "1")
    monkeypatch.setenv("HETRECO_NORMAL_POINTS", points)
    rng = np.random.default_rng(3 * n + nc)
    M = cplx(rng, n, n, nf)
    S = cplx(rng, n, n, nc)
    mask = np.asfortranarray((rng.random((n, n)) < 0.4).astype(np.float32))
    out, *_ = run(s, "sense_normal", [M, S, mask], (n, n, nf))
    assert relmax(out, o.sense_normal(M, S, mask)) <= TOL


@pytest.mark.parametrize("nc,nf,shift,masked", [(8, 1, False, True), (8, 1, True, True), (3, 2, False, False),
                                                (20, 1, True, True)])
def test_sense_normal_cluster_front_bitexact(s, monkeypatch, nc, nf, shift, masked):
    """HETRECO_NORMAL_CLUSTER=1 (fft_sense_cluster.cu): expand, x-FFT, DSMEM
    transpose and the masked y round trip in one 16-CTA-cluster kernel, bit-
    identical to the two-kernel front (20 coil images exceed the resident
    clusters, so clusters loop over images)."""
    rng = np.random.default_rng(nc * 10 + nf)
    M = cplx(rng, 256, 256, nf)
    S = cplx(rng, 256, 256, nc)
    inputs = [M, S] + ([np.asfortranarray((rng.random((256, 256)) < 0.4).astype(np.float32))] if masked else [])
    monkeypatch.setenv("HETRECO_NORMAL_CLUSTER", "1")
    a = run(s, "sense_normal", inputs, (256, 256, nf), {"shift": shift})[0]
    monkeypatch.delenv("HETRECO_NORMAL_CLUSTER")
    b = run(s, "sense_normal", inputs, (256, 256, nf), {"shift": shift})[0]
    assert np.array_equal(a, b)
