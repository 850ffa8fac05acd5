"""GPU parity: the CUDA path (through the C-ABI) against the oracle.

Bar (BASELINE.json north_star): negate, layout/indexing and the builtin
reference-ABI kernels are BIT-EXACT with the reference; the fused FFT and the
recon chains are within max|d|/max|ref| <= 1e-5 (fp32) of the oracle.
"""
import struct

import numpy as np
import pytest

from oracle import oracle as o
from paper_1807_11830_b200 import hetreco as h

pytestmark = pytest.mark.gpu

TOL = 1e-5  # max|d| / max|ref|, north_star


def relmax(a, ref):
    ref = np.asarray(ref)
    return float(np.abs(np.asarray(a) - ref).max() / max(float(np.abs(ref).max()), 1e-30))


def beq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes(order="F") == b.tobytes(order="F")


def cplx(rng, *shape):
    return np.asfortranarray((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64))


@pytest.fixture(scope="module")
def s():
    sess = h.ComputeSession("gpu")
    sess.load_builtin_kernels()
    yield sess
    sess.close()


def run_process(s, kind, inputs, out_shapes, params=None, kind_in=h.DataKind.KData):
    hin = s.register_data(h.Data(inputs, kind_in))
    hout = s.allocate_data(out_shapes, h.DataKind.XData)
    p = h.Process(s, kind).set_input(hin).set_output(hout).init(params or {})
    p.launch()
    res = s.fetch_data(hout).arrays
    s.release_data(hin)
    s.release_data(hout)
    return res, p


# ---- device, session plumbing -------------------------------------------------------------

def test_device_is_b200_class(s):
    d = s.device()
    assert d.device_type == h.DeviceType.Gpu and d.vendor == "NVIDIA"
    assert d.api_version.startswith("10."), d.api_version  # sm_100
    assert d.base_alignment_bytes == 256


def test_register_fetch_roundtrip_and_counters(s):
    rng = np.random.default_rng(1)
    arrays = [rng.integers(0, 255, (7, 3), dtype=np.uint8), rng.standard_normal((5,)).astype(np.float64),
              cplx(rng, 4, 4, 2), np.arange(11, dtype=np.int32)]
    s.reset_counters()
    hd = s.register_data(h.Data(arrays, h.DataKind.Generic))
    back = s.fetch_data(hd).arrays
    for a, b in zip(arrays, back):
        assert beq(a, b)
    assert s.counters() == {"host_to_device": 1, "device_to_host": 1}
    _, words = h.pack_layout(arrays)
    assert s.fetch_header_bytes(hd) == words.tobytes()
    s.release_data(hd)
    with pytest.raises(h.UnknownHandle):
        s.fetch_data(hd)
    with pytest.raises(h.UnknownHandle):
        s.release_data(hd)


def test_copy_array_and_shape_checks(s):
    a = np.arange(12, dtype=np.float32).reshape(3, 4, order="F")
    h1 = s.register_data([a, np.zeros(3, np.float32)])
    h2 = s.register_data([np.zeros(2, np.int32), np.zeros((3, 4), np.float32)])
    s.copy_array(h1, 0, h2, 1)
    assert beq(s.fetch_data(h2).arrays[1], a)
    with pytest.raises(h.ShapeMismatch):
        s.copy_array(h1, 1, h2, 1)
    with pytest.raises(h.InvalidArgument):
        s.copy_array(h1, 5, h2, 1)


def test_foreign_handle_rejected(s):
    other = h.ComputeSession("gpu")
    hd = other.register_data([np.zeros(4, np.float32)])
    with pytest.raises(h.UnknownHandle):
        s.fetch_data(hd)
    other.close()


def test_backend_capacity_and_ranges():
    b = h.CudaBackend(0, capacity_bytes=1 << 20)
    buf = b.allocate(1 << 19)
    with pytest.raises(h.AllocationFailure):
        b.allocate(1 << 20)
    with pytest.raises(h.InvalidArgument):
        b.upload(buf, (1 << 19) - 4, b"12345678")
    b.upload(buf, 8, b"abcd")
    assert b.download(buf, 0, 16) == b"\0" * 8 + b"abcd" + b"\0" * 4
    b.release(buf)
    with pytest.raises(h.UnknownHandle):
        b.release(buf)
    b.close()


def test_header_shadow_after_device_writes(s):
    """The backend keeps host shadows of uploaded layout headers so the fused
    layer-1 kernels read their shapes without a device round trip.  A header
    buffer last written by the device (D2D copy) and then patched by a partial
    upload must be read back from the device, not from a zero-assumed shadow."""
    rng = np.random.default_rng(5)
    nx, ny, nc, nf = 64, 32, 3, 2
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    hk = s.register_data(h.Data([Y, S], h.DataKind.KData))
    ho = s.allocate_data([((nx, ny, nf), np.complex64)])
    hin, hout = s.fetch_header_bytes(hk), s.fetch_header_bytes(ho)
    b = h.CudaBackend(0)
    lay = s.layout_of(hk)
    data = b.allocate(lay.total_bytes)
    for arr, rec in zip((Y, S), lay.records):
        b.upload(data, rec.offset_bytes, np.asfortranarray(arr).reshape(-1, order="F").view(np.uint8))
    staging = b.allocate(len(hin))
    b.upload(staging, 0, hin)                 # whole upload: shadowed
    hdr = b.allocate(len(hin))
    b.copy(staging, 0, hdr, 0, len(hin))      # device-written: no shadow
    b.upload(hdr, 0, hin[:8])                 # partial patch (same record count)
    out = b.allocate(nx * ny * nf * 8)
    ohdr = b.allocate(len(hout))
    b.upload(ohdr, 0, hout)
    b.execute("sens_recon", data, hdr, out, ohdr, b"", nx * ny * nf)
    b.synchronize()
    M = np.frombuffer(b.download(out, 0, nx * ny * nf * 8), np.complex64).reshape((nx, ny, nf), order="F")
    assert relmax(M, o.sens_recon(Y, S)) <= TOL
    b.close()
    s.release_data(hk)
    s.release_data(ho)


def test_builtin_registry(s):
    assert set(s.kernel_names()) == {"negate", "fft_radix2_pass", "complex_element_prod", "ximage_sum",
                                     "rss_combine", "matrix_add", "sens_recon", "rss_recon"}
    with pytest.raises(h.CompileError):  # source units go to NVRTC (tests/test_source_kernels.py)
        s.load_kernels([("broken.cl.src", "this is not a kernel")])
    assert len(s.kernel_names()) == 8
    hd = s.register_data([np.zeros(4, np.float32)])
    with pytest.raises(h.UnknownKernel):
        s.launch_kernel("nonexistent", hd, hd, b"", 4)
    with pytest.raises(h.InvalidArgument):
        s.launch_kernel("negate", hd, hd, struct.pack("<d", 1.0), 0)


# ---- reference-ABI kernels: bit-exact with the golden vectors ------------------------------------

def launch_one(s, name, inputs, out_like, params, gsize, in_place=False):
    hin = s.register_data(inputs)
    hout = hin if in_place else s.register_data([np.zeros_like(out_like)])
    s.launch_kernel(name, hin, hout, params, gsize)
    return s.fetch_data(hout).arrays[0]


def test_negate_kernel_bitexact(s, golden):
    x = golden["negate_u8_in"]
    for mv in (255.0, 200.0, 300.5, -3.0):
        got = launch_one(s, "negate", [x], x, struct.pack("<d", mv), x.size)
        assert beq(got, golden[f"negate_u8_out_{mv}"])
    f = golden["negate_f32_in"]
    assert beq(launch_one(s, "negate", [f], f, struct.pack("<d", 1.0), f.size), golden["negate_f32_out"])


def test_fft_radix2_pass_kernel_bitexact(s, golden):
    x = golden["pass_in"]
    rev = np.array([0, 4, 2, 6, 1, 5, 3, 7], np.uint32)
    p0 = struct.pack("<IIQQQfI", 0, 0, 8, 1, 0, 1.0, 0) + rev.tobytes()
    assert beq(launch_one(s, "fft_radix2_pass", [x], x, p0, x.size), golden["pass_mode0"])
    rev4 = np.array([0, 2, 1, 3], np.uint32)
    p1 = struct.pack("<IIQQQfI", 1, 0, 4, 8, 0, 1.0, 0) + rev4.tobytes()
    assert beq(launch_one(s, "fft_radix2_pass", [x], x, p1, x.size, in_place=True), golden["pass_mode1"])
    tw = np.array([1, 0, 0.70710677, -0.70710677, 0, -1, -0.70710677, -0.70710677], np.float32)
    p2 = struct.pack("<IIQQQfI", 2, 0, 8, 1, 2, 0.5, 0) + tw.tobytes()
    assert beq(launch_one(s, "fft_radix2_pass", [x], x, p2, x.size // 2, in_place=True), golden["pass_mode2"])


def test_combine_kernels_bitexact(s, golden):
    x, sm = golden["cep_x"], golden["cep_s"]
    assert beq(launch_one(s, "complex_element_prod", [x, sm], x, struct.pack("<I", 1), x.size), golden["cep_conj"])
    assert beq(launch_one(s, "complex_element_prod", [x, sm], x, struct.pack("<I", 0), x.size),
               golden["cep_noconj"])
    assert beq(launch_one(s, "ximage_sum", [x], golden["xsum_out"], b"", 16 * 8 * 3), golden["xsum_out"])
    assert beq(launch_one(s, "rss_combine", [x], golden["rss_out"], b"", 16 * 8 * 3), golden["rss_out"])


def test_matrix_add_kernel(s):
    rng = np.random.default_rng(2)
    a = rng.standard_normal(1000).astype(np.float32)
    b = rng.standard_normal(1000).astype(np.float32)
    assert beq(launch_one(s, "matrix_add", [a, b], a, b"", a.size), o.matrix_add(a, b))


# ---- processes ------------------------------------------------------------------------------------

def test_negate_process_bitexact_c1(s):
    rng = np.random.default_rng(1)
    x = np.asfortranarray(rng.random((512, 512), dtype=np.float32))
    (got,), p = run_process(s, "negate", [x], [((512, 512), np.float32)], {"max_value": 1.0})
    assert beq(got, o.negate(x, 1.0))
    u = np.asfortranarray(rng.integers(0, 256, (512, 509), dtype=np.uint8))  # ragged tail
    (got,), _ = run_process(s, "negate", [u], [((512, 509), np.uint8)])
    assert beq(got, o.negate(u, 255.0))
    (got,), _ = run_process(s, "negate", [u], [((512, 509), np.uint8)], {"max_value": 100.0})
    assert beq(got, o.negate(u, 100.0))


def test_negate_in_place_and_involution(s):
    x = np.array([0, 100, 255], np.uint8)
    hd = s.register_data([x])
    p = h.Process(s, "negate").set_input(hd).set_output(hd).init()
    p.launch()
    assert s.fetch_data(hd).arrays[0].tolist() == [255, 155, 0]
    p.launch()
    assert s.fetch_data(hd).arrays[0].tolist() == [0, 100, 255]


FFT_SHAPES = [(4, 4, 1), (16, 8, 3), (2, 64, 1), (256, 1, 1), (1, 32, 2), (32, 32, 2), (64, 128, 2),
              (128, 256, 1), (256, 256, 4), (512, 512, 2), (1024, 64, 1), (8, 2048, 1), (4096, 4, 1)]


@pytest.mark.parametrize("shape", FFT_SHAPES, ids=lambda t: "x".join(map(str, t)))
@pytest.mark.parametrize("direction", ["inverse", "forward"])
def test_fft2d_process_vs_oracle(s, shape, direction):
    rng = np.random.default_rng(sum(shape))
    x = cplx(rng, *shape)
    (got,), _ = run_process(s, "fft2d", [x], [(shape, np.complex64)], {"direction": direction})
    ref = o.fft2d(x, direction == "inverse")
    assert relmax(got, ref) <= TOL


@pytest.mark.parametrize("shape", [(16, 8, 3), (64, 32, 1), (256, 256, 1)])
def test_fft2d_radix2_algorithm_is_bitexact(s, shape):
    rng = np.random.default_rng(4)
    x = cplx(rng, *shape)
    for inverse in (True, False):
        (got,), _ = run_process(s, "fft2d", [x], [(shape, np.complex64)],
                                {"direction": "inverse" if inverse else "forward", "algorithm": "radix2"})
        assert beq(got, o.fft2d(x, inverse))


def test_fft2d_golden(s, golden):
    for name in ("fft_16x8x3", "fft_4x4", "fft_32x32x2", "fft_2x64", "fft_256x1"):
        x = golden[name + "_in"]
        (got,), _ = run_process(s, "fft2d", [x], [(x.shape, np.complex64)], {"direction": "inverse"})
        assert relmax(got, golden[name + "_inv"]) <= TOL


def test_fft2d_shift_is_exact_permutation(s):
    rng = np.random.default_rng(9)
    x = cplx(rng, 64, 32, 3)
    (plain,), _ = run_process(s, "fft2d", [x], [(x.shape, np.complex64)], {"direction": "inverse"})
    xs = np.asfortranarray(np.fft.ifftshift(x, axes=(0, 1)))
    (ref_shifted_in,), _ = run_process(s, "fft2d", [xs], [(x.shape, np.complex64)], {"direction": "inverse"})
    (got,), _ = run_process(s, "fft2d", [x], [(x.shape, np.complex64)], {"direction": "inverse", "shift": True})
    assert beq(got, np.asfortranarray(np.fft.fftshift(ref_shifted_in, axes=(0, 1))))
    ref = np.fft.fftshift(o.fft2d(np.asfortranarray(np.fft.ifftshift(x, axes=(0, 1))), True), axes=(0, 1))
    assert relmax(got, ref) <= TOL
    del plain


def test_fft2d_rejects_bad_shapes_and_params(s):
    x = np.zeros((100, 100), np.complex64)  # neither 2^k nor a mixed-radix side
    hin = s.register_data([x])
    hout = s.allocate_data([((100, 100), np.complex64)])
    with pytest.raises(h.ShapeMismatch):
        h.Process(s, "fft2d").set_input(hin).set_output(hout).init()
    x = np.zeros((160, 160), np.complex64)  # mixed radix: stockham only
    hin = s.register_data([x])
    hout = s.allocate_data([((160, 160), np.complex64)])
    with pytest.raises(h.ShapeMismatch):
        h.Process(s, "fft2d").set_input(hin).set_output(hout).init({"algorithm": "radix2"})
    y = s.register_data([np.zeros((16, 16), np.complex64)])
    z = s.allocate_data([((16, 8), np.complex64)])
    with pytest.raises(h.ShapeMismatch):
        h.Process(s, "fft2d").set_input(y).set_output(z).init()
    w = s.allocate_data([((16, 16), np.complex64)])
    with pytest.raises(h.InvalidParams):
        h.Process(s, "fft2d").set_input(y).set_output(w).init({"direction": "sideways"})
    with pytest.raises(h.InvalidParams):
        h.Process(s, "fft2d").set_input(y).set_output(w).init({"dirction": "inverse"})
    with pytest.raises(h.UnsupportedElementType):
        f = s.register_data([np.zeros((16, 16), np.float32)])
        h.Process(s, "fft2d").set_input(f).set_output(w).init()


def test_process_lifecycle(s):
    x = cplx(np.random.default_rng(0), 32, 32)
    hin = s.register_data([x])
    hout = s.allocate_data([((32, 32), np.complex64)])
    p = h.Process(s, "fft2d").set_input(hin).set_output(hout)
    with pytest.raises(h.NotInitialized):
        p.launch()
    p.init({"direction": "inverse"})
    with pytest.raises(h.AlreadyInitialized):
        p.init()
    s.reset_counters()
    for _ in range(100):
        p.launch()
    st = p.stats()
    assert st.init_calls == 1 and st.launches == 100
    assert st.total_launch_seconds > 0 and st.init_seconds > 0
    assert s.counters() == {"host_to_device": 0, "device_to_host": 0}
    assert relmax(s.fetch_data(hout).arrays[0], o.fft2d(x, True)) <= TOL
    # re-point the input between launches (SPEC process: re-point -> new handle consumed)
    x2 = cplx(np.random.default_rng(1), 32, 32)
    hin2 = s.register_data([x2])
    p.set_input(hin2)
    p.launch()
    assert relmax(s.fetch_data(hout).arrays[0], o.fft2d(x2, True)) <= TOL


@pytest.mark.parametrize("dims", [(16, 8, 4, 3), (32, 16, 1, 2), (64, 64, 8, 1), (256, 256, 8, 1),
                                  (128, 64, 3, 5), (4, 4, 2, 2), (512, 512, 4, 1), (256, 256, 32, 2)],
                         ids=lambda t: "x".join(map(str, t)))
def test_sens_recon_vs_oracle(s, dims):
    nx, ny, nc, nf = dims
    rng = np.random.default_rng(nx + nc)
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    (M,), _ = run_process(s, "sens_recon", [Y, S], [((nx, ny, nf), np.complex64)])
    assert relmax(M, o.sens_recon(Y, S)) <= TOL


@pytest.mark.parametrize("params", [{"accumulate": "fp64"}, {"accumulate": "fp64", "prefetch": False},
                                    {"prefetch": False}, {"chunk_frames": 3}, {"chunk_frames": 1, "shift": False}],
                         ids=lambda d: ",".join(f"{k}={v}" for k, v in d.items()))
@pytest.mark.parametrize("method", ["sens_recon", "rss_recon"])
def test_recon_variants_vs_oracle(s, params, method):
    nx, ny, nc, nf = 256, 256, 6, 7
    rng = np.random.default_rng(77)
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    if method == "sens_recon":
        (M,), _ = run_process(s, method, [Y, S], [((nx, ny, nf), np.complex64)], params)
        assert relmax(M, o.sens_recon(Y, S)) <= TOL
    else:
        (R,), _ = run_process(s, method, [Y], [((nx, ny, nf), np.float32)], params)
        assert relmax(R, o.rss_recon(Y)) <= TOL


def test_recon_fp64_accumulation_is_bitexact_combine(s):
    """With fp64 accumulation the fused combine repeats ximage_sum's arithmetic
    (fp32 products, fp64 coil-ordered sum): fed the same X it matches the
    reference-ABI kernels bit for bit, so chain == fused up to the FFT only."""
    rng = np.random.default_rng(78)
    nx, ny, nc, nf = 64, 64, 5, 2
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    (M,), _ = run_process(s, "sens_recon", [Y, S], [((nx, ny, nf), np.complex64)], {"accumulate": "fp64"})
    (X,), _ = run_process(s, "fft2d", [Y], [((nx, ny, nc, nf), np.complex64)], {"direction": "inverse"})
    ref = o.ximage_sum(o.complex_element_prod(X, S, True))
    assert relmax(M, ref) <= 1e-6


def test_recon_rejects_bad_params(s):
    Y = np.zeros((16, 16, 2, 1), np.complex64)
    S = np.zeros((16, 16, 2), np.complex64)
    hin = s.register_data(h.Data([Y, S], h.DataKind.KData))
    hout = s.allocate_data([((16, 16, 1), np.complex64)])
    with pytest.raises(h.InvalidParams):
        h.Process(s, "sens_recon").set_input(hin).set_output(hout).init({"accumulate": "fp16"})
    with pytest.raises(h.InvalidParams):
        h.Process(s, "sens_recon").set_input(hin).set_output(hout).init({"chunk_frames": -1})
    bad = s.allocate_data([((16, 8, 1), np.complex64)])
    with pytest.raises(h.ShapeMismatch):
        h.Process(s, "sens_recon").set_input(hin).set_output(bad).init()
    smaps_wrong = s.register_data(h.Data([Y, np.zeros((16, 16, 3), np.complex64)], h.DataKind.KData))
    with pytest.raises(h.ShapeMismatch):
        h.Process(s, "sens_recon").set_input(smaps_wrong).set_output(hout).init()


@pytest.mark.parametrize("dims", [(16, 8, 4, 3), (256, 256, 8, 1), (128, 32, 1, 4), (512, 512, 4, 1)],
                         ids=lambda t: "x".join(map(str, t)))
def test_rss_recon_vs_oracle(s, dims):
    nx, ny, nc, nf = dims
    rng = np.random.default_rng(nx * 3 + nc)
    Y = cplx(rng, nx, ny, nc, nf)
    (R,), _ = run_process(s, "rss_recon", [Y], [((nx, ny, nf), np.float32)])
    ref = o.rss_recon(Y)
    assert relmax(R, ref) <= TOL
    assert (R >= 0).all()


def test_recon_golden(s, golden):
    Y, S = golden["sens_Y"], golden["sens_S"]
    (M,), _ = run_process(s, "sens_recon", [Y, S], [((32, 16, 3), np.complex64)])
    assert relmax(M, golden["sens_M"]) <= TOL
    (R,), _ = run_process(s, "rss_recon", [golden["rss_Y"]], [((32, 16, 3), np.float32)])
    assert relmax(R, golden["rss_R"]) <= TOL


def test_spec_recon_examples(s):
    # N=1, S=1 -> M = IFFT(Y); Y=0 -> M=0; 3-4-5 RSS pixel
    rng = np.random.default_rng(8)
    Y = cplx(rng, 16, 16, 1, 2)
    S = np.ones((16, 16, 1), np.complex64)
    (M,), _ = run_process(s, "sens_recon", [Y, S], [((16, 16, 2), np.complex64)])
    assert relmax(M, o.fft2d(Y[:, :, 0, :], True)) <= TOL
    Z = np.zeros((16, 16, 2, 1), np.complex64)
    (M0,), _ = run_process(s, "sens_recon", [Z, np.ones((16, 16, 2), np.complex64)], [((16, 16, 1), np.complex64)])
    assert not M0.any()
    img = np.zeros((8, 8, 2, 1), np.complex64)
    img[3, 5, 0, 0], img[3, 5, 1, 0] = 3.0, 4.0j
    Yk = np.asfortranarray(np.fft.fft2(img, axes=(0, 1)).astype(np.complex64))
    (R,), _ = run_process(s, "rss_recon", [Yk], [((8, 8, 1), np.float32)])
    assert abs(R[3, 5, 0] - 5.0) <= 1e-5


def test_sense_forward_model_roundtrip(s):
    # SPEC.md:430 / acceptance 1: recovers M_true within rel-L2 1e-4
    rng = np.random.default_rng(12)
    nx, ny, nc, nf = 128, 128, 8, 16
    G = cplx(rng, nx, ny, nc)
    S = np.asfortranarray((G / np.sqrt((np.abs(G) ** 2).sum(axis=2, keepdims=True))).astype(np.complex64))
    M = cplx(rng, nx, ny, nf)
    Y = np.asfortranarray(np.fft.fft2(S[..., None] * M[:, :, None, :], axes=(0, 1)).astype(np.complex64))
    (rec,), _ = run_process(s, "sens_recon", [Y, S], [((nx, ny, nf), np.complex64)])
    assert np.linalg.norm(rec - M) / np.linalg.norm(M) <= 1e-4


def test_sens_recon_shift(s):
    rng = np.random.default_rng(21)
    Y = cplx(rng, 64, 32, 4, 2)
    S = cplx(rng, 64, 32, 4)
    (M,), _ = run_process(s, "sens_recon", [Y, S], [((64, 32, 2), np.complex64)], {"shift": True})
    X = np.fft.fftshift(o.fft2d(np.asfortranarray(np.fft.ifftshift(Y, axes=(0, 1))), True), axes=(0, 1))
    ref = o.ximage_sum(o.complex_element_prod(np.asfortranarray(X), S, True))
    assert relmax(M, ref) <= TOL


def test_chain_matches_fused_and_oracle(s):
    # chain(fft2d INVERSE, complex_element_prod conj, ximage_sum) == SimpleMRIRecon
    rng = np.random.default_rng(5)
    nx, ny, nc, nf = 64, 32, 4, 3
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    hk = s.register_data(h.Data([Y], h.DataKind.KData))
    hx = s.register_data(h.Data([np.zeros_like(Y), S], h.DataKind.XData))
    hp = s.allocate_data([((nx, ny, nc, nf), np.complex64)], h.DataKind.XData)
    hm = s.allocate_data([((nx, ny, nf), np.complex64)], h.DataKind.XData)
    f = h.Process(s, "fft2d").set_input(hk).set_output(hx)
    c = h.Process(s, "complex_element_prod").set_input(hx).set_output(hp)
    x = h.Process(s, "ximage_sum").set_input(hp).set_output(hm)
    f.init({"direction": "inverse"})
    c.init({"conjugate_s": True})
    comp = h.chain(s, "simple_mri_recon", [f, c, x])
    comp.init()
    s.reset_counters()
    for _ in range(3):
        comp.launch()
    assert s.counters() == {"host_to_device": 0, "device_to_host": 0}  # zero-copy chaining
    M = s.fetch_data(hm).arrays[0]
    assert s.counters() == {"host_to_device": 0, "device_to_host": 1}
    assert relmax(M, o.sens_recon(Y, S)) <= TOL
    assert comp.stats().launches == 3


def test_chain_mismatch(s):
    a = s.register_data([np.zeros((8, 8), np.complex64)])
    b = s.allocate_data([((8, 8), np.complex64)])
    c = s.allocate_data([((8, 8), np.complex64)])
    p1 = h.Process(s, "fft2d").set_input(a).set_output(b)
    p2 = h.Process(s, "fft2d").set_input(c).set_output(a)
    with pytest.raises(h.ChainMismatch):
        h.chain(s, "bad", [p1, p2])


def test_chain_stage_error_carries_index(s):
    a = s.register_data([np.zeros((8, 8), np.complex64)])
    b = s.allocate_data([((8, 8), np.complex64)])
    c = s.allocate_data([((8, 4), np.complex64)])
    p1 = h.Process(s, "fft2d").set_input(a).set_output(b)
    p2 = h.Process(s, "fft2d").set_input(b).set_output(c)
    comp = h.chain(s, "bad", [p1, p2])
    with pytest.raises(h.ChainStageError) as e:
        comp.init()
    assert "stage 1" in str(e.value)


def test_streaming_matches_process(s):
    rng = np.random.default_rng(17)
    nx, ny, nc, nf = 128, 128, 8, 10
    Y = h.pinned_empty((nx, ny, nc, nf), np.complex64)
    Y[...] = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    out = h.pinned_empty((nx, ny, nf), np.complex64)
    st = h.StreamingRecon(s, "sense", nx, ny, nc, 3, S)  # ragged last chunk (10 = 3+3+3+1)
    st.run(Y, out)
    assert relmax(out, o.sens_recon(np.asarray(Y), S)) <= TOL
    outr = h.pinned_empty((nx, ny, nf), np.float32)
    h.StreamingRecon(s, "rss", nx, ny, nc, 4).run(Y, outr)
    assert relmax(outr, o.rss_recon(np.asarray(Y))) <= TOL


def test_c3_full_size_properties(s):
    """Full BASELINE C3 size (256^2 x 32 coils x 30 frames): oracle parity on
    frames sampled from the same launch, plus linearity."""
    rng = np.random.default_rng(30)
    nx, ny, nc, nf = 256, 256, 32, 30
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    hin = s.register_data(h.Data([Y, S], h.DataKind.KData))
    hout = s.allocate_data([((nx, ny, nf), np.complex64)], h.DataKind.XData)
    p = h.Process(s, "sens_recon").set_input(hin).set_output(hout).init()
    p.launch()
    M = s.fetch_data(hout).arrays[0]
    for f in (0, 17, 29):
        ref = o.sens_recon(np.asfortranarray(Y[..., f:f + 1]), S)
        assert relmax(M[..., f:f + 1], ref) <= TOL
    # linearity: recon(2.5 Y) == 2.5 recon(Y)
    h2 = s.register_data(h.Data([np.asfortranarray(Y * np.float32(2.5)), S], h.DataKind.KData))
    p.set_input(h2)
    p.launch()
    M2 = s.fetch_data(hout).arrays[0]
    assert relmax(M2, 2.5 * M) <= TOL


# ---- single-pass cluster kernel (algorithm="cluster", fft_cluster.cu) -------------------

@pytest.mark.parametrize("cluster_size", [8, 16])
@pytest.mark.parametrize("method", ["sens_recon", "rss_recon"])
@pytest.mark.parametrize("nc,nf,max_clusters,shift", [(6, 5, 0, False), (5, 3, 7, False), (4, 3, 5, True),
                                                       (3, 2, 1, True), (7, 1, 3, False)],
                         ids=lambda v: str(v))
def test_cluster_recon_vs_oracle(s, method, cluster_size, nc, nf, max_clusters, shift):
    """TMA tile loads + DSMEM transpose + register coil accumulation, including
    frames split across clusters (max_clusters not dividing frames*coils: the
    last-arriving piece adds the partial sums)."""
    rng = np.random.default_rng(100 + nc * 10 + nf)
    Y = cplx(rng, 256, 256, nc, nf)
    S = cplx(rng, 256, 256, nc)
    prm = {"algorithm": "cluster", "cluster_size": cluster_size, "max_clusters": max_clusters, "shift": shift}
    ax = (0, 1)
    Yo = np.asfortranarray(np.fft.ifftshift(Y, axes=ax)) if shift else Y
    if method == "sens_recon":
        So = np.asfortranarray(np.fft.ifftshift(S, axes=ax)) if shift else S
        ref = o.sens_recon(Yo, So)
        (M,), p = run_process(s, method, [Y, S], [((256, 256, nf), np.complex64)], prm)
    else:
        ref = o.rss_recon(Yo)
        (M,), p = run_process(s, method, [Y], [((256, 256, nf), np.float32)], prm)
    if shift:
        ref = np.fft.fftshift(ref, axes=ax)
    assert relmax(M, ref) <= TOL


def test_cluster_recon_relaunch_and_two_pass_agreement(s):
    """Counters self-reset: repeated launches give identical results; with
    whole frames per cluster the result is bit-identical to the two-pass chain
    (same per-coil arithmetic, same coil order)."""
    nx, nc, nf = 256, 3, 12  # enough lines for the coil-serial combine (the coil-parallel one sums in another order)
    rng = np.random.default_rng(5)
    Y = cplx(rng, nx, nx, nc, nf)
    S = cplx(rng, nx, nx, nc)
    hin = s.register_data(h.Data([Y, S], h.DataKind.KData))
    outs = []
    for prm in ({"algorithm": "cluster", "max_clusters": 7},        # frames split across clusters
                {"algorithm": "cluster", "max_clusters": nf},       # one frame per cluster
                {"algorithm": "two_pass"}):
        hout = s.allocate_data([((nx, nx, nf), np.complex64)])
        p = h.Process(s, "sens_recon").set_input(hin).set_output(hout).init(prm)
        p.launch()
        first = s.fetch_data(hout).arrays[0]
        for _ in range(3):
            p.launch()
        again = s.fetch_data(hout).arrays[0]
        assert np.array_equal(first, again)
        outs.append(first)
    assert relmax(outs[0], outs[2]) <= TOL
    assert np.array_equal(outs[1], outs[2])


def test_cluster_recon_rejects_unsupported(s):
    rng = np.random.default_rng(6)
    Y = cplx(rng, 128, 128, 2, 1)
    S = cplx(rng, 128, 128, 2)
    hin = s.register_data(h.Data([Y, S], h.DataKind.KData))
    hout = s.allocate_data([((128, 128, 1), np.complex64)])
    with pytest.raises(h.InvalidParams):
        h.Process(s, "sens_recon").set_input(hin).set_output(hout).init({"algorithm": "cluster"})
    Y2 = cplx(rng, 256, 256, 2, 1)
    hin2 = s.register_data(h.Data([Y2, cplx(rng, 256, 256, 2)], h.DataKind.KData))
    hout2 = s.allocate_data([((256, 256, 1), np.complex64)])
    with pytest.raises(h.InvalidParams):
        h.Process(s, "sens_recon").set_input(hin2).set_output(hout2).init({"algorithm": "cluster", "accumulate": "fp64"})
    with pytest.raises(h.InvalidParams):
        h.Process(s, "sens_recon").set_input(hin2).set_output(hout2).init({"algorithm": "cluster", "cluster_size": 4})
    with pytest.raises(h.InvalidParams):
        h.Process(s, "sens_recon").set_input(hin2).set_output(hout2).init({"algorithm": "fastest"})


@pytest.mark.parametrize("stages", ["2", "4"])
@pytest.mark.parametrize("nx,ny,nc,nf,shift", [(256, 256, 6, 5, False), (256, 4, 3, 2, True), (512, 64, 2, 3, False),
                                               (160, 96, 4, 2, True)])
def test_recon_tma_combine_vs_oracle(s, monkeypatch, stages, nx, ny, nc, nf, shift):
    """Opt-in TMA bulk-copy ring combine (fft_combine_tma.cu), incl. partial
    row groups (ny=4 < the 8 rows a CTA owns at 256) and mixed radix."""
    monkeypatch.setenv("HETRECO_COMBINE_TMA", "1")
    monkeypatch.setenv("HETRECO_TMA_STAGES", stages)
    rng = np.random.default_rng(nx + ny + nc)
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    ax = (0, 1)
    Yr = np.fft.ifftshift(Y, axes=ax) if shift else Y
    Sr = np.fft.ifftshift(S, axes=ax) if shift else S
    X = np.fft.ifft2(Yr.astype(np.complex128), axes=ax)
    ref = (np.conj(Sr.astype(np.complex128))[..., None] * X).sum(axis=2)
    rss = np.sqrt((np.abs(X) ** 2).sum(axis=2))
    if shift:
        ref, rss = np.fft.fftshift(ref, axes=ax), np.fft.fftshift(rss, axes=ax)
    (M,), _ = run_process(s, "sens_recon", [Y, S], [((nx, ny, nf), np.complex64)], {"shift": shift})
    assert relmax(M, ref) <= TOL
    (R,), _ = run_process(s, "rss_recon", [Y], [((nx, ny, nf), np.float32)], {"shift": shift})
    assert relmax(R, rss) <= TOL


@pytest.mark.parametrize("nx,nc,nf,shift", [(256, 8, 1, False), (256, 8, 2, True), (512, 5, 1, False), (160, 6, 1, True),
                                           (64, 3, 4, False)])
def test_coil_parallel_combine_small_problems(s, nx, nc, nf, shift):
    """Few frames -> the coil-parallel combine (fft_combine_cp.cu): one CTA per
    output line, coil groups in parallel, partials summed in group order."""
    rng = np.random.default_rng(nx * nc + nf)
    Y = cplx(rng, nx, nx, nc, nf)
    S = cplx(rng, nx, nx, nc)
    ax = (0, 1)
    Yr = np.fft.ifftshift(Y, axes=ax) if shift else Y
    Sr = np.fft.ifftshift(S, axes=ax) if shift else S
    X = np.fft.ifft2(Yr.astype(np.complex128), axes=ax)
    ref = (np.conj(Sr.astype(np.complex128))[..., None] * X).sum(axis=2)
    rss = np.sqrt((np.abs(X) ** 2).sum(axis=2))
    if shift:
        ref, rss = np.fft.fftshift(ref, axes=ax), np.fft.fftshift(rss, axes=ax)
    (M,), _ = run_process(s, "sens_recon", [Y, S], [((nx, nx, nf), np.complex64)], {"shift": shift})
    assert relmax(M, ref) <= TOL
    (R,), _ = run_process(s, "rss_recon", [Y], [((nx, nx, nf), np.float32)], {"shift": shift})
    assert relmax(R, rss) <= TOL


@pytest.mark.parametrize("nx,ny,nc,nf,shift", [(256, 256, 5, 13, False), (256, 128, 3, 9, True), (512, 512, 2, 9, True),
                                               (160, 160, 3, 17, False), (64, 32, 4, 20, True)])
def test_staged_map_combine(s, monkeypatch, nx, ny, nc, nf, shift):
    """SENSE combine with the map row staged in shared memory (fft_combine_ss.cu,
    forced on for every size): frame groups with a partial tail, shift, mixed
    radix; bit-identical to the register-prefetch combine."""
    rng = np.random.default_rng(nx + nf)
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    monkeypatch.setenv("HETRECO_COMBINE_SS", "1")
    (M,), _ = run_process(s, "sens_recon", [Y, S], [((nx, ny, nf), np.complex64)], {"shift": shift})
    monkeypatch.setenv("HETRECO_COMBINE_SS", "0")
    (M0,), _ = run_process(s, "sens_recon", [Y, S], [((nx, ny, nf), np.complex64)], {"shift": shift})
    assert beq(M, M0)
    ax = (0, 1)
    Yr = np.fft.ifftshift(Y, axes=ax) if shift else Y
    Sr = np.fft.ifftshift(S, axes=ax) if shift else S
    ref = (np.conj(Sr.astype(np.complex128))[..., None] * np.fft.ifft2(Yr.astype(np.complex128), axes=ax)).sum(axis=2)
    if shift:
        ref = np.fft.fftshift(ref, axes=ax)
    assert relmax(M, ref) <= TOL


@pytest.mark.parametrize("n,stages", [(512, "3"), (512, "4"), (512, "5"), (512, "2x16"), (256, "2")])
@pytest.mark.parametrize("shift", [False, True])
def test_strided_ring(s, monkeypatch, n, stages, shift):
    """256/512-point axis-1 pass through the cp.async shared-memory ring
    (k_fft_strided_ring): bit-identical to the register-prefetch pass for
    fft2d both directions and the SENSE chain (partial last wave of tiles)."""
    rng = np.random.default_rng(n + len(stages))
    Y = cplx(rng, n, n, 3, 5)
    S = cplx(rng, n, n, 3)
    k, _, tx = stages.partition("x")  # "2x16" is the default configuration
    monkeypatch.setenv("HETRECO_RING_TX", tx or "8")
    outs = {}
    for ring in ("0", k):
        monkeypatch.setenv("HETRECO_STRIDED_RING", ring)
        (M,), _ = run_process(s, "sens_recon", [Y, S], [((n, n, 5), np.complex64)], {"shift": shift})
        x = Y[:, :, :, 0]
        (fw,), _ = run_process(s, "fft2d", [x], [(x.shape, np.complex64)], {"direction": "forward", "shift": shift})
        (bw,), _ = run_process(s, "fft2d", [x], [(x.shape, np.complex64)], {"direction": "inverse", "shift": shift})
        outs[ring] = (M, fw, bw)
    for a, b in zip(outs["0"], outs[k]):
        assert beq(a, b)


@pytest.mark.parametrize("n,planes", [(256, (3, 5)), (512, (2, 3)), (256, (32, 2))])
@pytest.mark.parametrize("shift", [False, True])
def test_strided_tma_ring(s, monkeypatch, n, planes, shift):
    """The axis-1 column-tile ring fed by TMA boxes (k_fft_strided_tma,
    HETRECO_STRIDED_TMA=1) gives the same bits as the cp.async ring for the
    SENSE chain and fft2d in both directions."""
    nc, nf = planes
    rng = np.random.default_rng(n + nc)
    Y = cplx(rng, n, n, nc, nf)
    S = cplx(rng, n, n, nc)
    outs = {}
    for tma in ("0", "1"):
        monkeypatch.setenv("HETRECO_STRIDED_TMA", tma)
        (M,), _ = run_process(s, "sens_recon", [Y, S], [((n, n, nf), np.complex64)], {"shift": shift})
        x = np.asfortranarray(Y[:, :, :, 0])
        (fw,), _ = run_process(s, "fft2d", [x], [(x.shape, np.complex64)], {"direction": "forward", "shift": shift})
        (bw,), _ = run_process(s, "fft2d", [x], [(x.shape, np.complex64)], {"direction": "inverse", "shift": shift})
        outs[tma] = (M, fw, bw)
    for a, b in zip(outs["0"], outs["1"]):
        assert beq(a, b)


@pytest.mark.parametrize("method", ["sens_recon", "rss_recon"])
def test_recon_overlap_pipeline_bitexact(s, method):
    """"overlap": true -- chunked axis-1/combine graph branches (fork/join over a
    side stream in the captured graph) give the same bits as the serial chain."""
    nx, nc, nf = 256, 3, 21
    rng = np.random.default_rng(21)
    Y = cplx(rng, nx, nx, nc, nf)
    S = cplx(rng, nx, nx, nc)
    ins = [Y, S] if method == "sens_recon" else [Y]
    dt = np.complex64 if method == "sens_recon" else np.float32
    (A,), p = run_process(s, method, ins, [((nx, nx, nf), dt)], {"overlap": True})
    (B,), _ = run_process(s, method, ins, [((nx, nx, nf), dt)], {"overlap": False})
    assert beq(A, B)


def test_launch_timing_modes(s):
    """LaunchStats under "launch_timing": every launch timed, every 16th
    (the default; totals extrapolated), or off; bad values rejected."""
    x = np.asfortranarray(np.random.default_rng(3).random((256, 256), dtype=np.float32))
    hx = s.register_data([x])
    hy = s.allocate_data([((256, 256), np.float32)])
    for mode in ("every", "sampled", "off", None):
        params = {"max_value": 1.0} if mode is None else {"max_value": 1.0, "launch_timing": mode}
        p = h.Process(s, "negate").set_input(hx).set_output(hy).init(params)
        for _ in range(40):
            p.launch()
        st = p.stats()
        assert st.launches == 40 and st.init_calls == 1
        if mode == "off":
            assert st.total_launch_seconds == 0.0
        else:
            assert st.total_launch_seconds > 0 and st.last_launch_seconds > 0
            assert abs(st.mean_launch_seconds() * 40 - st.total_launch_seconds) < 1e-9
        assert beq(s.fetch_data(hy).arrays[0], o.negate(x, 1.0))
    with pytest.raises(h.InvalidParams):
        h.Process(s, "negate").set_input(hx).set_output(hy).init({"launch_timing": "sometimes"})


def test_large_pageable_transfers_through_staging_ring(s):
    """register_data / fetch_data of pageable arrays >= 4 MiB go through the
    pinned staging ring (host_stager.cpp): multi-array packing, sizes that
    are not multiples of the 16 MiB slot, and page-locked buffers (direct)."""
    rng = np.random.default_rng(11)
    a = rng.integers(0, 255, 5 * 2**20 + 13, dtype=np.uint8)
    b = np.asfortranarray(rng.standard_normal((1031, 977, 5)).astype(np.complex64))   # ~38 MiB
    c = rng.standard_normal(2 * 2**20).astype(np.float64)                             # 16 MiB exactly
    # floor(n / parts) a multiple of 64 with a remainder, for every pool size 2..8
    d = rng.integers(0, 255, 840 * 64 * 79 + 1, dtype=np.uint8)
    hdd = s.register_data(h.Data([d], h.DataKind.Generic))
    assert beq(s.fetch_data(hdd).arrays[0], d)
    s.release_data(hdd)
    s.reset_counters()
    hd = s.register_data(h.Data([a, b, c], h.DataKind.Generic))
    assert s.counters() == {"host_to_device": 1, "device_to_host": 0}
    got = s.fetch_data(hd).arrays
    assert beq(got[0], a) and beq(got[1], b) and beq(got[2], c)
    pinned = h.pinned_empty(b.shape, b.dtype)
    pinned[...] = 0
    out = s.fetch_data(hd, [np.empty_like(a), pinned, np.empty_like(c)]).arrays
    assert beq(out[1], b) and beq(out[0], a) and beq(out[2], c)
    hp = s.register_data(h.Data([pinned], h.DataKind.Generic))  # page-locked source: direct DMA
    assert beq(s.fetch_data(hp).arrays[0], b)
    s.release_data(hd)
    s.release_data(hp)


@pytest.mark.parametrize("nx,ny,nc,nf", [(1024, 64, 8, 1), (2048, 32, 3, 1), (4096, 16, 2, 1), (1024, 96, 5, 2)])
def test_coil_parallel_combine_wide_lines(s, monkeypatch, nx, ny, nc, nf):
    """Coil-parallel combine with lines wider than a warp (T = 64/128/256
    threads per coil group at N = 1024/2048/4096): the group exchange needs a
    named barrier (or the CTA barrier), not __syncwarp."""
    rng = np.random.default_rng(nx + ny + nc)
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    X = np.fft.ifft2(Y.astype(np.complex128), axes=(0, 1))
    ref = (np.conj(S.astype(np.complex128))[..., None] * X).sum(axis=2)
    rss = np.sqrt((np.abs(X) ** 2).sum(axis=2))
    for forced in ("1", ""):
        monkeypatch.setenv("HETRECO_COMBINE_CP", forced)
        for _ in range(3):  # a race shows up as run-to-run differences too
            (M,), _ = run_process(s, "sens_recon", [Y, S], [((nx, ny, nf), np.complex64)])
            assert relmax(M, ref) <= TOL
            (R,), _ = run_process(s, "rss_recon", [Y], [((nx, ny, nf), np.float32)])
            assert relmax(R, rss) <= TOL


def test_launch_stats_exclude_interleaved_work(s):
    """LaunchStats chain a launch to the same process' previous stop event only
    when nothing else was queued on the compute stream in between; a cheap
    process interleaved with an expensive one must not absorb its time
    (ADVICE r1, medium)."""
    rng = np.random.default_rng(5)
    x = np.asfortranarray(rng.random((64, 64), dtype=np.float32))
    hx = s.register_data([x])
    hy = s.allocate_data([((64, 64), np.float32)])
    small = h.Process(s, "negate").set_input(hx).set_output(hy).init({"max_value": 1.0, "launch_timing": "every"})
    Y = cplx(rng, 256, 256, 16, 8)
    S = cplx(rng, 256, 256, 16)
    hk = s.register_data(h.Data([Y, S], h.DataKind.KData))
    hm = s.allocate_data([((256, 256, 8), np.complex64)], h.DataKind.XData)
    big = h.Process(s, "sens_recon").set_input(hk).set_output(hm).init({"launch_timing": "every"})
    s.synchronize()
    for _ in range(30):
        small.launch()
        big.launch()
    sm, bg = small.stats(), big.stats()
    assert sm.launches == 30 and bg.launches == 30
    assert sm.mean_launch_seconds() < 0.5 * bg.mean_launch_seconds(), (sm.mean_launch_seconds(), bg.mean_launch_seconds())
    # back-to-back launches of one process still chain (and stay positive)
    for _ in range(20):
        big.launch()
    bg2 = big.stats()
    assert bg2.launches == 50 and bg2.last_launch_seconds > 0
    for hd in (hx, hy, hk, hm):
        s.release_data(hd)


def test_chain_failure_leaves_stages_usable(s):
    """hetreco_chain_create validates everything before taking ownership: a
    repeated handle or a foreign-session stage fails and the caller's stage
    handles keep working."""
    rng = np.random.default_rng(9)
    x = np.asfortranarray(rng.random((32, 32), dtype=np.float32))
    ha = s.register_data([x])
    hb = s.allocate_data([((32, 32), np.float32)])
    p1 = h.Process(s, "negate").set_input(ha).set_output(hb)
    p2 = h.Process(s, "negate").set_input(hb).set_output(hb)
    with pytest.raises(h.HetrecoError):
        h.chain(s, "dup", [p1, p1])
    s2 = h.ComputeSession("gpu")
    try:
        y2 = s2.register_data([x])
        q = h.Process(s2, "negate").set_input(y2).set_output(y2)
        with pytest.raises(h.HetrecoError):
            h.chain(s, "foreign", [p1, q])
        q.init({"max_value": 1.0}).launch()
        assert beq(s2.fetch_data(y2).arrays[0], o.negate(x, 1.0))
        del q
    finally:
        s2.close()
    with pytest.raises(h.HetrecoError):
        h.chain(s, "empty", [])
    p1.init({"max_value": 1.0}).launch()
    assert beq(s.fetch_data(hb).arrays[0], o.negate(x, 1.0))
    c = h.chain(s, "ok", [p1, p2])  # still chainable after the failures
    c.init().launch()
    assert beq(s.fetch_data(hb).arrays[0], o.negate(o.negate(x, 1.0), 1.0))


def test_repoint_same_shapes_patches_graph(s):
    """set_input/set_output after init with the same shapes re-points the
    baked plan (cudaGraphExecUpdate, no rebake) -- results follow the new
    handles; a shape change still re-validates and re-plans."""
    rng = np.random.default_rng(17)
    nx, nc, nf = 128, 4, 3
    Ys = [cplx(rng, nx, nx, nc, nf) for _ in range(2)]
    S = cplx(rng, nx, nx, nc)
    hins = [s.register_data(h.Data([Y, S], h.DataKind.KData)) for Y in Ys]
    houts = [s.allocate_data([((nx, nx, nf), np.complex64)], h.DataKind.XData) for _ in range(2)]
    refs = [o.sens_recon(Y, S) for Y in Ys]
    p = h.Process(s, "sens_recon").set_input(hins[0]).set_output(houts[0]).init()
    for it in range(6):
        i, k = it % 2, (it // 2) % 2
        p.set_input(hins[i]).set_output(houts[k])
        p.launch()
        assert relmax(s.fetch_data(houts[k]).arrays[0], refs[i]) <= TOL
    # negate re-pointed between two images, and fft2d
    xs = [np.asfortranarray(rng.random((64, 64), dtype=np.float32)) for _ in range(2)]
    hx = [s.register_data([x]) for x in xs]
    hy = s.allocate_data([((64, 64), np.float32)])
    q = h.Process(s, "negate").set_input(hx[0]).set_output(hy).init({"max_value": 1.0})
    for i in (1, 0, 1):
        q.set_input(hx[i])
        q.launch()
        assert beq(s.fetch_data(hy).arrays[0], o.negate(xs[i], 1.0))
    # shape change: 5 frames instead of 3 -> full re-plan, still correct
    Y5 = cplx(rng, nx, nx, nc, 5)
    h5 = s.register_data(h.Data([Y5, S], h.DataKind.KData))
    o5 = s.allocate_data([((nx, nx, 5), np.complex64)], h.DataKind.XData)
    p.set_input(h5).set_output(o5)
    p.launch()
    assert relmax(s.fetch_data(o5).arrays[0], o.sens_recon(Y5, S)) <= TOL
    for hd in hins + houts + hx + [hy, h5, o5]:
        s.release_data(hd)


@pytest.mark.parametrize("shift", [False, True])
def test_fused_recon_as_abi_kernels(s, shift):
    """"sens_recon" / "rss_recon" in the layer-1 kernel table (fused_recon.hpp):
    launch_kernel over [Y, S] -> [M] equals the layer-2 process; shape,
    global-size and params errors are reported."""
    rng = np.random.default_rng(23)
    nx, ny, nc, nf = 128, 64, 5, 3
    Y = cplx(rng, nx, ny, nc, nf)
    S = cplx(rng, nx, ny, nc)
    flags = struct.pack("<I", int(shift))
    M = launch_one(s, "sens_recon", [Y, S], np.zeros((nx, ny, nf), np.complex64, order="F"), flags, nx * ny * nf)
    R = launch_one(s, "rss_recon", [Y], np.zeros((nx, ny, nf), np.float32, order="F"), flags, nx * ny * nf)
    (Mp,), _ = run_process(s, "sens_recon", [Y, S], [((nx, ny, nf), np.complex64)], {"shift": shift})
    (Rp,), _ = run_process(s, "rss_recon", [Y], [((nx, ny, nf), np.float32)], {"shift": shift})
    assert beq(M, Mp) and beq(R, Rp)
    if not shift:
        assert relmax(M, o.sens_recon(Y, S)) <= TOL
        assert relmax(R, o.rss_recon(Y)) <= TOL
    out = np.zeros((nx, ny, nf), np.complex64, order="F")
    with pytest.raises(h.InvalidArgument):  # global size is one item per output pixel
        launch_one(s, "sens_recon", [Y, S], out, b"", 7)
    with pytest.raises(h.InvalidArgument):
        launch_one(s, "sens_recon", [Y, S], out, b"\x01\x00", nx * ny * nf)
    with pytest.raises(h.ShapeMismatch):
        launch_one(s, "sens_recon", [Y, S], np.zeros((nx, ny, nf + 1), np.complex64, order="F"), b"", nx * ny * (nf + 1))
    with pytest.raises(h.HetrecoError):  # SENSE needs the maps array
        launch_one(s, "sens_recon", [Y], out, b"", nx * ny * nf)
