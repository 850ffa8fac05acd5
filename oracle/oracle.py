"""ctypes front-end for the oracles.  TEST INFRASTRUCTURE ONLY.

Two checkers live here, both CPU:

* ``port``      -- oracle/hetreco_oracle.c, the plain-C restatement of the
                   reference kernels and FFT plan (liboracle.so, built by
                   ``build()``; rebuilt on demand from the committed C source,
                   so it also works on the GPU box).
* ``reference`` -- oracle/_ref/libhetreco_refdrv.so, the reference library
                   itself compiled from /root/reference by build_ref.sh and
                   driven through its own ComputeSession API (ref_driver.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  Arrays follow the
reference's column-major convention: a numpy array in Fortran order whose
``shape`` equals the reference ``dims`` (ndarray.hpp:61-67).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhetreco_refdrv.so")
# the reference library on the B200 via integration/reference_cuda_backend.cpp
REF_ON_B200_SO = os.path.join(HERE, "_ref", "libhetreco_ref_on_b200.so")

# ElementType codes: include/hetreco/ndarray.hpp:17-24 (wire format)
UINT8, INT32, FLOAT32, COMPLEX64, FLOAT64, COMPLEX128 = 1, 2, 3, 4, 5, 6
NP_OF_CODE = {UINT8: np.uint8, INT32: np.int32, FLOAT32: np.float32,
              COMPLEX64: np.complex64, FLOAT64: np.float64, COMPLEX128: np.complex128}
CODE_OF_NP = {np.dtype(v): k for k, v in NP_OF_CODE.items()}

_lock = threading.Lock()
_port = None
_ref = None

_vp, _u64, _f32, _f64, _i32 = C.c_void_p, C.c_uint64, C.c_float, C.c_double, C.c_int


def build_port(force: bool = False) -> str:
    """Compile the C restatement (gcc is in the image, here and on the box)."""
    src = os.path.join(HERE, "hetreco_oracle.c")
    if force or not os.path.exists(PORT_SO) or os.path.getmtime(PORT_SO) < os.path.getmtime(src):
        tmp = PORT_SO + ".%d.tmp" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", tmp, src, "-lm"])
        os.replace(tmp, PORT_SO)
    return PORT_SO


def build_reference() -> bool:
    """Build oracle/_ref from /root/reference when present.  False if absent."""
    if not os.path.isdir(os.environ.get("HETRECO_REFERENCE", "/root/reference")):
        return os.path.exists(REF_SO)
    subprocess.check_call([os.path.join(HERE, "build_ref.sh")])
    return True


def port():
    global _port
    with _lock:
        if _port is None:
            lib = C.CDLL(build_port())
            lib.oracle_negate_u8.argtypes = [_vp, _vp, _u64, _f64]
            lib.oracle_negate_f32.argtypes = [_vp, _vp, _u64, _f64]
            lib.oracle_fft_radix2_pass.argtypes = [_vp, _vp, _u64, C.c_uint32, _u64, _u64, _u64,
                                                   _f32, _vp]
            lib.oracle_fft2d.argtypes = [_vp, _vp, _u64, _u64, _u64, _i32]
            lib.oracle_complex_element_prod.argtypes = [_vp, _u64, _vp, _u64, _vp, _i32]
            lib.oracle_ximage_sum.argtypes = [_vp, _vp, _u64, _u64, _u64]
            lib.oracle_rss_combine.argtypes = [_vp, _vp, _u64, _u64, _u64]
            lib.oracle_matrix_add_f32.argtypes = [_vp, _vp, _vp, _u64]
            lib.oracle_sens_recon.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _u64, _vp]
            lib.oracle_rss_recon.argtypes = [_vp, _vp, _u64, _u64, _u64, _u64, _vp]
            lib.oracle_sense_forward.argtypes = [_vp, _vp, _vp, _vp, _u64, _u64, _u64, _u64, _vp]
            _port = lib
        return _port


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def reference():
    global _ref
    with _lock:
        if _ref is None:
            if not os.path.exists(REF_SO):
                raise RuntimeError("oracle/_ref not built (needs /root/reference at build time)")
            lib = C.CDLL(REF_SO)
            lib.refdrv_last_error.restype = C.c_char_p
            lib.refdrv_run_kernel.argtypes = [C.c_char_p, _i32, _i32, _vp, _vp, _i32, _i32, _vp,
                                              _vp, _i32, _i32, _vp, _vp, _i32, _vp, _u64, _u64]
            lib.refdrv_fft2d.argtypes = [_vp, _vp, _u64, _u64, _u64, _i32]
            lib.refdrv_recon.argtypes = [_i32, _vp, _vp, _vp, _u64, _u64, _u64, _u64, _i32,
                                         C.POINTER(_f64), C.POINTER(_f64)]
            lib.refdrv_recon_e2e.argtypes = [_i32, _vp, _vp, _vp, _u64, _u64, _u64, _u64, _i32,
                                             C.POINTER(_f64)]
            lib.refdrv_layout_header.argtypes = [_i32, _vp, _vp, _vp, _u64, _vp, C.POINTER(_u64)]
            if hasattr(lib, "refdrv_builtin_source_count"):
                lib.refdrv_builtin_source_name.restype = C.c_char_p
                lib.refdrv_builtin_source_name.argtypes = [_i32]
                lib.refdrv_builtin_source_text.restype = C.c_char_p
                lib.refdrv_builtin_source_text.argtypes = [_i32]
            _ref = lib
        return _ref


class _RefOnB200:
    """The unmodified reference session code on the CUDA adapter: the same
    refdrv_* entry points, named refcuda_*."""

    def __init__(self):
        L = C.CDLL(REF_ON_B200_SO)
        L.refcuda_last_error.restype = C.c_char_p
        L.refcuda_run_kernel.argtypes = [C.c_char_p, _i32, _i32, _vp, _vp, _i32, _i32, _vp, _vp, _i32, _i32,
                                         _vp, _vp, _i32, _vp, _u64, _u64]
        L.refcuda_fft2d.argtypes = [_vp, _vp, _u64, _u64, _u64, _i32]
        L.refcuda_recon.argtypes = [_i32, _vp, _vp, _vp, _u64, _u64, _u64, _u64, _i32, C.POINTER(_f64),
                                    C.POINTER(_f64)]
        L.refcuda_set_source_mode.argtypes = [_i32]
        self.L = L

    def __getattr__(self, name):  # refdrv_x -> refcuda_x
        return getattr(self.L, name.replace("refdrv_", "refcuda_"))


_ref_b200 = None


def ref_on_b200_available() -> bool:
    return os.path.exists(REF_ON_B200_SO)


def use_reference_on_b200(source_kernels: bool = False):
    """Context in which the ref_* helpers below run the reference's session
    code on the B200 (integration adapter) instead of its CPU backend.
    source_kernels=True: the adapter reports source support, so the
    reference's load_builtin_kernels compiles its embedded kernel sources with
    NVRTC for sm_100a (session.cpp:139-148) instead of using the precompiled
    builtins."""
    import contextlib

    @contextlib.contextmanager
    def ctx():
        global _ref, _ref_b200
        saved = reference()
        if _ref_b200 is None:
            _ref_b200 = _RefOnB200()
        _ref = _ref_b200
        got = _ref_b200.L.refcuda_set_source_mode(1 if source_kernels else 0)
        if source_kernels and not got:
            raise RuntimeError("B200 adapter has no source-kernel support (NVRTC missing)")
        try:
            yield
        finally:
            _ref_b200.L.refcuda_set_source_mode(0)
            _ref = saved
    return ctx()


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _f(a, dtype) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=dtype))


def _check_ref(rc):
    if rc != 0:
        raise RuntimeError("reference: " + reference().refdrv_last_error().decode())


# ---------------------------------------------------------------------------
# port (C restatement)
# ---------------------------------------------------------------------------

def negate(x: np.ndarray, max_value: float) -> np.ndarray:
    x = np.asfortranarray(x)
    out = np.empty_like(x, order="F")
    if x.dtype == np.uint8:
        port().oracle_negate_u8(_p(x), _p(out), x.size, float(max_value))
    elif x.dtype == np.float32:
        port().oracle_negate_f32(_p(x), _p(out), x.size, float(max_value))
    else:
        raise TypeError(x.dtype)
    return out


def fft_radix2_pass(data_in, data_out, mode, L, S, m, scale, payload: np.ndarray) -> np.ndarray:
    """One reference pass; returns the updated copy of data_out."""
    out = _f(data_out, np.complex64).copy(order="F")
    din = _f(data_in, np.complex64) if data_in is not None else out
    pl = np.ascontiguousarray(payload)
    port().oracle_fft_radix2_pass(_p(din), _p(out), out.size, mode, L, S, m, float(scale), _p(pl))
    return out


def fft2d(x: np.ndarray, inverse: bool) -> np.ndarray:
    x = _f(x, np.complex64)
    nx, ny = x.shape[0], (x.shape[1] if x.ndim > 1 else 1)
    batch = x.size // (nx * ny)
    out = np.empty_like(x, order="F")
    if port().oracle_fft2d(_p(x), _p(out), nx, ny, batch, int(bool(inverse))) != 0:
        raise ValueError("fft2d: dims must be powers of two")
    return out


def complex_element_prod(x, s, conjugate: bool) -> np.ndarray:
    x = _f(x, np.complex64)
    s = _f(s, np.complex64)
    out = np.empty_like(x, order="F")
    port().oracle_complex_element_prod(_p(x), x.size, _p(s), s.size, _p(out), int(conjugate))
    return out


def ximage_sum(x) -> np.ndarray:
    x = _f(x, np.complex64)
    nx, ny, nc = x.shape[:3]
    nf = x.size // (nx * ny * nc)
    out = np.empty((nx, ny) + x.shape[3:], np.complex64, order="F")
    port().oracle_ximage_sum(_p(x), _p(out), nx * ny, nc, nf)
    return out


def rss_combine(x) -> np.ndarray:
    x = _f(x, np.complex64)
    nx, ny, nc = x.shape[:3]
    nf = x.size // (nx * ny * nc)
    out = np.empty((nx, ny) + x.shape[3:], np.float32, order="F")
    port().oracle_rss_combine(_p(x), _p(out), nx * ny, nc, nf)
    return out


def matrix_add(a, b) -> np.ndarray:
    a = _f(a, np.float32)
    b = _f(b, np.float32)
    out = np.empty_like(a, order="F")
    port().oracle_matrix_add_f32(_p(a), _p(b), _p(out), a.size)
    return out


def sens_recon(Y, S) -> np.ndarray:
    Y = _f(Y, np.complex64)
    S = _f(S, np.complex64)
    nx, ny, nc, nf = (Y.shape + (1,))[:4]
    M = np.empty((nx, ny, nf), np.complex64, order="F")
    scratch = np.empty(2 * Y.size, np.complex64)
    if port().oracle_sens_recon(_p(Y), _p(S), _p(M), nx, ny, nc, nf, _p(scratch)) != 0:
        raise ValueError("sens_recon: dims must be powers of two")
    return M


def rss_recon(Y) -> np.ndarray:
    Y = _f(Y, np.complex64)
    nx, ny, nc, nf = (Y.shape + (1,))[:4]
    R = np.empty((nx, ny, nf), np.float32, order="F")
    scratch = np.empty(Y.size, np.complex64)
    if port().oracle_rss_recon(_p(Y), _p(R), nx, ny, nc, nf, _p(scratch)) != 0:
        raise ValueError("rss_recon: dims must be powers of two")
    return R


def sense_forward(M, S, mask=None) -> np.ndarray:
    """Y[:,:,c,f] = mask . FFT2_forward(S_c . M_f) (no reference kernel; composed
    from complex_element_prod + the restated FFT plan)."""
    M = _f(M, np.complex64)
    S = _f(S, np.complex64)
    nx, ny = M.shape[:2]
    nf = M.size // (nx * ny)
    nc = S.size // (nx * ny)
    Y = np.empty((nx, ny, nc, nf), np.complex64, order="F")
    mk = _f(mask, np.float32) if mask is not None else None
    scratch = np.empty(nx * ny, np.complex64)
    if port().oracle_sense_forward(_p(M), _p(S), _p(mk) if mk is not None else None, _p(Y), nx, ny, nc, nf,
                                   _p(scratch)) != 0:
        raise ValueError("sense_forward: dims must be powers of two")
    return Y


def sense_normal(M, S, mask=None) -> np.ndarray:
    """E^H E M = sens_recon(sense_forward(M, S, mask), S)."""
    return sens_recon(sense_forward(M, S, mask), S)


def phantom_blobs(nx: int, ny: int, seed: int):
    """Blob parameters (amp, radius, angle, sigma) x 3 drawn from mt19937_64(seed)
    with 53-bit uniforms -- restates hetreco::phantom_blobs (phantom.cpp), the
    rule SPEC.md:452 leaves open ("centers/widths drawn from seeded generator")."""
    mt = _MT19937_64(seed)
    L = float(min(nx, ny))
    out = []
    for _ in range(3):
        u = [float(mt.next() >> 11) * (1.0 / 9007199254740992.0) for _ in range(4)]
        out.append((0.5 + 0.5 * u[0], 0.25 * L * u[1], 6.283185307179586 * u[2], L * (0.04 + 0.08 * u[3])))
    return out


class _MT19937_64:
    """The standard 64-bit Mersenne Twister (std::mt19937_64), scalar Python."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def next(self) -> int:
        M = 0xFFFFFFFFFFFFFFFF
        if self.i >= 312:
            for k in range(312):
                x = (self.mt[k] & 0xFFFFFFFF80000000) | (self.mt[(k + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[k] = self.mt[(k + 156) % 312] ^ xa
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & M


def gen_phantom(nx: int, ny: int, frames: int, coils: int, seed: int):
    """CPU port of gen_phantom (phantom.cu formulas) in fp64,
    rounded once to complex64; Y = sense_forward(M_true, S) (the restated
    forward FFT).  Returns (Y, S, M_true)."""
    blobs = phantom_blobs(nx, ny, seed)
    u = (np.arange(nx, dtype=np.float64) - 0.5 * nx)[:, None]
    v = (np.arange(ny, dtype=np.float64) - 0.5 * ny)[None, :]
    M = np.zeros((nx, ny, frames), np.complex64, order="F")
    for f in range(frames):
        th = 6.283185307179586476925286766559 * f / frames
        m = np.zeros((nx, ny))
        for amp, rad, ang, sig in blobs:
            cu, cv = rad * np.cos(ang + th), rad * np.sin(ang + th)
            m += amp * np.exp(-((u - cu) ** 2 + (v - cv) ** 2) / (2.0 * sig * sig))
        M[:, :, f] = m.astype(np.float32)
    L = float(min(nx, ny))
    R, W = 0.5 * L, 0.4 * L
    G = np.empty((nx, ny, coils))
    be = 6.283185307179586476925286766559 * np.arange(coils) / coils
    for c in range(coils):
        G[:, :, c] = np.exp(-((u - R * np.cos(be[c])) ** 2 + (v - R * np.sin(be[c])) ** 2) / (2.0 * W * W))
    G /= np.sqrt((G * G).sum(axis=2, keepdims=True))
    S = np.asfortranarray((G * np.exp(1j * be)[None, None, :]).astype(np.complex64))
    return sense_forward(M, S), S, M


# ---------------------------------------------------------------------------
# reference (the real library, oracle/_ref)
# ---------------------------------------------------------------------------

def _dims(a: np.ndarray):
    d = np.array(a.shape if a.ndim else (1,), dtype=np.uint64)
    return d, len(d)


def ref_run_kernel(name: str, x: np.ndarray, params: bytes, gsize: int, out_like=None,
                   extra: np.ndarray | None = None, in_place: bool = False) -> np.ndarray:
    """Run one builtin kernel through ComputeSession::launch_kernel."""
    x = np.asfortranarray(x)
    xd, xr = _dims(x)
    if extra is not None:
        extra = np.asfortranarray(extra)
        ed, er = _dims(extra)
        et = CODE_OF_NP[extra.dtype]
    else:
        ed, er, et = np.zeros(1, np.uint64), 0, 0
    if in_place:
        out = x.copy(order="F")
    else:
        out = np.zeros_like(out_like, order="F") if out_like is not None else np.zeros_like(x)
    od, orank = _dims(out)
    pb = np.frombuffer(bytes(params) or b"\0", np.uint8).copy()
    _check_ref(reference().refdrv_run_kernel(
        name.encode(), CODE_OF_NP[x.dtype], xr, _p(xd), _p(x), et, er, _p(ed),
        _p(extra) if extra is not None else None, CODE_OF_NP[out.dtype], orank, _p(od), _p(out),
        int(in_place), _p(pb), len(params), gsize))
    return out


def ref_fft2d(x: np.ndarray, inverse: bool) -> np.ndarray:
    x = _f(x, np.complex64)
    nx, ny = x.shape[0], x.shape[1]
    out = np.empty_like(x, order="F")
    _check_ref(reference().refdrv_fft2d(_p(x), _p(out), nx, ny, x.size // (nx * ny),
                                        int(bool(inverse))))
    return out


def ref_recon(method: str, Y: np.ndarray, S: np.ndarray | None = None, reps: int = 1):
    """Returns (result, mean_seconds_per_launch, init_seconds)."""
    Y = _f(Y, np.complex64)
    nx, ny, nc, nf = (Y.shape + (1,))[:4]
    if method == "sens":
        S = _f(S, np.complex64)
        out = np.empty((nx, ny, nf), np.complex64, order="F")
    else:
        out = np.empty((nx, ny, nf), np.float32, order="F")
    mean_s, init_s = C.c_double(), C.c_double()
    _check_ref(reference().refdrv_recon(0 if method == "sens" else 1, _p(Y),
                                        _p(S) if S is not None else None, _p(out), nx, ny, nc,
                                        nf, reps, C.byref(mean_s), C.byref(init_s)))
    return out, mean_s.value, init_s.value


def ref_recon_e2e(method: str, Y: np.ndarray, S: np.ndarray | None = None, reps: int = 1):
    """Per-step register(Y) + chain + fetch through the reference API.
    Returns (result, mean_seconds_per_step)."""
    Y = _f(Y, np.complex64)
    nx, ny, nc, nf = (Y.shape + (1,))[:4]
    if method == "sens":
        S = _f(S, np.complex64)
        out = np.empty((nx, ny, nf), np.complex64, order="F")
    else:
        out = np.empty((nx, ny, nf), np.float32, order="F")
    mean_s = C.c_double()
    _check_ref(reference().refdrv_recon_e2e(0 if method == "sens" else 1, _p(Y),
                                            _p(S) if S is not None else None, _p(out), nx, ny, nc, nf,
                                            reps, C.byref(mean_s)))
    return out, mean_s.value


def ref_builtin_sources():
    """The reference library's embedded builtin kernel units [(unit_name, text)]
    (kernels.hpp:52-57) -- inputs for source-kernel equivalence tests."""
    L = reference()
    return [(L.refdrv_builtin_source_name(i).decode(), L.refdrv_builtin_source_text(i).decode())
            for i in range(L.refdrv_builtin_source_count())]


def ref_pool_threads() -> int:
    return int(reference().refdrv_pool_threads())


def ref_layout_header(arrays, alignment: int = 256):
    """arrays: list of (type_code, dims).  Returns (u64 words, total_bytes)."""
    n = len(arrays)
    types = np.array([t for t, _ in arrays], np.int32)
    ranks = np.array([len(d) for _, d in arrays], np.int32)
    dims8 = np.ones((n, 8), np.uint64)
    for i, (_, d) in enumerate(arrays):
        dims8[i, :len(d)] = d
    words = np.zeros(1 + 11 * n, np.uint64)
    total = C.c_uint64()
    _check_ref(reference().refdrv_layout_header(n, _p(types), _p(ranks), _p(dims8), alignment,
                                                _p(words), C.byref(total)))
    return words, total.value
