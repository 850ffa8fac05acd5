"""Source kernels compiled at run time by NVRTC for sm_100a (SURVEY.md §8
f.4; the role of the reference's cpujit backend, cpujit_backend.cpp:121-177):
units in the reference's HETRECO_KERNEL dialect -> load_kernels -> the same
launch_kernel path as the precompiled builtins.

Parity anchor: the reference's OWN embedded builtin sources (read from the
reference library, oracle/_ref) compiled through this path reproduce the
golden vectors bit for bit -- acceptance criteria 8 (CompileError with the
unit's log) and 11 (backend equivalence) of SPEC.md:575-578.
"""
import os
import struct

import numpy as np
import pytest

from oracle import oracle as o
from paper_1807_11830_b200 import hetreco as h

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

AXPY = r"""
/* axpy: out = a * x + y (FLOAT32, uncontracted), a = f32 param at byte 0 */
HETRECO_KERNEL(axpy) {
    (void)gsize;
    float a = hetreco_param_f32(args, 0);
    const float* x = (const float*)hetreco_array_in(args, 0);
    const float* y = (const float*)hetreco_array_in(args, 1);
    float* out = (float*)hetreco_array_out(args, 0);
    out[gid] = a * x[gid] + y[gid];
}
// HETRECO_KERNEL(commented_out) must not be registered
"""
TWO = r"""
static float sq(float v) { return v * v; }   /* helpers are device code too */
HETRECO_KERNEL(square) {
    (void)gsize;
    const float* x = (const float*)hetreco_array_in(args, 0);
    ((float*)hetreco_array_out(args, 0))[gid] = sq(x[gid]);
}
HETRECO_KERNEL(cmul_conj) {
    (void)gsize;
    const hetreco_cfloat* x = (const hetreco_cfloat*)hetreco_array_in(args, 0);
    const hetreco_cfloat* s = (const hetreco_cfloat*)hetreco_array_in(args, 1);
    hetreco_cfloat* out = (hetreco_cfloat*)hetreco_array_out(args, 0);
    uint64_t ns = hetreco_layout_elements(args->in_layout, 1);
    out[gid] = hetreco_cmul(x[gid], hetreco_conjf(s[gid % ns]));
}
"""
BROKEN = "HETRECO_KERNEL(broken) {\n    int x = ;\n}\n"

needs_nvrtc = pytest.mark.skipif(not h.nvrtc_available(), reason="libnvrtc not available")


# ---- CPU: compile only ------------------------------------------------------------------

@needs_nvrtc
def test_compile_check_names_and_log():
    names, _ = h.compile_check("axpy.cl.src", AXPY)
    assert names == ["axpy"]
    names, _ = h.compile_check("two.cl.src", TWO)
    assert names == ["square", "cmul_conj"]
    with pytest.raises(h.CompileError) as e:
        h.compile_check("broken.cl.src", BROKEN)
    msg = str(e.value)
    assert "broken.cl.src" in msg and "error" in msg and "(2)" in msg  # unit name + line of the error


@needs_nvrtc
@pytest.mark.skipif(not o.reference_available(), reason="oracle/_ref not built")
def test_reference_builtin_sources_compile_for_sm100a():
    units = o.ref_builtin_sources()
    assert len(units) == 6
    for name, text in units:
        names, _ = h.compile_check(name, text)
        assert names == [name.split(".")[0]]


# ---- GPU ---------------------------------------------------------------------------------

@pytest.fixture(scope="module")
def s():
    sess = h.ComputeSession("gpu")
    yield sess
    sess.close()


def launch_one(s, name, inputs, out_like, params, gsize, in_place=False):
    hin = s.register_data(inputs)
    hout = hin if in_place else s.register_data([np.zeros_like(out_like)])
    s.launch_kernel(name, hin, hout, params, gsize)
    out = s.fetch_data(hout).arrays[0]
    s.release_data(hin)
    if not in_place:
        s.release_data(hout)
    return out


def beq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes(order="F") == b.tobytes(order="F")


@pytest.mark.gpu
def test_source_kernels_run_bitexact(s):
    assert s.device().supports_source_kernels
    s.load_kernels([("axpy.cl.src", AXPY), ("two.cl.src", TWO)])
    assert {"axpy", "square", "cmul_conj"} <= set(s.kernel_names())
    assert "commented_out" not in s.kernel_names()
    rng = np.random.default_rng(3)
    x = rng.standard_normal(100003).astype(np.float32)
    y = rng.standard_normal(100003).astype(np.float32)
    got = launch_one(s, "axpy", [x, y], x, struct.pack("<f", 1.7), x.size)
    assert beq(got, (np.float32(1.7) * x) + y)  # two roundings, no FMA
    assert beq(launch_one(s, "square", [x], x, b"", x.size), x * x)
    xc = (rng.standard_normal(4096) + 1j * rng.standard_normal(4096)).astype(np.complex64)
    sc = (rng.standard_normal(1024) + 1j * rng.standard_normal(1024)).astype(np.complex64)
    got = launch_one(s, "cmul_conj", [xc, sc], xc, b"", xc.size)
    ref = o.complex_element_prod(xc, sc, True)
    assert beq(got, ref)


@pytest.mark.gpu
def test_source_kernel_errors_leave_registry_unchanged(s):
    before = s.kernel_names()
    with pytest.raises(h.CompileError) as e:  # a broken unit among good ones: nothing registered
        s.load_kernels([("ok.cl.src", AXPY.replace("(axpy)", "(axpy2)")), ("broken.cl.src", BROKEN)])
    assert "broken.cl.src" in str(e.value)
    assert s.kernel_names() == before
    s.load_kernels([("dup1.cl.src", AXPY.replace("(axpy)", "(dup_k)"))])
    with pytest.raises(h.DuplicateKernel):
        s.load_kernels([("x.cl.src", AXPY.replace("(axpy)", "(fresh_k)")), ("dup2.cl.src", AXPY.replace("(axpy)", "(dup_k)"))])
    assert "fresh_k" not in s.kernel_names()


@pytest.mark.gpu
@pytest.mark.skipif(not o.reference_available(), reason="oracle/_ref not built")
def test_reference_sources_on_b200_match_golden(golden):
    """The reference's own builtin kernel sources, compiled by NVRTC for
    sm_100a, reproduce the golden vectors bit for bit (the precompiled
    builtins' contract), i.e. backend equivalence at 0 ulp."""
    sess = h.ComputeSession("gpu")  # no precompiled builtins in this session
    sess.load_kernels(o.ref_builtin_sources())
    x = golden["negate_u8_in"]
    for mv in (255.0, 200.0, 300.5, -3.0):
        assert beq(launch_one(sess, "negate", [x], x, struct.pack("<d", mv), x.size), golden[f"negate_u8_out_{mv}"])
    f = golden["negate_f32_in"]
    assert beq(launch_one(sess, "negate", [f], f, struct.pack("<d", 1.0), f.size), golden["negate_f32_out"])
    x = golden["pass_in"]
    rev = np.array([0, 4, 2, 6, 1, 5, 3, 7], np.uint32)
    p0 = struct.pack("<IIQQQfI", 0, 0, 8, 1, 0, 1.0, 0) + rev.tobytes()
    assert beq(launch_one(sess, "fft_radix2_pass", [x], x, p0, x.size), golden["pass_mode0"])
    rev4 = np.array([0, 2, 1, 3], np.uint32)
    p1 = struct.pack("<IIQQQfI", 1, 0, 4, 8, 0, 1.0, 0) + rev4.tobytes()
    assert beq(launch_one(sess, "fft_radix2_pass", [x], x, p1, x.size, in_place=True), golden["pass_mode1"])
    tw = np.array([1, 0, 0.70710677, -0.70710677, 0, -1, -0.70710677, -0.70710677], np.float32)
    p2 = struct.pack("<IIQQQfI", 2, 0, 8, 1, 2, 0.5, 0) + tw.tobytes()
    assert beq(launch_one(sess, "fft_radix2_pass", [x], x, p2, x.size // 2, in_place=True), golden["pass_mode2"])
    x, sm = golden["cep_x"], golden["cep_s"]
    assert beq(launch_one(sess, "complex_element_prod", [x, sm], x, struct.pack("<I", 1), x.size), golden["cep_conj"])
    assert beq(launch_one(sess, "ximage_sum", [x], golden["xsum_out"], b"", 16 * 8 * 3), golden["xsum_out"])
    assert beq(launch_one(sess, "rss_combine", [x], golden["rss_out"], b"", 16 * 8 * 3), golden["rss_out"])
    a = np.arange(1000, dtype=np.float32)
    assert beq(launch_one(sess, "matrix_add", [a, a[::-1].copy()], a, b"", a.size), o.matrix_add(a, a[::-1].copy()))
    sess.close()
