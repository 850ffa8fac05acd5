"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Runs the reference library compiled from /root/reference (oracle/_ref, see
oracle/build_ref.sh) through its own ComputeSession API and stores seeded
inputs with the reference's outputs.  Run here (the GPU box has no
/root/reference):

    python tests/golden/make_golden.py

The fixtures pin both the C restatement (tests/test_oracle.py, bit-exact) and
the CUDA path (tests/test_gpu_parity.py).  They are kept small (< 1 MB).
"""
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as o  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def cplx(rng, *shape):
    return np.asfortranarray(
        (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64))


def fft_pass_params(mode, L, S, m, scale, payload: bytes) -> bytes:
    return struct.pack("<IIQQQfI", mode, 0, L, S, m, scale, 0) + payload


def main():
    o.build_reference()
    rng = np.random.default_rng(20180730)
    g = {}

    # negate (kernels/negate.cl.src; SPEC.md:393-395 examples folded in)
    u8 = rng.integers(0, 256, 4096).astype(np.uint8)
    u8[:3] = [0, 100, 255]
    for mv in (255.0, 200.0, 300.5, -3.0):
        g[f"negate_u8_in"] = u8
        g[f"negate_u8_out_{mv}"] = o.ref_run_kernel("negate", u8, struct.pack("<d", mv), u8.size)
    f32 = np.asfortranarray(rng.random((64, 64), dtype=np.float32))
    g["negate_f32_in"] = f32
    g["negate_f32_out"] = o.ref_run_kernel("negate", f32, struct.pack("<d", 1.0), f32.size)

    # one fft_radix2_pass of each mode (kernels/fft_radix2_pass.cl.src:22-69)
    x = cplx(rng, 8, 4, 3)
    rev = np.array([0, 4, 2, 6, 1, 5, 3, 7], np.uint32)
    g["pass_in"] = x
    g["pass_mode0"] = o.ref_run_kernel("fft_radix2_pass", x,
                                       fft_pass_params(0, 8, 1, 0, 1.0, rev.tobytes()), x.size,
                                       out_like=x)
    rev4 = np.array([0, 2, 1, 3], np.uint32)
    g["pass_mode1"] = o.ref_run_kernel("fft_radix2_pass", x,
                                       fft_pass_params(1, 4, 8, 0, 1.0, rev4.tobytes()), x.size,
                                       in_place=True)
    tw = np.array([1, 0, 0.70710677, -0.70710677, 0, -1, -0.70710677, -0.70710677], np.float32)
    g["pass_mode2"] = o.ref_run_kernel("fft_radix2_pass", x,
                                       fft_pass_params(2, 8, 1, 2, 0.5, tw.tobytes()),
                                       x.size // 2, in_place=True)

    # full 2-D FFTs via the restated plan
    for name, shape in (("fft_16x8x3", (16, 8, 3)), ("fft_4x4", (4, 4, 1)),
                        ("fft_32x32x2", (32, 32, 2)), ("fft_2x64", (2, 64, 1)),
                        ("fft_256x1", (256, 1, 1))):
        x = cplx(rng, *shape)
        g[name + "_in"] = x
        g[name + "_inv"] = o.ref_fft2d(x, True)
        g[name + "_fwd"] = o.ref_fft2d(x, False)

    # combine kernels
    x = cplx(rng, 16, 8, 4, 3)
    s = cplx(rng, 16, 8, 4)
    g["cep_x"], g["cep_s"] = x, s
    g["cep_conj"] = o.ref_run_kernel("complex_element_prod", x, struct.pack("<I", 1), x.size,
                                     out_like=x, extra=s)
    g["cep_noconj"] = o.ref_run_kernel("complex_element_prod", x, struct.pack("<I", 0), x.size,
                                       out_like=x, extra=s)
    outm = np.zeros((16, 8, 3), np.complex64, order="F")
    g["xsum_out"] = o.ref_run_kernel("ximage_sum", x, b"", 16 * 8 * 3, out_like=outm)
    outr = np.zeros((16, 8, 3), np.float32, order="F")
    g["rss_out"] = o.ref_run_kernel("rss_combine", x, b"", 16 * 8 * 3, out_like=outr)

    # full chains
    Y = cplx(rng, 32, 16, 4, 3)
    S = cplx(rng, 32, 16, 4)
    g["sens_Y"], g["sens_S"] = Y, S
    g["sens_M"] = o.ref_recon("sens", Y, S)[0]
    g["rss_Y"] = Y
    g["rss_R"] = o.ref_recon("rss", Y)[0]

    # layout headers (src/layout.cpp:57-102)
    cases = [[(4, [160, 160])], [(3, [3]), (3, [2])], [(4, [32, 16, 4, 3]), (4, [32, 16, 4])],
             [(1, [7]), (6, [3, 5]), (2, [1, 1, 9]), (5, [2, 2, 2, 2, 2, 2, 2, 2])]]
    for i, case in enumerate(cases):
        w, total = o.ref_layout_header(case)
        g[f"layout{i}_words"] = w
        g[f"layout{i}_total"] = np.array([total], np.uint64)

    path = os.path.join(OUT, "reference_vectors.npz")
    np.savez_compressed(path, **g)
    print("wrote", path, os.path.getsize(path), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
