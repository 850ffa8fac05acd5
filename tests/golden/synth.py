"""Seeded synthetic k-space / sensitivity maps that do not depend on the numpy
version: splitmix64 of (seed, element index) mapped to uniform [-1, 1).  Used
by the large-shape golden fixtures (tests/golden/large_shapes.json), so the
inputs can be regenerated bit for bit on any box from the seed alone."""
import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x * _G + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, n: int) -> np.ndarray:
    """n float32 values in [-1, 1), exactly representable (24-bit grid)."""
    idx = np.arange(n, dtype=np.uint64) + np.uint64(seed) * np.uint64(0x100000000)
    bits = _splitmix64(idx) >> np.uint64(40)  # 24 random bits
    return (bits.astype(np.float64) / float(1 << 23) - 1.0).astype(np.float32)


def cplx(seed: int, *shape) -> np.ndarray:
    n = int(np.prod(shape))
    re, im = uniform(2 * seed, n), uniform(2 * seed + 1, n)
    return np.asfortranarray((re + 1j * im).astype(np.complex64).reshape(shape, order="F"))
