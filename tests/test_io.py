"""File formats either side of the reconstruction path (the
reference's io module): MAT-file Level 5, PGM/PPM, raw +
sidecar.  Host-only (no GPU): the readers and writers are C++ in
libhetreco_b200.so, called through the C-ABI.

Parity anchors: the SPEC examples, the acceptance criterion
"writers/readers are inverses on 200 random arrays; compressed element ->
UnsupportedFeature('compression')", and interoperability with
an independent MAT implementation (scipy.io) in both directions.
"""
import os
import struct

import numpy as np
import pytest

from paper_1807_11830_b200 import hetreco as h

sio = pytest.importorskip("scipy.io")

DTYPES = [np.uint8, np.int32, np.float32, np.float64, np.complex64, np.complex128]


def rand_array(rng, dtype, shape):
    if np.issubdtype(dtype, np.integer):
        info = np.iinfo(dtype)
        return rng.integers(info.min, info.max, shape, dtype=dtype, endpoint=True)
    a = rng.standard_normal(shape)
    if np.issubdtype(dtype, np.complexfloating):
        a = a + 1j * rng.standard_normal(shape)
    return a.astype(dtype)


def test_mat_roundtrip_200_random_arrays(tmp_path):
    rng = np.random.default_rng(2024)
    for i in range(200):
        dtype = DTYPES[i % len(DTYPES)]
        rank = int(rng.integers(2, 9))
        shape = tuple(int(x) for x in rng.integers(1, 5, rank))
        a = np.asfortranarray(rand_array(rng, dtype, shape))
        p = tmp_path / f"v{i}.mat"
        h.write_mat(str(p), {f"var_{i}": a})
        back = h.read_mat(str(p))
        assert list(back) == [f"var_{i}"]
        b = back[f"var_{i}"]
        assert b.dtype == a.dtype and b.shape == a.shape
        assert a.tobytes(order="F") == b.tobytes(order="F")  # bit-identical payload


def test_mat_spec_examples(tmp_path):
    # 2x3 FLOAT32 round trip -> bit-identical payload and dims
    a = np.asfortranarray(np.array([[1.5, -2, 3], [4, 5e-30, np.inf]], np.float32))
    h.write_mat(str(tmp_path / "a.mat"), {"a": a})
    b = h.read_mat(str(tmp_path / "a.mat"))["a"]
    assert b.shape == (2, 3) and b.tobytes() == a.tobytes()
    # complex single keeps re/im separately
    z = np.asfortranarray(np.array([[1 + 2j, -3 - 0j], [np.nan + 1j, 0 - 7j]], np.complex64))
    h.write_mat(str(tmp_path / "z.mat"), [("z", z)])
    zb = h.read_mat(str(tmp_path / "z.mat"))["z"]
    assert zb.tobytes(order="F") == z.tobytes(order="F")
    # empty variable list -> valid header-only file
    h.write_mat(str(tmp_path / "e.mat"), {})
    raw = (tmp_path / "e.mat").read_bytes()
    assert len(raw) == 128 and raw.startswith(b"MATLAB 5.0 MAT-file, created by hetreco")
    assert raw[124:128] == b"\x00\x01IM"
    assert h.read_mat(str(tmp_path / "e.mat")) == {}
    # names: nonempty, <= 63 bytes
    h.write_mat(str(tmp_path / "n.mat"), {"x" * 63: a})
    with pytest.raises(h.InvalidParams):
        h.write_mat(str(tmp_path / "n.mat"), {"x" * 64: a})
    with pytest.raises(h.InvalidParams):
        h.write_mat(str(tmp_path / "n.mat"), {"": a})


def test_mat_multiple_variables_keep_order(tmp_path):
    rng = np.random.default_rng(3)
    vs = [("kdata", rand_array(rng, np.complex64, (8, 8, 4, 2))), ("smaps", rand_array(rng, np.complex64, (8, 8, 4))),
          ("mask", rand_array(rng, np.float32, (8, 8))), ("n", np.int32([[7]]))]
    h.write_mat(str(tmp_path / "m.mat"), vs)
    back = h.read_mat(str(tmp_path / "m.mat"))
    assert list(back) == [n for n, _ in vs]
    for n, a in vs:
        assert np.array_equal(back[n], a)


def test_mat_interop_with_scipy(tmp_path):
    rng = np.random.default_rng(4)
    Y = rand_array(rng, np.complex64, (16, 8, 3, 2))
    S = rand_array(rng, np.complex128, (16, 8, 3))
    R = rand_array(rng, np.float32, (5, 7))
    # ours -> scipy
    h.write_mat(str(tmp_path / "ours.mat"), {"Y": Y, "S": S, "R": R})
    m = sio.loadmat(str(tmp_path / "ours.mat"))
    assert np.array_equal(m["Y"], Y) and m["Y"].dtype == np.complex64
    assert np.array_equal(m["S"], S) and np.array_equal(m["R"], R)
    # scipy -> ours (includes MATLAB-style narrowed storage of integral doubles)
    ints = np.arange(12, dtype=np.float64).reshape(3, 4)
    sio.savemat(str(tmp_path / "sp.mat"), {"Y": Y, "S": S, "ints": ints, "u": np.uint8([[1, 2, 255]])},
                do_compression=False)
    b = h.read_mat(str(tmp_path / "sp.mat"))
    assert np.array_equal(b["Y"], Y) and b["Y"].dtype == np.complex64
    assert np.array_equal(b["S"], S) and np.array_equal(b["ints"], ints)
    assert np.array_equal(b["u"], np.uint8([[1, 2, 255]]))


def test_mat_rejects_unsupported_features(tmp_path):
    a = np.ones((3, 3), np.complex64)
    sio.savemat(str(tmp_path / "c.mat"), {"a": a}, do_compression=True)
    with pytest.raises(h.UnsupportedFeature, match="compression"):
        h.read_mat(str(tmp_path / "c.mat"))
    sio.savemat(str(tmp_path / "cell.mat"), {"c": np.array([np.ones(2), np.ones(3)], dtype=object)})
    with pytest.raises(h.UnsupportedFeature, match="cell"):
        h.read_mat(str(tmp_path / "cell.mat"))
    sio.savemat(str(tmp_path / "st.mat"), {"s": {"a": 1.0}})
    with pytest.raises(h.UnsupportedFeature, match="struct"):
        h.read_mat(str(tmp_path / "st.mat"))
    sio.savemat(str(tmp_path / "ch.mat"), {"t": "hello"})
    with pytest.raises(h.UnsupportedFeature, match="char"):
        h.read_mat(str(tmp_path / "ch.mat"))
    import scipy.sparse as sp
    sio.savemat(str(tmp_path / "sp.mat"), {"m": sp.eye(3, format="csc")})
    with pytest.raises(h.UnsupportedFeature, match="sparse"):
        h.read_mat(str(tmp_path / "sp.mat"))
    # big-endian header
    h.write_mat(str(tmp_path / "le.mat"), {"a": a})
    raw = bytearray((tmp_path / "le.mat").read_bytes())
    raw[126:128] = b"MI"
    with pytest.raises(h.UnsupportedFeature, match="big-endian"):
        h.parse_mat(bytes(raw))
    with pytest.raises(h.IoError):
        h.read_mat(str(tmp_path / "missing.mat"))


def test_mat_fuzz_never_crashes(tmp_path):
    """Readers never crash on corrupted input: they raise a hetreco error."""
    rng = np.random.default_rng(5)
    h.write_mat(str(tmp_path / "f.mat"), {"Y": rand_array(rng, np.complex64, (4, 4, 2)),
                                          "R": rand_array(rng, np.float64, (3, 2))})
    good = (tmp_path / "f.mat").read_bytes()
    for trial in range(400):
        b = bytearray(good)
        if trial % 3 == 0:
            b = b[: int(rng.integers(0, len(b)))]
        else:
            for _ in range(int(rng.integers(1, 6))):
                b[int(rng.integers(0, len(b)))] = int(rng.integers(0, 256))
        try:
            h.parse_mat(bytes(b))
        except h.HetrecoError:
            pass


def test_mat_rejects_oversized_dimensions():
    """A corrupt dimension block must be rejected before any allocation."""
    hdr = b"MATLAB 5.0 MAT-file".ljust(116, b" ") + b"\x00" * 8 + struct.pack("<H", 0x0100) + b"IM"
    body = struct.pack("<II", 6, 8) + struct.pack("<II", 7, 0)          # flags: single
    body += struct.pack("<II", 5, 8) + struct.pack("<ii", 2**30, 2**30)  # dims 2^30 x 2^30
    body += struct.pack("<HH", 1, 1) + b"a\x00\x00\x00"                  # small-element name
    body += struct.pack("<II", 7, 8) + b"\x00" * 8                      # 2 floats of data
    blob = hdr + struct.pack("<II", 14, len(body)) + body
    with pytest.raises(h.MalformedFile):
        h.parse_mat(blob)


# ---- PGM / PPM ------------------------------------------------------------------------------

def test_pnm_roundtrip_and_spec_examples(tmp_path):
    rng = np.random.default_rng(6)
    for i in range(200):
        w, hh = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        color = i % 2 == 1
        a = rng.integers(0, 256, (3, w, hh) if color else (w, hh), dtype=np.uint8)
        p = str(tmp_path / f"i{i}.{'ppm' if color else 'pgm'}")
        h.write_image(p, a)
        assert np.array_equal(h.read_image(p), a)
    # "P5 2 2 255" + 4 bytes -> 2x2 array; comments allowed in the header
    (tmp_path / "s.pgm").write_bytes(b"P5\n# comment\n2 2\n255\n" + bytes([0, 64, 128, 255]))
    s = h.read_image(str(tmp_path / "s.pgm"))
    assert s.shape == (2, 2) and s.dtype == np.uint8
    assert s[:, 0].tolist() == [0, 64] and s[:, 1].tolist() == [128, 255]  # rows are x-fastest
    # ASCII variant and maxval != 255 are unsupported
    (tmp_path / "a.pgm").write_bytes(b"P2\n2 2\n255\n0 1 2 3\n")
    with pytest.raises(h.UnsupportedFeature):
        h.read_image(str(tmp_path / "a.pgm"))
    (tmp_path / "m.pgm").write_bytes(b"P5\n1 1\n65535\n\x00\x00")
    with pytest.raises(h.UnsupportedFeature):
        h.read_image(str(tmp_path / "m.pgm"))
    (tmp_path / "t.pgm").write_bytes(b"P5\n4 4\n255\n\x00")
    with pytest.raises(h.MalformedFile):
        h.read_image(str(tmp_path / "t.pgm"))
    # FLOAT32 in [0,1] maps by round(v*255), clamped
    f = np.array([[0.0, 0.5], [1.0, 2.0]], np.float32)
    h.write_image(str(tmp_path / "f.pgm"), f)
    assert h.read_image(str(tmp_path / "f.pgm")).tolist() == [[0, 128], [255, 255]]


# ---- raw + sidecar ------------------------------------------------------------------------------

def test_raw_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(7)
    for i in range(200):
        dtype = DTYPES[i % len(DTYPES)]
        shape = tuple(int(x) for x in rng.integers(1, 5, int(rng.integers(1, 9))))
        a = np.asfortranarray(rand_array(rng, dtype, shape))
        p, sc = str(tmp_path / f"r{i}.raw"), str(tmp_path / f"r{i}.txt")
        h.write_raw(p, sc, a)
        b = h.read_raw(p, sc)
        assert b.dtype == a.dtype and b.shape == a.shape and b.tobytes(order="F") == a.tobytes(order="F")
    a = np.ones((4, 4), np.float32)
    p, sc = str(tmp_path / "x.raw"), str(tmp_path / "x.txt")
    h.write_raw(p, sc, a)
    # truncated payload -> SizeMismatch
    with open(p, "r+b") as fh:
        fh.truncate(60)
    with pytest.raises(h.SizeMismatch):
        h.read_raw(p, sc)
    # sidecar rank 9 -> MalformedSidecar
    with open(sc, "w") as fh:
        fh.write("hetreco-raw 1\nelement_type 3\nrank 9\ndims 1 1 1 1 1 1 1 1 1\nbyte_order little\n")
    with pytest.raises(h.MalformedSidecar):
        h.read_raw(p, sc)
    with open(sc, "w") as fh:
        fh.write("hetreco-raw 1\nelement_type 3\nrank 2\ndims 4 4\nbyte_order big\n")
    with pytest.raises(h.MalformedSidecar):
        h.read_raw(p, sc)
    assert os.path.exists(p)
