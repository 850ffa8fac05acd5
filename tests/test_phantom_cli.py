"""gen_phantom and the `hetreco` CLI (SPEC.md:449-457 and
the cli module :535-579).

CPU part: the seeded blob parameters of the C++ generator equal the oracle
port's (same mt19937_64 stream), CLI usage errors and `devices`.
GPU part (marked): the device phantom vs the CPU port, the forward-model
acceptance criterion (sens_recon recovers M_true <= 1e-4 rel. L2), and the
CLI's gen-phantom -> reconstruct / negate / bench commands end to end.
"""
import csv
import io
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as o
from paper_1807_11830_b200 import hetreco as h

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1807_11830_b200", "bin", "hetreco")


def run_cli(*args, check=True):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    if check and r.returncode != 0:
        raise AssertionError(f"hetreco {' '.join(map(str, args))} -> {r.returncode}: {r.stderr}")
    return r


def rel_l2(a, ref):
    return float(np.linalg.norm((np.asarray(a) - ref).ravel()) / np.linalg.norm(np.asarray(ref).ravel()))


# ---- CPU ---------------------------------------------------------------------------------

@pytest.mark.parametrize("nx,ny,seed", [(128, 128, 1), (256, 64, 7), (16, 16, 2**40 + 3)])
def test_phantom_blobs_match_port(nx, ny, seed):
    assert h.phantom_blobs(nx, ny, seed) == [tuple(b) for b in o.phantom_blobs(nx, ny, seed)]


def test_cli_usage_errors_and_devices(tmp_path):
    assert os.path.exists(CLI), "CLI not built (python -m paper_1807_11830_b200.build)"
    r = run_cli("devices")
    assert r.returncode == 0 and "backend" in r.stdout
    devs = json.loads(run_cli("devices", "--json").stdout)
    assert isinstance(devs, list) and all(d["vendor"] == "NVIDIA" for d in devs)
    assert run_cli("frobnicate", check=False).returncode == 2
    r = run_cli("reconstruct", "--kdata", tmp_path / "k.mat", "--method", "sens", "--output", tmp_path / "o.mat",
                check=False)
    assert r.returncode == 2 and "--smaps" in r.stderr and r.stderr.count("\n") == 1  # one-line diagnostic
    r = run_cli("bench", "--op", "rss", check=False)
    assert r.returncode == 2 and "--sizes" in r.stderr
    r = run_cli("negate", "--input", tmp_path / "missing.pgm", "--output", tmp_path / "o.pgm", check=False)
    assert r.returncode != 0 and "missing.pgm" in r.stderr


def test_cli_compile_surfaces_log(tmp_path):
    """A deliberately broken unit: CompileError whose log reaches the CLI's
    exit message verbatim."""
    if not h.nvrtc_available():
        pytest.skip("libnvrtc not available")
    good = tmp_path / "good.cl.src"
    good.write_text("HETRECO_KERNEL(twice) { (void)gsize; float* o = (float*)hetreco_array_out(args, 0);"
                    " o[gid] = 2.0f * ((const float*)hetreco_array_in(args, 0))[gid]; }\n")
    r = run_cli("compile", "--source", good)
    assert r.returncode == 0 and "good.cl.src: twice" in r.stdout
    bad = tmp_path / "bad.cl.src"
    bad.write_text("HETRECO_KERNEL(bad) {\n  undeclared_thing = 1;\n}\n")
    r = run_cli("compile", "--source", good, "--source", bad, check=False)
    assert r.returncode == 4
    assert "bad.cl.src(2): error" in r.stderr and "undeclared_thing" in r.stderr


# ---- GPU ---------------------------------------------------------------------------------

@pytest.fixture(scope="module")
def s():
    sess = h.ComputeSession("gpu")
    yield sess
    sess.close()


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,nf,nc,seed", [(128, 128, 16, 8, 1), (64, 32, 3, 1, 5), (256, 256, 2, 12, 9)])
def test_gen_phantom_vs_port(s, nx, ny, nf, nc, seed):
    Y, S, M = h.gen_phantom(s, nx, ny, nf, nc, seed)
    Yo, So, Mo = o.gen_phantom(nx, ny, nf, nc, seed)
    assert np.abs(M - Mo).max() <= 1e-6 * np.abs(Mo).max()
    assert np.abs(S - So).max() <= 1e-6
    assert np.abs(Y - Yo).max() <= 1e-5 * np.abs(Yo).max()
    # sum_i |S_i|^2 = 1 +- 1e-6 everywhere
    assert np.abs((np.abs(S.astype(np.complex128)) ** 2).sum(axis=2) - 1).max() <= 1e-6
    # determinism: same seed twice -> bit-identical
    Y2, S2, M2 = h.gen_phantom(s, nx, ny, nf, nc, seed)
    assert Y.tobytes() == Y2.tobytes() and S.tobytes() == S2.tobytes() and M.tobytes() == M2.tobytes()


@pytest.mark.gpu
def test_phantom_forward_model_recovery(s):
    """Acceptance criterion 1: gen_phantom(128,128,16,8,seed=1);
    sens_recon recovers M_true with relative L2 error <= 1e-4."""
    Y, S, M = h.gen_phantom(s, 128, 128, 16, 8, 1)
    hin = s.register_data(h.Data([Y, S], h.DataKind.KData))
    hout = s.allocate_data([((128, 128, 16), np.complex64)])
    p = h.Process(s, "sens_recon").set_input(hin).set_output(hout).init()
    p.launch()
    R = s.fetch_data(hout).arrays[0]
    assert rel_l2(R, M) <= 1e-4
    with pytest.raises(h.InvalidParams):
        h.gen_phantom(s, 100, 128, 2, 2, 1)


@pytest.mark.gpu
def test_cli_phantom_reconstruct_roundtrip(tmp_path):
    k, sm, t, out = (str(tmp_path / n) for n in ("k.mat", "s.mat", "t.mat", "o.mat"))
    run_cli("gen-phantom", "--nx", 128, "--ny", 128, "--frames", 16, "--coils", 8, "--seed", 1,
            "--out-kdata", k, "--out-smaps", sm, "--out-truth", t)
    truth = h.read_mat(t)["truth"]
    assert h.read_mat(k)["kdata"].shape == (128, 128, 8, 16) and h.read_mat(sm)["smaps"].shape == (128, 128, 8)
    run_cli("reconstruct", "--kdata", k, "--smaps", sm, "--method", "sens", "--output", out)
    img = h.read_mat(out)["image"]
    assert img.dtype == np.complex64 and rel_l2(img, truth) <= 1e-4
    # rss on 1-coil data = modulus image
    k1 = str(tmp_path / "k1.mat")
    run_cli("gen-phantom", "--nx", 64, "--ny", 64, "--frames", 2, "--coils", 1, "--seed", 3,
            "--out-kdata", k1, "--out-smaps", str(tmp_path / "s1.mat"), "--out-truth", str(tmp_path / "t1.mat"))
    run_cli("reconstruct", "--kdata", k1, "--method", "rss", "--output", out)
    rss = h.read_mat(out)["image"]
    t1 = h.read_mat(str(tmp_path / "t1.mat"))["truth"]
    s1 = h.read_mat(str(tmp_path / "s1.mat"))["smaps"]
    assert rss.dtype == np.float32
    assert np.abs(rss - np.abs(t1 * s1[..., :1])).max() <= 1e-5 * np.abs(t1).max()
    assert run_cli("gen-phantom", "--nx", 100, "--out-kdata", k, "--out-smaps", sm, "--out-truth", t,
                   check=False).returncode != 0


@pytest.mark.gpu
def test_cli_negate(tmp_path):
    black = np.zeros((17, 9), np.uint8)
    h.write_image(str(tmp_path / "b.pgm"), black)
    run_cli("negate", "--input", tmp_path / "b.pgm", "--output", tmp_path / "w.pgm")
    assert (h.read_image(str(tmp_path / "w.pgm")) == 255).all()  # black -> white
    rng = np.random.default_rng(1)
    a = rng.integers(0, 256, (33, 20), dtype=np.uint8)
    h.write_image(str(tmp_path / "a.pgm"), a)
    run_cli("negate", "--input", tmp_path / "a.pgm", "--output", tmp_path / "n.pgm")
    run_cli("negate", "--input", tmp_path / "n.pgm", "--output", tmp_path / "nn.pgm")
    assert np.array_equal(h.read_image(str(tmp_path / "nn.pgm")), a)  # involution


@pytest.mark.gpu
def test_cli_bench_csv(tmp_path):
    c = str(tmp_path / "b.csv")
    run_cli("bench", "--op", "matadd", "--sizes", "256,512,1024", "--repeats", 20, "--csv", c)
    rows = list(csv.DictReader(open(c)))
    assert [r["size"] for r in rows] == ["256", "512", "1024"]
    for r in rows:
        assert int(r["repeats"]) == 20 and float(r["mean_s"]) > 0 and float(r["init_s"]) > 0
        assert float(r["stddev_s"]) >= 0 and float(r["speedup"]) > 0
    out = run_cli("bench", "--op", "rss", "--sizes", "128x128x16x8", "--repeats", 10).stdout
    rows = list(csv.DictReader(io.StringIO(out)))
    assert len(rows) == 1 and rows[0]["op"] == "rss" and float(rows[0]["mean_s"]) > 0 and rows[0]["speedup"] == ""
    for op, size in (("sens", "256x256x4x8"), ("fft", "256x256x4"), ("negate", "512")):
        assert float(list(csv.DictReader(io.StringIO(run_cli("bench", "--op", op, "--sizes", size, "--repeats",
                                                                5).stdout)))[0]["mean_s"]) > 0
    # deterministic timing -> byte-identical CSV
    a = run_cli("bench", "--op", "matadd", "--sizes", "64", "--repeats", 1, "--deterministic-timing").stdout
    b = run_cli("bench", "--op", "matadd", "--sizes", "64", "--repeats", 1, "--deterministic-timing").stdout
    assert a == b
