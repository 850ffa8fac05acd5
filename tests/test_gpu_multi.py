"""Multi-GPU frame-slab reconstruction through the library (hetreco_multi_*).

One host volume is split into contiguous frame slabs, one worker thread +
ComputeSession + streaming pipeline per backend id.  The round's GPU box has a
single B200, so the slabs run on repeated ids ("cuda0" twice / three times):
the partition, the per-slab byte ranges, the stitching and the error paths are
the same code an 8-GPU box runs with "cuda0".."cuda7".  Oracle: the C port
(reference-pinned, tests/test_oracle.py) of the SENSE / RSS chains.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as o
from paper_1807_11830_b200 import hetreco as h

pytestmark = pytest.mark.gpu

TOL = 1e-5
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def relmax(a, ref):
    return float(np.abs(np.asarray(a) - ref).max() / max(float(np.abs(ref).max()), 1e-30))


def volume(rng, nx, ny, nc, nf):
    Y = h.pinned_empty((nx, ny, nc, nf), np.complex64)
    Y[...] = rng.standard_normal((nx, ny, nc, nf)) + 1j * rng.standard_normal((nx, ny, nc, nf))
    S = np.asfortranarray((rng.standard_normal((nx, ny, nc)) + 1j * rng.standard_normal((nx, ny, nc)))
                          .astype(np.complex64))
    return Y, S


@pytest.mark.parametrize("method", ["sense", "rss"])
@pytest.mark.parametrize("slabs,nf,chunk", [(2, 9, 2), (3, 2, 1), (4, 30, 3), (1, 5, 5)])
def test_multi_gpu_slabs_stitch_to_oracle(method, slabs, nf, chunk):
    rng = np.random.default_rng(slabs * 100 + nf)
    nx, ny, nc = 64, 32, 4
    Y, S = volume(rng, nx, ny, nc, nf)
    ref = o.sens_recon(np.asfortranarray(Y), S) if method == "sense" else o.rss_recon(np.asfortranarray(Y))
    out = h.pinned_empty((nx, ny, nf), np.complex64 if method == "sense" else np.float32)
    out[...] = np.nan
    mg = h.MultiGpuRecon(["cuda0"] * slabs, method, nx, ny, nc, chunk, S if method == "sense" else None)
    mg.run(Y, out)
    assert relmax(out, ref) <= TOL
    info = mg.slabs()
    assert [(d["first_frame"], d["first_frame"] + d["frames"]) for d in info] == \
        [h.frame_slab(i, slabs, nf) for i in range(slabs)]
    assert sum(d["frames"] for d in info) == nf
    # re-run: same bits (the workers and their pipelines are persistent)
    again = np.empty_like(out)
    mg.run(Y, again)
    assert again.tobytes() == out.tobytes()
    mg.close()


def test_multi_gpu_matches_single_stream_bitexact():
    """Slabbing changes nothing numerically: every frame is reconstructed by
    the same kernels whichever slab it lands in (chunk 1 on both sides, so the
    launch shapes agree frame for frame)."""
    rng = np.random.default_rng(7)
    nx, ny, nc, nf = 128, 128, 6, 7
    Y, S = volume(rng, nx, ny, nc, nf)
    s = h.ComputeSession("gpu")
    one = h.pinned_empty((nx, ny, nf), np.complex64)
    h.StreamingRecon(s, "sense", nx, ny, nc, 1, S).run(Y, one)
    two = h.pinned_empty((nx, ny, nf), np.complex64)
    h.MultiGpuRecon(["cuda0", "cuda0"], "sense", nx, ny, nc, 1, S).run(Y, two)
    assert one.tobytes() == two.tobytes()
    s.close()


def test_multi_gpu_c5_shape_two_slabs():
    """C5 geometry (512^2 x 32 coils, 2-frame chunks, ragged tail) split over
    two slabs, RSS, against the oracle port."""
    rng = np.random.default_rng(55)
    nx = ny = 512
    nc, nf = 32, 5
    Y, _ = volume(rng, nx, ny, nc, nf)
    out = h.pinned_empty((nx, ny, nf), np.float32)
    h.MultiGpuRecon(["cuda0", "cuda0"], "rss", nx, ny, nc, 2).run(Y, out)
    for f in (0, 2, 4):  # one frame of each slab and the tail, oracle cost bounded
        ref = o.rss_recon(np.asfortranarray(Y[..., f:f + 1]))
        assert relmax(out[..., f:f + 1], ref) <= TOL


def test_multi_gpu_errors():
    with pytest.raises(h.HetrecoError):
        h.MultiGpuRecon([], "rss", 64, 64, 2, 1)
    with pytest.raises(h.HetrecoError):
        h.MultiGpuRecon(["cuda0", "cuda99"], "rss", 64, 64, 2, 1)  # unknown backend: nothing leaks
    with pytest.raises(h.HetrecoError):
        h.MultiGpuRecon(["cuda0"], "rss", 100, 64, 2, 1)  # unsupported FFT size
    with pytest.raises(h.HetrecoError):
        h.MultiGpuRecon(["cuda0"], "sense", 64, 64, 2, 1)  # SENSE without maps
    mg = h.MultiGpuRecon(["cuda0"], "rss", 64, 64, 2, 1)
    out = np.zeros((64, 64, 0), np.float32, order="F")
    mg.run(np.zeros((64, 64, 2, 0), np.complex64, order="F"), out)  # zero frames: no-op
    assert mg.slabs()[0]["frames"] == 0


def test_one_context_per_process():
    """Enumerating devices opens no CUDA context (lazy backends): a process
    that lists every GPU and uses one of them holds exactly one context, so N
    ranks on an N-GPU box hold N contexts, not N^2."""
    code = (
        "import ctypes, sys\n"
        "sys.path.insert(0, %r)\n"
        "from paper_1807_11830_b200 import hetreco as h\n"
        "devs = h.enumerate_devices()\n"
        "cu = ctypes.CDLL('libcuda.so.1')\n"
        "def ctxs():\n"
        "    n = 0\n"
        "    for i in range(len(devs)):\n"
        "        dev = ctypes.c_int(); cu.cuDeviceGet(ctypes.byref(dev), i)\n"
        "        flags = ctypes.c_uint(); active = ctypes.c_int()\n"
        "        cu.cuDevicePrimaryCtxGetState(dev, ctypes.byref(flags), ctypes.byref(active))\n"
        "        n += active.value\n"
        "    return n\n"
        "cu.cuInit(0)\n"
        "before = ctxs()\n"
        "s = h.ComputeSession(device=devs[-1])\n"
        "s.register_data([__import__('numpy').zeros(4, 'f4')])\n"
        "print(len(devs), before, ctxs())\n" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    n, before, after = map(int, r.stdout.split()[-3:])
    assert n >= 1 and before == 0 and after == 1, r.stdout


def test_bench_two_ranks_on_one_gpu():
    """The multi-rank bench path (torchrun, one process per rank, frame slabs of
    one C3 volume, no data-path collective) as a dry run: two ranks pinned to
    GPU 0 with gloo carrying only the barrier and the max-over-ranks timing."""
    import json
    import os
    env = dict(os.environ, HETRECO_BENCH_DEVICE="0", HETRECO_BENCH_DIST="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-extras", "--no-cpu-baseline",
           "--no-session-flow", "--no-weak"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    b = lines[0]
    assert b["n_gpus"] == 2 and b["scaling"] == "strong" and b["value"] > 0
    assert b["sharding"]["frames_per_gpu"] == [15, 15]
    assert b["e2e"]["matches_resident"] is True
    assert b["config"]["parallelism"].startswith("frame-slab x2")
