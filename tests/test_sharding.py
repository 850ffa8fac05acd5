"""Multi-GPU host logic on CPU: frame slabs cover the frame axis exactly once
with no overlap, and the only cross-rank exchange (max of the timing scalar)
works over a world_size-2 gloo group (the same code path bench.py uses over
NCCL)."""
import os

import pytest

from paper_1807_11830_b200.sharding import frame_slab, imbalance, max_over_ranks, slab_bytes


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("frames", [1, 7, 30, 256])
def test_slabs_partition_frames(world, frames):
    covered = []
    for r in range(world):
        b, e = frame_slab(r, world, frames)
        assert 0 <= b <= e <= frames
        covered.extend(range(b, e))
        assert abs((e - b) - frames / world) < 1
    assert covered == list(range(frames))


def test_c3_imbalance_and_bytes():
    assert [frame_slab(r, 8, 30) for r in range(8)][0] == (0, 3)
    assert abs(imbalance(8, 30) - (4 / 3.75 - 1)) < 1e-12
    off, n = slab_bytes(4, 8, 256, 256, 32)
    assert off == 4 * 256 * 256 * 32 * 8 and n == 4 * 256 * 256 * 32 * 8


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = frame_slab(rank, world, 30)
    t = max_over_ranks(float(rank + 1) * 0.5)
    q.put((rank, b, e, t))
    dist.destroy_process_group()


def test_gloo_world2_max_over_ranks():
    import multiprocessing as mp
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(b, e) for _, b, e, _ in res] == [(0, 15), (15, 30)]
    assert all(t == 1.0 for *_, t in res)


def test_numa_cpulist_and_bind():
    """Host placement helpers used by each rank before it allocates its pinned
    slab (SURVEY.md §8 e)."""
    import os

    from paper_1807_11830_b200 import hetreco as h
    assert h.parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert h.parse_cpulist("5") == [5]
    with pytest.raises(h.InvalidArgument):
        h.parse_cpulist("3-1")
    with pytest.raises(h.InvalidArgument):
        h.parse_cpulist("a-b")
    assert h.bind_numa_node(-1) == 0  # no NUMA information: no-op
    before = os.sched_getaffinity(0)
    try:
        if os.path.exists("/sys/devices/system/node/node0/cpulist"):
            n = h.bind_numa_node(0)
            node0 = set(h.parse_cpulist(open("/sys/devices/system/node/node0/cpulist").read()))
            assert n == len(node0) and os.sched_getaffinity(0) <= node0
    finally:
        os.sched_setaffinity(0, before)


@pytest.mark.parametrize("count", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("frames", [0, 1, 7, 30, 256])
def test_library_frame_slab_matches_python(count, frames):
    """The C++ partition (hetreco_frame_slab, used by MultiGpuRecon) and the
    Python one (bench.py's ranks) agree slab for slab."""
    from paper_1807_11830_b200 import hetreco as h
    for i in range(count):
        assert h.frame_slab(i, count, frames) == frame_slab(i, count, frames)
    with pytest.raises(h.InvalidArgument):
        h.frame_slab(count, count, frames)


def _slab_worker(rank, world, port, q):
    """One rank of the strong-scaling path on CPU: reconstruct its frame slab
    with the oracle port (stand-in for its GPU), exchange nothing but the
    timing scalar, and hand its slab back for stitching."""
    import numpy as np
    import torch.distributed as dist

    from oracle import oracle as o
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nc, nf = 16, 8, 3, 7
    rng = np.random.default_rng(0)  # every rank sees the same volume
    Y = np.asfortranarray((rng.standard_normal((nx, ny, nc, nf)) + 1j * rng.standard_normal((nx, ny, nc, nf)))
                          .astype(np.complex64))
    S = np.asfortranarray((rng.standard_normal((nx, ny, nc)) + 1j * rng.standard_normal((nx, ny, nc)))
                          .astype(np.complex64))
    b, e = frame_slab(rank, world, nf)
    M = o.sens_recon(np.asfortranarray(Y[..., b:e]), S) if e > b else np.zeros((nx, ny, 0), np.complex64)
    t = max_over_ranks(float(e - b))
    q.put((rank, b, e, t, M.tobytes(order="F")))
    dist.destroy_process_group()


def test_gloo_world2_strong_scaling_stitches_slabs():
    """world_size-2 gloo: each rank reconstructs only its contiguous frame
    slab; the slabs stitch into the single-process result bit for bit."""
    import multiprocessing as mp
    import socket

    import numpy as np

    from oracle import oracle as o
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_slab_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted((q.get(timeout=120) for _ in ps), key=lambda r: r[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(b, e) for _, b, e, _, _ in res] == [(0, 3), (3, 7)]
    assert all(r[3] == 4.0 for r in res)  # max slab size over ranks
    nx, ny, nc, nf = 16, 8, 3, 7
    rng = np.random.default_rng(0)
    Y = np.asfortranarray((rng.standard_normal((nx, ny, nc, nf)) + 1j * rng.standard_normal((nx, ny, nc, nf)))
                          .astype(np.complex64))
    S = np.asfortranarray((rng.standard_normal((nx, ny, nc)) + 1j * rng.standard_normal((nx, ny, nc)))
                          .astype(np.complex64))
    full = o.sens_recon(Y, S)
    stitched = b"".join(r[4] for r in res)
    assert stitched == full.tobytes(order="F")
