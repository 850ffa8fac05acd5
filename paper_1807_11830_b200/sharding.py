"""Frame-slab partitioning for multi-GPU reconstruction (SURVEY.md §8 e).

Frames are independent (Eq. 1 is per frame), so N GPUs split the frame axis
into contiguous slabs -- one contiguous byte range of the column-major
[nx, ny, coils, frames] k-space per GPU, one cudaMemcpyAsync each, no gather
and no collective on the data path.  Only timing scalars cross ranks.
"""
from __future__ import annotations


def frame_slab(rank: int, world: int, frames: int) -> tuple[int, int]:
    """[begin, end) frames of `rank` (floor partition, sizes differ by <= 1)."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world of {world}")
    return (rank * frames) // world, ((rank + 1) * frames) // world


def slab_bytes(begin: int, end: int, nx: int, ny: int, coils: int, elem: int = 8) -> tuple[int, int]:
    """(byte offset, byte length) of a frame slab inside [nx, ny, coils, frames]."""
    per = nx * ny * coils * elem
    return begin * per, (end - begin) * per


def imbalance(world: int, frames: int) -> float:
    """max slab / mean slab - 1 (e.g. 30 frames on 8 GPUs -> 4,4,4,4,4,4,3,3 = 6.7 %)."""
    sizes = [e - b for b, e in (frame_slab(r, world, frames) for r in range(world))]
    return max(sizes) / (frames / world) - 1.0


def max_over_ranks(value: float, group=None) -> float:
    """All-reduce MAX of one timing scalar (the only cross-rank traffic)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
