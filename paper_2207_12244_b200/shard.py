"""Multi-GPU work partitioning.

Two forms, both from the reference's data independence:
  * independent keyframes (config C3): keyframe k -> rank k mod N, frames of a
    keyframe stay sequential on that rank; no data-path
    collective;
  * row bands of one large keyframe (config C4): rank g owns rows
    [r_g, r_{g+1}); its PCG needs a one-row halo of p per iteration and the
    CG scalars all-reduced.

Only the host-side bookkeeping lives here; it is exercised on CPU with the
gloo backend (tests/test_dist_cpu.py).
"""
from __future__ import annotations


def keyframes_for_rank(n_keyframes: int, world: int, rank: int) -> list[int]:
    """Round-robin keyframe ownership: k -> k mod world."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(rank, n_keyframes, world))


def row_bands(height: int, world: int) -> list[tuple[int, int]]:
    """Near-equal contiguous row bands [r0, r1) per rank."""
    if world <= 0 or height <= 0:
        raise ValueError("bad height/world")
    return [(height * g // world, height * (g + 1) // world) for g in range(world)]


def band_halo(height: int, world: int, rank: int) -> tuple[int, int]:
    """Rows a rank reads beyond its band for one 5-point stencil sweep:
    (rows above, rows below) -- one each way unless at the raster edge."""
    r0, r1 = row_bands(height, world)[rank]
    return (1 if r0 > 0 else 0, 1 if r1 < height else 0)


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar (timing is reported as the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    backend = dist.get_backend()
    dev = "cuda" if backend == "nccl" else "cpu"
    if dev == "cuda":
        dev = f"cuda:{torch.cuda.current_device()}"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
