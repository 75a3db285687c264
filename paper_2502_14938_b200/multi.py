"""Multi-GPU plumbing: one process per GPU, the scene
replicated, frames of the trajectory partitioned by view.  There is no
collective on the per-frame path: each rank's worker owns a private cache
 and renders a contiguous block of frames; torch.distributed is
used only for the start barrier and the max-over-ranks timing reduction."""
from __future__ import annotations

import os


def dist_env():
    """(rank, world_size, local_rank) from the torchrun environment (defaults 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def frame_block(rank: int, world: int, n_traj: int, count: int) -> list[int]:
    """Contiguous block partition (throughput mode): rank r starts
    at frame floor(r * n_traj / world) and renders `count` consecutive frames,
    wrapping around the trajectory.  Each rank's cache sees consecutive frames,
    so its hit rate matches a single-GPU run of that block."""
    if world < 1 or not (0 <= rank < world) or n_traj < 1 or count < 0:
        raise ValueError("bad partition arguments")
    start = (rank * n_traj) // world
    return [(start + k) % n_traj for k in range(count)]


def round_robin(rank: int, world: int, n_traj: int) -> list[int]:
    """Live/latency mode (paper's shared queue): frame f goes to rank f mod world."""
    return list(range(rank, n_traj, world))


def init(backend: str | None = None):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        dist.init_process_group(backend=backend)
    return rank, world, local


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def max_over_ranks(x: float, device=None) -> float:
    """Max of a scalar over all ranks (the slowest rank's time defines the box's rate)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
