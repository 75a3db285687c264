"""Multi-GPU plumbing: one process per GPU, the scene
replicated, frames of the trajectory partitioned by view.  There is no
collective on the per-frame path of the throughput mode: each rank's worker
owns a private cache and renders a contiguous block of frames;
torch.distributed is used only for the start barrier and the max-over-ranks
timing reduction.  Two optional pieces of SURVEY §8(e): the eye-split latency
mode (ranks 2k and 2k+1 render the left and right eye of the same frames, each
with its own monocular pipeline) and the final image gather to rank 0 (the
paper gathers the results to the HMD's buffer) -- the one collective,
NCCL on the GPU box."""
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


def eye_split(rank: int, world: int, n_traj: int, count: int):
    """Eye-split latency mode: ranks 2k and 2k+1 form pair k and render the left (even rank)
    and right (odd rank) eye of the same frames; the world // 2 pairs take contiguous frame blocks.
    Returns (eye, frames).  Each eye pipeline culls and derives on its own (no de-redundancy across the
    pair), so this mode trades throughput for per-frame latency."""
    if world < 2 or world % 2:
        raise ValueError("eye-split needs an even number of ranks")
    return rank % 2, frame_block(rank // 2, world // 2, n_traj, count)


def gather_images(img, dst: int = 0):
    """Gather every rank's image tensor (same shape and dtype on all ranks) to rank `dst`: the list of
    images in rank order on dst, None elsewhere (NCCL on the GPU: device tensors; gloo: CPU tensors)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [img]
    rank = dist.get_rank()
    out = [torch.empty_like(img) for _ in range(dist.get_world_size())] if rank == dst else None
    dist.gather(img, gather_list=out, dst=dst)
    return out
