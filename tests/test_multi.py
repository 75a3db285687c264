"""Host logic of the N > 1 path on CPU with gloo, world size 2:
frame partition by view, start barrier, max-over-ranks timing."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2502_14938_b200 import multi


def test_frame_block_partition():
    T = 600
    for world in (1, 2, 4, 8):
        blocks = [multi.frame_block(r, world, T, T // world) for r in range(world)]
        flat = sorted(f for b in blocks for f in b)
        assert flat == list(range(T))                      # every frame exactly once
        for b in blocks:
            assert all((y - x) % T == 1 for x, y in zip(b, b[1:]))   # consecutive (private cache reuse)
    # weak scaling: K frames per rank, wrapping around the trajectory
    assert multi.frame_block(1, 2, 10, 8) == [5, 6, 7, 8, 9, 0, 1, 2]
    assert multi.round_robin(1, 4, 10) == [1, 5, 9]
    with pytest.raises(ValueError):
        multi.frame_block(2, 2, 10, 1)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    r, w, _ = multi.init(backend="gloo")
    multi.barrier()
    t = 10.0 + 5.0 * r                                 # per-rank elapsed time
    tmax = multi.max_over_ranks(t)
    frames = multi.frame_block(r, w, 600, 300)
    total = multi.sum_over_ranks(len(frames))
    q.put((r, w, tmax, total, frames[0]))
    import torch.distributed as dist
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [x[0] for x in res] == [0, 1] and all(x[1] == 2 for x in res)
    assert all(x[2] == 15.0 for x in res)          # the slowest rank defines the box time
    assert all(x[3] == 600 for x in res)           # value = units of all ranks / max time
    assert [x[4] for x in res] == [0, 300]


def test_eye_split_assignment():
    """Eye-split latency mode: pairs (2k, 2k+1) render the two eyes of the same frames; the pairs split the
    trajectory in contiguous blocks."""
    for world in (2, 4, 8):
        got = [multi.eye_split(r, world, 600, 600 // (world // 2)) for r in range(world)]
        for k in range(world // 2):
            (el, fl), (er, fr) = got[2 * k], got[2 * k + 1]
            assert (el, er) == (0, 1) and fl == fr
        flat = sorted(f for r in range(0, world, 2) for f in got[r][1])
        assert flat == list(range(600))
    with pytest.raises(ValueError):
        multi.eye_split(0, 3, 10, 1)


def _gather_worker(rank, world, port, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    multi.init(backend="gloo")
    img = torch.full((4, 6, 4), rank + 1, dtype=torch.uint8)       # a rank's RGBA8 eye image
    out = multi.gather_images(img, dst=0)
    q.put((rank, None if out is None else [int(t.float().mean()) for t in out]))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_gloo_world2_image_gather():
    """The final image gather: rank 0 receives every rank's image in rank order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == [1, 2] and res[1] is None
