"""Batch sharding across GPUs.

Images are independent (Eq. 1 has no cross-image term), so the
path shards by image with no collective on the data path.  This module holds
the host-side logic only: which images a rank owns, the process group setup,
and the two reductions the bench needs (barrier, max/sum of a scalar over
ranks).  It runs under NCCL on GPUs and under gloo on CPU (tests).
"""
from __future__ import annotations

import os


def dist_env():
    """(world_size, rank, local_rank) from the torchrun environment."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def shard_range(n_total, rank, ws):
    """Images [lo, hi) of rank `rank` when n_total images are split over ws
    ranks as evenly as possible (strong scaling, e.g. C5's 1024 images)."""
    if ws < 1 or not 0 <= rank < ws or n_total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_total, ws)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def image_start(set_index, rank, ws, n_per_rank):
    """Global index of the first image of input set `set_index` on `rank` when
    every rank processes its own n_per_rank images (weak scaling).  Sets of all
    ranks tile the global image sequence, so the data never depends on ws."""
    return (set_index * ws + rank) * n_per_rank


def shares_gpus():
    """SC_DIST_BACKEND=gloo: a functional check of the multi-rank path on a box with fewer GPUs
    than ranks -- ranks share GPUs round-robin and synchronise over gloo on the host (their
    kernels never wait on one another: no collective on the data path).  Not a scaling number."""
    return os.environ.get("SC_DIST_BACKEND", "nccl") == "gloo"


def init(ws, local, backend=None):
    """Bind this process to its GPU and, for ws > 1, join the process group (NCCL, one GPU
    per rank; gloo with GPUs shared round-robin when SC_DIST_BACKEND=gloo)."""
    import torch
    gloo = shares_gpus() if backend is None else backend == "gloo"
    idx = local % max(1, torch.cuda.device_count()) if gloo else local
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(idx)
        if not dist.is_initialized():
            if gloo:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", idx))
    dev = torch.device("cuda", idx if ws > 1 else 0)
    torch.cuda.set_device(dev)
    return dev


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def _reduce(value, ws, device, op):
    if ws == 1:
        return float(value)
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "gloo":
        device = None  # host tensors (gloo)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(value, ws, device=None):
    """Max of a per-rank scalar (device-timed elapsed times: the job takes as
    long as its slowest rank)."""
    if ws == 1:
        return float(value)
    import torch.distributed as dist
    return _reduce(value, ws, device, dist.ReduceOp.MAX)


def sum_over_ranks(value, ws, device=None):
    if ws == 1:
        return float(value)
    import torch.distributed as dist
    return _reduce(value, ws, device, dist.ReduceOp.SUM)


def finalize(ws):
    if ws > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
