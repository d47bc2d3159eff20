"""Host-side multi-GPU logic on CPU:
batch sharding by image (Eq. 1 has no cross-image term), the
shard-independence of the seeded data, and the max/sum-over-ranks reductions
the bench uses -- exercised with world_size-2 gloo process groups."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1704_07724_b200 import datagen, shard


@pytest.mark.parametrize("n_total,ws", [(1024, 1), (1024, 2), (1024, 8), (1000, 3), (5, 8), (0, 2)])
def test_shard_range_partitions_the_batch(n_total, ws):
    ranges = [shard.shard_range(n_total, r, ws) for r in range(ws)]
    covered = [i for lo, hi in ranges for i in range(lo, hi)]
    assert covered == list(range(n_total))                      # disjoint, ordered, complete
    sizes = [hi - lo for lo, hi in ranges]
    assert max(sizes) - min(sizes) <= 1                         # balanced


def test_shard_range_rejects_bad_arguments():
    for args in ((10, 2, 2), (10, -1, 2), (10, 0, 0), (-1, 0, 1)):
        with pytest.raises(ValueError):
            shard.shard_range(*args)


def test_weak_scaling_sets_tile_the_image_sequence():
    n = 4
    for ws in (1, 2, 8):
        starts = sorted(shard.image_start(si, r, ws, n) for si in range(3) for r in range(ws))
        assert starts == [n * i for i in range(3 * ws)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        env = shard.dist_env()
        assert env == (ws, rank, rank)
        shp = datagen.C5_LAYERS[0].with_batch(8)
        lo, hi = shard.shard_range(shp.n, rank, ws)
        x = datagen.activations(shp, datagen.C5_FIRST_SPARSITY, start=lo, count=hi - lo)
        # every rank's slice, gathered (verification-only collective)
        parts = [None] * ws
        dist.all_gather_object(parts, (lo, hi, [datagen.sha256(xi) for xi in x]))
        shard.barrier(ws)
        mx = shard.max_over_ranks(float(rank + 1) * 1.5, ws)
        sm = shard.sum_over_ranks(float(hi - lo), ws)
        q.put((rank, parts, mx, sm))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_reduce():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shp = datagen.C5_LAYERS[0].with_batch(8)
    ref = datagen.activations(shp, datagen.C5_FIRST_SPARSITY)   # one process, the whole batch
    for rank, parts, mx, sm in results:
        assert mx == 3.0                                          # max over ranks of 1.5*(rank+1)
        assert sm == 8.0                                          # every image counted once
        seen = []
        for lo, hi, hashes in parts:
            assert hashes == [datagen.sha256(ref[i]) for i in range(lo, hi)]   # shard-independent data
            seen += list(range(lo, hi))
        assert seen == list(range(8))
