"""Multi-rank host logic on CPU (gloo, world size 2): track sharding covers every
track exactly once with rank-independent seeds/videos; max-over-ranks and
trajectory gathering (the only collectives, timing/reporting only)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_00763_b200.sharding import gather_trajectories, max_over_ranks, shard_tracks


def test_shard_partition_properties():
    for total in (2, 7, 8, 8192, 10_001):
        for world in (1, 2, 3, 4, 8):
            if total < world:
                with pytest.raises(ValueError):
                    shard_tracks(total, world, 0)
                continue
            shards = [shard_tracks(total, world, r) for r in range(world)]
            idx = [s.first + i for s in shards for i in range(s.count)]
            assert idx == list(range(total))
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1
            seeds = [x for s in shards for x in s.seeds(42)]
            assert seeds == [42 + i for i in range(total)]
            vids = [x for s in shards for x in s.videos(8)]
            assert vids == [i % 8 for i in range(total)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = shard_tracks(5, world, rank)
        local = np.stack([np.full((3, 2), float(g)) for g in range(sh.first, sh.first + sh.count)])
        allt = gather_trajectories(local, dist)
        m = max_over_ranks(10.0 + rank, dist)
        q.put((rank, allt[:, 0, 0].tolist(), m))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, tracks, m in res:
        assert tracks == [0.0, 1.0, 2.0, 3.0, 4.0]
        assert m == 11.0
