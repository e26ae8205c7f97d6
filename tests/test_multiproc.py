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


# ---- sharded giant filter (C5): the exchange protocol on gloo --------------
class _GlooComm:
    def __init__(self, dist_):
        self.dist = dist_

    def allgather(self, obj):
        out = [None] * self.dist.get_world_size()
        self.dist.all_gather_object(out, obj)
        return out


def _shard_worker(rank, world, port, q, K, mode):
    import sys

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import reference_port as rp
        from oracle import sharded

        frames, _ = rp.generate_video(rp.Params(), 4, 64, 48, (30.0, 20.0), 11)
        traj = sharded.run_shard(frames, K, mode, 9, rank, world, _GlooComm(dist))
        q.put((rank, traj))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,K", [("fp16", 5000), ("fp64", 3100), ("fp32", 4097)])
def test_gloo_sharded_filter_protocol_equals_single(mode, K):
    """Two ranks, one filter split by particle range, exchanging only the max,
    (mass total, subtree roots) and peer-read table/CDF/positions: equals the
    unsharded fused algorithm bit-for-bit."""
    from oracle import fused
    from oracle import reference_port as rp

    frames, _ = rp.generate_video(rp.Params(), 4, 64, 48, (30.0, 20.0), 11)
    ref, _ = fused.run(frames, K, mode, 9)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q, K, mode)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, traj in res:
        assert np.array_equal(traj, ref), (rank, traj[:2], ref[:2])


def test_shard_layout_matches_library_rule():
    from oracle.sharded import shard_tiles
    from paper_2308_00763_b200.sharded import shard_layout

    for K in (2048, 10_000, 300_007, 1 << 30):
        for S in (2, 3, 4, 8):
            try:
                st, lay = shard_layout(K, S)
            except ValueError:
                with pytest.raises(ValueError):
                    shard_tiles(K, S)
                continue
            assert st == shard_tiles(K, S)
            assert st & (st - 1) == 0
            assert sum(c for _, c in lay) == K and all(c > 0 for _, c in lay)
            assert [f for f, _ in lay] == [r * st * 1024 for r in range(S)]


def test_bench_relaunches_under_torchrun(monkeypatch):
    # `python bench.py --gpus N` (no launcher) re-runs itself under torchrun,
    # one rank per GPU on a 127.0.0.1 rendezvous
    import sys as _sys

    import bench

    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(_sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    bench.main()
    (cmd,) = calls
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]


def test_bench_rejects_world_size_mismatch(monkeypatch):
    import sys as _sys

    import bench

    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(_sys, "argv", ["bench.py", "--gpus", "4"])
    with pytest.raises(SystemExit):
        bench.main()
