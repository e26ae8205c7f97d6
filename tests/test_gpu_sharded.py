"""GPU parity of the sharded giant filter.

One filter's particles are split by range over S shards; every frame the
shards exchange their max keys and (mass, moment) sums and read remote source
tiles peer-to-peer.  The sharded filter must be BIT-IDENTICAL to the same
filter on one device (which is itself bit-exact against oracle/fused.py):
trajectories in all three precisions, for shard counts that split tiles
unevenly, windows that straddle shard boundaries, and the multi-chunk table.
"""

import os
import socket
import sys

import numpy as np
import pytest

from oracle import fused
from oracle import reference_port as rp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_2308_00763_b200 as pf

    return pf


@pytest.mark.parametrize("mode", ["fp64", "fp32", "fp16"])
@pytest.mark.parametrize("K,S", [(10_000, 2), (10_000, 3), (40_961, 2), (300_007, 3), (2_000_000, 8)])
def test_local_shards_equal_single_device(pf, mode, K, S):
    from paper_2308_00763_b200.sharded import LocalShards

    frames, _ = rp.generate_video(rp.Params(), 8, 96, 80, (40.0, 30.0), 17)
    one = pf.Filter(K, mode, 96, 80, 5, start_hint=(40.0, 30.0)).run(frames)
    sh = LocalShards(K, mode, 96, 80, 5, n_shards=S, start_hint=(40.0, 30.0))
    traj = sh.run(frames)
    sh.close()
    assert np.array_equal(traj, one)


def test_invalid_layout_raises(pf):
    from paper_2308_00763_b200.sharded import LocalShards

    with pytest.raises(ValueError, match="too few tiles"):
        LocalShards(40_961, "fp16", 96, 80, 5, n_shards=4)


def test_local_shards_match_oracle(pf):
    from paper_2308_00763_b200.sharded import LocalShards

    frames, truth = rp.generate_video(rp.Params(), 6, 128, 128, (64.0, 64.0), 42)
    sh = LocalShards(20_000, "fp16", 128, 128, 42, n_shards=3)
    traj = sh.run(frames)
    ref, _ = fused.run(frames, 20_000, "fp16", 42)
    assert np.array_equal(traj, ref)
    assert float(np.mean(np.hypot(*(traj - truth).T))) < 2.0


@pytest.mark.parametrize("mode", ["fp32", "fp16"])
def test_local_shards_multichunk_table(pf, mode):
    # 1,061 tiles over 2 shards: 1024 + 37 tiles, 4 table chunks on shard 0;
    # the single-device run uses the chunked (multi-CTA) table
    from paper_2308_00763_b200.sharded import LocalShards

    K = (1 << 20) + 37 * 1024 - 5
    frames, _ = rp.generate_video(rp.Params(), 5, 128, 128, (64.0, 64.0), 42)
    one = pf.Filter(K, mode, 128, 128, 42).run(frames)
    sh = LocalShards(K, mode, 128, 128, 42, n_shards=2)
    assert sh.shards[0].n_local == 1024 and sh.shards[1].n_local == 37
    traj = sh.run(frames)
    assert np.array_equal(traj, one)


def test_local_shards_reset_and_rerun(pf):
    from paper_2308_00763_b200.sharded import LocalShards

    frames, _ = rp.generate_video(rp.Params(), 4, 64, 64, (32.0, 32.0), 3)
    sh = LocalShards(9000, "fp16", 64, 64, 3, n_shards=2)
    a = sh.run(frames)
    sh.reset()
    b = sh.run(frames)
    assert np.array_equal(a, b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dist_worker(rank, world, port, K, mode, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import reference_port as rp_
    from paper_2308_00763_b200.sharded import DistShard

    frames, _ = rp_.generate_video(rp_.Params(), 6, 96, 80, (40.0, 30.0), 17)
    sh = DistShard(K, mode, 96, 80, 5, start_hint=(40.0, 30.0), device=0, host_staged=True)
    traj = sh.run(frames)
    np.save(os.path.join(out_dir, f"traj{rank}.npy"), traj)
    sh.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["fp16", "fp64"])
def test_two_processes_ipc_peer_reads(pf, mode, tmp_path):
    # two ranks sharing the one GPU: peer buffers through CUDA IPC, the
    # 8 / 32 B exchanges host-staged over gloo (NCCL needs one GPU per rank)
    import torch.multiprocessing as mp

    K = 30_001
    frames, _ = rp.generate_video(rp.Params(), 6, 96, 80, (40.0, 30.0), 17)
    one = pf.Filter(K, mode, 96, 80, 5, start_hint=(40.0, 30.0)).run(frames)
    mp.spawn(_dist_worker, args=(2, _free_port(), K, mode, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"traj{r}.npy"), one)


@pytest.mark.parametrize("mode", ["fp64", "fp16"])
@pytest.mark.parametrize("K", [10_000, 2_000_000])
def test_split_table_equals_chunked(pf, mode, K, monkeypatch):
    # tracks too large for the co-resident chunked table (2^30 on one GPU) run
    # the sharded table kernels with one shard; forced here at small K
    frames, _ = rp.generate_video(rp.Params(), 6, 96, 80, (40.0, 30.0), 17)
    one = pf.Filter(K, mode, 96, 80, 5, start_hint=(40.0, 30.0)).run(frames)
    monkeypatch.setenv("PF_FORCE_SPLIT_TABLE", "1")
    two = pf.Filter(K, mode, 96, 80, 5, start_hint=(40.0, 30.0)).run(frames)
    assert np.array_equal(one, two)


def _n_gpus():
    import torch

    return torch.cuda.device_count()


def _nccl_worker(rank, world, port, K, mode, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import reference_port as rp_
    from paper_2308_00763_b200.sharded import DistShard

    frames, _ = rp_.generate_video(rp_.Params(), 6, 96, 80, (40.0, 30.0), 17)
    sh = DistShard(K, mode, 96, 80, 5, start_hint=(40.0, 30.0), device=rank)  # NCCL all-gathers
    traj = sh.run(frames)
    np.save(os.path.join(out_dir, f"traj{rank}.npy"), traj)
    sh.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif("_n_gpus() < 2")
@pytest.mark.parametrize("mode", ["fp16", "fp64"])
def test_two_gpus_nccl_bit_identical(pf, mode, tmp_path):
    # one shard per GPU: NCCL all-gathers on the library stream, remote
    # ancestors read over CUDA-IPC peer mappings (NVLink) -- must equal the
    # single-device filter bit for bit
    import torch.multiprocessing as mp

    K = 30_001
    frames, _ = rp.generate_video(rp.Params(), 6, 96, 80, (40.0, 30.0), 17)
    one = pf.Filter(K, mode, 96, 80, 5, start_hint=(40.0, 30.0)).run(frames)
    mp.spawn(_nccl_worker, args=(2, _free_port(), K, mode, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"traj{r}.npy"), one)


@pytest.mark.skipif("_n_gpus() < 2")
def test_local_shards_on_distinct_devices(pf):
    # shards on different GPUs in one process: pf_shard_set_peer enables peer
    # access, the fused kernels read remote source tiles directly
    from paper_2308_00763_b200.sharded import LocalShards

    frames, _ = rp.generate_video(rp.Params(), 5, 96, 80, (40.0, 30.0), 17)
    n = min(_n_gpus(), 4)
    one = pf.Filter(50_000, "fp32", 96, 80, 5, start_hint=(40.0, 30.0)).run(frames)
    sh = LocalShards(50_000, "fp32", 96, 80, 5, n_shards=n, start_hint=(40.0, 30.0), devices=list(range(n)))
    assert np.array_equal(sh.run(frames), one)
    sh.close()


def test_set_peer_rejects_host_memory(pf):
    # peer buffers must be device memory (pf_shard_set_peer checks each pointer)
    import ctypes

    from paper_2308_00763_b200.sharded import _Shard

    s = _Shard(10_000, "fp32", 64, 64, 1, 2, 0)
    host = [ctypes.addressof(ctypes.c_char.from_buffer(bytearray(64))) for _ in range(8)]
    with pytest.raises(Exception):
        s.set_peer(1, host)
    s.close()
