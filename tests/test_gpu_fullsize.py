"""Full-size checks (BASELINE.json configs) through size-independent
properties -- the oracle cannot run 10^6..10^9 particles, so at these sizes
the device path is held to invariants that the bit-exact small-size tests
(test_gpu_fused.py) make meaningful:

* determinism: the same run twice is bit-identical;
* threads-per-block independence: 128 vs 256 threads give bit-identical
  trajectories and states (the fused algorithm's exact, canonical reductions);
* batching independence (C4): a track's trajectory is the same alone and
  inside an 8192-track batch;
* sharding independence (C5 layout): the particle-range-sharded filter equals
  the single-device filter bit-for-bit;
* the local CDF of every tile is non-decreasing, within [0, 1] and ends at
  exactly 1 (the rescaled-CDF invariant);
* tracking accuracy against the ground-truth trajectory.
"""

import numpy as np
import pytest

from oracle import reference_port as rp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_2308_00763_b200 as pf

    return pf


def _cdf_invariants(c, K):
    c = np.asarray(c, dtype=np.float64)
    n = -(-K // 1024)
    for b in range(n):
        t = c[b * 1024: min(K, (b + 1) * 1024)]
        assert np.all(np.diff(t) >= 0.0), b
        assert t.min() >= 0.0 and t.max() == 1.0, b
        assert t[-1] == 1.0, b


def test_c2_full_size(pf):
    frames, truth = rp.generate_video(rp.Params(), 100, 128, 128, (64.0, 64.0), 42)
    out = {}
    for tpb in (128, 256):
        f = pf.Filter(1_000_000, "fp16-packed", 128, 128, 42, tpb=tpb)
        a = f.run(frames)
        f.reset()
        b = f.run(frames)
        assert np.array_equal(a, b)  # deterministic
        out[tpb] = (a, f.state())
        f.close()
    assert np.array_equal(out[128][0], out[256][0])
    for i in range(3):
        assert np.array_equal(out[128][1][i].view(np.uint16), out[256][1][i].view(np.uint16))
    _cdf_invariants(out[128][1][2], 1_000_000)
    assert np.mean(np.hypot(*(out[128][0] - truth).T)) < 0.3


@pytest.mark.parametrize("mode", ["fp16-packed", "fp32"])
def test_c3_full_size(pf, mode):
    import torch

    F = 25
    frames, truth = rp.generate_video(rp.Params(), F, 1024, 1024, (512.0, 512.0), 42)
    dev = torch.from_numpy(frames).cuda()
    trajs = []
    for tpb in (256, 128):
        f = pf.Filter(1 << 24, mode, 1024, 1024, 42, tpb=tpb)
        trajs.append(f.run_frames(dev, F)[0])
        if tpb == 256:
            _cdf_invariants(f.state()[2], 1 << 24)
        f.close()
    assert np.array_equal(trajs[0], trajs[1])
    assert np.mean(np.hypot(*(trajs[0] - truth).T)) < 0.05


def test_c4_batch_equals_single_tracks(pf):
    vids = [rp.generate_video(rp.Params(), 20, 128, 128, (64.0, 64.0), 42 + j)[0] for j in range(8)]
    frames = np.ascontiguousarray(np.stack(vids))
    seeds = [42 + i for i in range(8192)]
    f = pf.Filter(65536, "fp16-packed", 128, 128, seeds=seeds, n_tracks=8192, n_videos=8)
    batch = f.run_frames(frames, 20)
    f.close()
    for i in (0, 5, 4097, 8191):
        g = pf.Filter(65536, "fp16-packed", 128, 128, seed=42 + i)
        single = g.run(vids[i % 8])
        g.close()
        assert np.array_equal(batch[i], single), i


def test_c5_layout_sharded_equals_single(pf):
    # C5's layout at 2^28 particles (one B200 holds both): 2 shards of 2^27
    from paper_2308_00763_b200.sharded import LocalShards

    frames, truth = rp.generate_video(rp.Params(), 4, 1024, 1024, (512.0, 512.0), 42)
    K = 1 << 28
    one = pf.Filter(K, "fp16-packed", 1024, 1024, 42)
    a = one.run(frames)
    one.close()
    sh = LocalShards(K, "fp16-packed", 1024, 1024, 42, n_shards=2)
    assert sh.shards[0].K_local == 1 << 27
    b = sh.run(frames)
    sh.close()
    assert np.array_equal(a, b)
    assert np.mean(np.hypot(*(a - truth).T)) < 0.05
