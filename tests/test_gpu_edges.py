"""Edge cases of the fused path against the oracle, bit-exact: tiny frames,
degenerate templates, radii larger than the frame, the smallest particle
counts, and several tracks with odd particle counts (unaligned track bases:
the plain-copy staging path instead of the bulk copy)."""

import numpy as np
import pytest

from oracle import fused
from oracle import reference_port as rp

pytestmark = pytest.mark.gpu


def _pf():
    import paper_2308_00763_b200 as pf

    return pf


@pytest.mark.parametrize("mode", ["fp64", "fp32", "fp16-packed"])
@pytest.mark.parametrize("W,H,r", [(1, 1, 5), (2, 7, 1), (64, 48, 20), (33, 17, 1)])
def test_shapes_and_radii(mode, W, H, r):
    pf = _pf()
    p = rp.Params(disk_radius=r)
    if W == 1:  # (the reference video model's bounce loop never ends on a 1-pixel axis)
        frames = np.random.default_rng(1).integers(0, 256, (5, H, W), dtype=np.uint8)
    else:
        frames, _ = rp.generate_video(p, 5, W, H, ((W - 1) / 2.0, (H - 1) / 2.0), 3)
    P = pf.ModelParams(disk_radius=r)
    got = pf.Filter(2000, mode, W, H, 9, params=P).run(frames)
    ref, _ = fused.run(frames, 2000, mode, 9, params=p, offsets=rp.disk_offsets(r))
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("mode", ["fp64", "fp16"])
@pytest.mark.parametrize("K", [2, 3, 1023, 1024, 1025, 2047])
def test_multitrack_odd_counts(mode, K):
    pf = _pf()
    frames, _ = rp.generate_video(rp.Params(), 4, 80, 60, (40.0, 30.0), 5)
    seeds = [11, 12, 13]
    f = pf.Filter(K, mode, 80, 60, seeds=seeds, n_tracks=3)
    batch = f.run(frames)
    for i, sd in enumerate(seeds):
        ref, _ = fused.run(frames, K, mode, sd)
        assert np.array_equal(batch[i], ref), (i, K)


def test_asymmetric_template_fused():
    pf = _pf()
    offs = np.array([[0, 0], [3, -2], [-1, 4], [2, 2], [-4, -1], [1, 0]], dtype=np.int64)
    frames, _ = rp.generate_video(rp.Params(), 5, 64, 64, (32.0, 32.0), 2)
    for mode in ("fp64", "fp16-packed"):
        got = pf.Filter(5000, mode, 64, 64, 4, template=pf.PixelTemplate(offs)).run(frames)
        ref, _ = fused.run(frames, 5000, mode, 4, offsets=offs)
        assert np.array_equal(got, ref), mode


@pytest.mark.parametrize("mode", ["fp16-packed", "fp64"])
@pytest.mark.parametrize("W,F", [(512, 43), (384, 100)])
def test_chunked_host_upload_equals_device_frames(mode, W, F):
    # host frames of >= 8 MB are uploaded in chunks on a copy stream with each
    # chunk's maps started as it lands: same trajectory as device-resident frames
    import torch

    import paper_2308_00763_b200 as pf

    frames, _ = rp.generate_video(rp.Params(), F, W, W, (W / 2.0, W / 2.0), 42)
    assert frames.nbytes >= 8 << 20
    f = pf.Filter(20_000, mode, W, W, 42)
    dev = f.run_frames(torch.from_numpy(frames).cuda(), F)
    f.reset()
    host = f.run_frames(frames, F)
    f.reset()
    pinned = f.run_frames(torch.from_numpy(frames).pin_memory().numpy(), F)
    f.close()
    assert np.array_equal(dev, host) and np.array_equal(dev, pinned)
