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


@pytest.fixture(scope="module")
def pf():
    return _pf()


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


def test_frame_validation(pf):
    import torch

    f = pf.Filter(2048, "fp32", 64, 48, 1)
    good = np.zeros((3, 48, 64), dtype=np.uint8)
    f.run(good)
    for bad in (np.zeros((3, 64, 48), np.uint8), np.zeros((3, 48, 63), np.uint8), np.zeros((48, 64), np.uint8),
                np.zeros((2, 3, 48, 64), np.uint8), np.zeros((0, 48, 64), np.uint8)):
        with pytest.raises(ValueError):
            f.run(bad)
    with pytest.raises(ValueError):
        f.run(good.astype(np.float32))
    with pytest.raises(ValueError):
        f.step(np.zeros((48, 65), np.uint8))
    t = torch.zeros((3, 48, 128), dtype=torch.uint8, device="cuda")[:, :, ::2]
    with pytest.raises(ValueError):  # non-contiguous
        f.run(t)
    with pytest.raises(ValueError):
        f.run(torch.zeros((3, 48, 64), dtype=torch.int16, device="cuda"))
    assert f.step(np.zeros((48, 64), np.uint8)) is not None
    f.close()


def test_stream_ordered_run(pf):
    # frames produced by torch work still in flight on a side stream: the
    # stream-ordered call waits for them; the trajectory lands on the device
    import torch

    F, K = 6, 20_000
    frames, _ = rp.generate_video(rp.Params(), F, 128, 128, (64.0, 64.0), 42)
    ref = pf.Filter(K, "fp16-packed", 128, 128, 42).run(frames)
    f = pf.Filter(K, "fp16-packed", 128, 128, 42)
    side = torch.cuda.Stream()
    src = torch.from_numpy(frames).pin_memory()
    with torch.cuda.stream(side):
        torch.cuda._sleep(20_000_000)  # keep the side stream busy before the copy lands
        dev = src.to("cuda", non_blocking=True)
        traj = torch.empty((1, F, 2), dtype=torch.float64, device="cuda")
        f.run_async(dev, traj)
        out = traj.cpu()  # ordered after the run on the same stream
    f.sync()
    assert np.array_equal(out.numpy()[0], ref)
    # the blocking API with device frames orders itself after torch's current stream
    with torch.cuda.stream(side):
        torch.cuda._sleep(20_000_000)
        dev2 = src.to("cuda", non_blocking=True)
        f.reset()
        assert np.array_equal(f.run(dev2), ref)
    f.close()
