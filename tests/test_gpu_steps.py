"""Per-frame API (filter.py:617-654 frame loop, one call per frame): Filter.step
and the stream-ordered pf_step_async run as one graph launch per frame with
updated kernel-node arguments -- results must equal the whole-video run."""

import ctypes as C

import numpy as np
import pytest

from oracle import reference_port as rp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_2308_00763_b200 as pf

    return pf


@pytest.fixture(scope="module")
def video():
    return rp.generate_video(rp.Params(), 12, 128, 128, (64.0, 64.0), 42)


@pytest.mark.parametrize("mode", ["fp64", "fp32", "fp16", "fp16-packed"])
def test_steps_equal_run(pf, video, mode):
    import torch

    frames, _ = video
    F, K = frames.shape[0], 30_000
    f = pf.Filter(K, mode, 128, 128, 42)
    ref = f.run(frames)
    for src in (frames, torch.from_numpy(frames).cuda()):
        f.reset()
        steps = np.array([f.step(src[t]) for t in range(F)])
        assert np.array_equal(steps, ref), mode
    # steps continue a run (and a run continues steps): same trajectory
    f.reset()
    head = f.run(frames[:5])
    tail = np.array([f.step(frames[t]) for t in range(5, F)])
    assert np.array_equal(np.concatenate([head, tail]), ref)
    f.close()


def test_async_steps_pipelined(pf, video):
    import torch

    from paper_2308_00763_b200 import _native as N

    frames, _ = video
    F, K = frames.shape[0], 50_000
    f = pf.Filter(K, "fp16-packed", 128, 128, 7)
    ref = f.run(frames)
    f.reset()
    dev = torch.from_numpy(frames).cuda()
    outs = torch.empty((F, 2), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for t in range(F):  # enqueued back to back, one synchronisation
        assert N.lib().pf_step_async(f._h, C.c_void_p(dev[t].data_ptr()), 1, C.c_void_p(outs[t].data_ptr()),
                                     C.c_void_p(s)) == 0
    assert N.lib().pf_sync(f._h) == 0
    assert np.array_equal(outs.cpu().numpy(), ref)
    f.close()


def test_steps_on_reference_stream_and_tracks(pf, video):
    frames, _ = video
    f = pf.Filter(20_000, "fp64", 128, 128, 3, rng="numpy-philox")
    ref = f.run(frames)
    f.reset()
    assert np.array_equal(np.array([f.step(frames[t]) for t in range(frames.shape[0])]), ref)
    f.close()
    vids = np.stack([frames, frames[::-1].copy()])
    g = pf.Filter(8192, "fp32", 128, 128, n_tracks=3, n_videos=2)
    ref3 = g.run_frames(vids)
    g.reset()
    steps = np.stack([g.step(vids[:, t]) for t in range(frames.shape[0])], axis=1)
    assert np.array_equal(steps, ref3)
    g.close()


@pytest.mark.parametrize("mode", ["fp64", "fp32"])
def test_fused_degeneracy_reported(pf, video, mode):
    """A degenerate frame (here: NaN positions injected with set_state, so the
    weighted estimate is not finite) raises DegeneracyError with that frame's
    index -- through a whole run and through per-frame steps (the tile table
    reports it through host-mapped memory for synchronous calls), and the
    handle recovers after reset().  (Binary16 modes keep exact integer
    moments of rint(x * 2^10): a NaN position converts to 0 there, and every
    tile's maximum weight is 2^20 > 0, so the stabilised filter cannot
    degenerate.)"""
    frames, _ = video
    K = 4096
    f = pf.Filter(K, mode, 128, 128, 42)
    nan = np.full(K, np.nan)
    f.set_state(nan, nan, 3)
    with pytest.raises(pf.DegeneracyError) as info:
        f.run(frames[3:8])
    assert info.value.frame == 3
    f.set_state(nan, nan, 5)
    with pytest.raises(pf.DegeneracyError) as info:
        f.step(frames[5])
    assert info.value.frame == 5
    f.reset()
    ref = pf.Filter(K, mode, 128, 128, 42).run(frames)
    assert np.array_equal(f.run(frames), ref)
    f.close()
