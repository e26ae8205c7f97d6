"""Device NumPy-compatible stream (PhiloxRngStream) and the staged engine on the
reference's OWN draws: the unmodified reference configuration end to end."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_2308_00763_b200 as pf

    return pf


@pytest.mark.parametrize("seed", [42, 7, 123456789])
def test_device_philox_stream_equals_numpy(pf, seed):
    dev = pf.PhiloxRngStream(seed)
    ref = np.random.Generator(np.random.Philox(seed))
    for n in (128, 10_000, 250_000, 3):
        assert np.array_equal(dev.normals(n), ref.standard_normal((n, 2)))
        assert dev.uniform() == float(ref.random())


@pytest.mark.parametrize("mode", ["fp16", "fp16-packed"])
def test_staged_reference_stream_binary16_bit_exact(pf, acceptance_video, monkeypatch, mode):
    import paper_2308_00763_b200.filter as F

    monkeypatch.setattr(F, "RngStream", pf.PhiloxRngStream)
    frames, truth = acceptance_video
    res = pf.run(pf.Video(frames, truth), 128, mode, 42, start_hint=(64.0, 64.0), engine="staged")
    assert np.array_equal(res.trajectory, golden("acceptance_k128.npz")[f"philox_{mode}_traj"])


@pytest.mark.parametrize("mode,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_staged_reference_stream_wide(pf, acceptance_video, c1_video, monkeypatch, mode, tol):
    import paper_2308_00763_b200.filter as F

    monkeypatch.setattr(F, "RngStream", pf.PhiloxRngStream)
    frames, truth = acceptance_video
    res = pf.run(pf.Video(frames, truth), 128, mode, 42, start_hint=(64.0, 64.0), engine="staged")
    ref = golden("acceptance_k128.npz")[f"philox_{mode}_traj"]
    assert np.max(np.abs(res.trajectory - ref) / np.abs(ref)) <= tol
    if mode == "fp64":  # test_acceptance.py:40
        err = float(np.mean(np.hypot(*(res.trajectory - truth).T)))
        assert err == pytest.approx(1.255495438119523, rel=1e-12)
    f1, t1 = c1_video
    r1 = pf.run(pf.Video(f1, t1), 10_000, mode, 42, engine="staged")
    ref1 = golden("c1_k10000.npz")[f"philox_{mode}_traj"]
    assert np.max(np.abs(r1.trajectory - ref1) / np.abs(ref1)) <= tol


# ---- the fused product path on the reference's own stream ----


@pytest.mark.parametrize("mode,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_fused_on_reference_stream(pf, acceptance_video, c1_video, mode, tol):
    # the unmodified reference configuration (Generator(Philox(42))) through
    # the fused kernels: trajectories of the real halfpf run within tolerance
    frames, truth = acceptance_video
    res = pf.run(pf.Video(frames, truth), 128, mode, 42, start_hint=(64.0, 64.0), rng="numpy-philox")
    assert res.launches > 0
    ref = golden("acceptance_k128.npz")[f"philox_{mode}_traj"]
    assert np.max(np.abs(res.trajectory - ref) / np.abs(ref)) <= tol
    if mode == "fp64":  # test_acceptance.py:40 FP64_MEAN_ERR
        err = float(np.mean(np.hypot(*(res.trajectory - truth).T)))
        assert err == pytest.approx(1.255495438119523, rel=1e-9)
    f1, t1 = c1_video
    r1 = pf.run(pf.Video(f1, t1), 10_000, mode, 42, rng="numpy-philox")
    ref1 = golden("c1_k10000.npz")[f"philox_{mode}_traj"]
    assert np.max(np.abs(r1.trajectory - ref1) / np.abs(ref1)) <= tol


@pytest.mark.parametrize("mode", ["fp16", "fp16-packed"])
def test_fused_fp16_on_reference_stream_within_bound(pf, acceptance_video, mode):
    frames, truth = acceptance_video
    traj = pf.Filter(128, mode, 128, 128, 42, start_hint=(64.0, 64.0), rng="numpy-philox").run(frames)
    err = float(np.mean(np.hypot(*(traj - truth).T)))
    assert err <= 2.0 * 1.255495438119523  # test_acceptance.py:144-146


@pytest.mark.parametrize("mode", ["fp64", "fp32", "fp16-packed"])
def test_fused_philox_bit_exact_vs_oracle(pf, mode):
    # the fused oracle fed NumPy's own draws == the device (parallel stream +
    # buffered-noise kernel), across several frames and an odd tile count
    from oracle import fused
    from oracle import reference_port as rp

    K = 40_962
    frames, _ = rp.generate_video(rp.Params(), 5, 96, 80, (48.0, 40.0), 5)
    f = pf.Filter(K, mode, 96, 80, 9, rng="numpy-philox")
    traj = f.run(frames)
    g = np.random.Generator(np.random.Philox(9))
    tr = fused.FusedTrack(mode, K, 96, 80, 9, (48.0, 40.0))
    ref = []
    for t in range(5):
        noise = g.standard_normal((K, 2))
        ref.append(tr.step(tr.loglik_map(frames[t]), noise, float(g.random())))
    assert np.array_equal(traj, np.array(ref))
    # reset rewinds the stream; per-frame steps continue it
    f.reset()
    steps = np.array([f.step(frames[t]) for t in range(5)])
    assert np.array_equal(steps, traj)
    f.close()


def test_parallel_stream_long_and_throughput(pf):
    import ctypes

    import torch

    from paper_2308_00763_b200 import _native as N

    seed = 2024
    dev = pf.PhiloxRngStream(seed)
    ref = np.random.Generator(np.random.Philox(seed))
    n = 1 << 22  # 4M normals (C2's 2K normals per frame is 2M)
    assert np.array_equal(dev.normals(n // 2).reshape(-1), ref.standard_normal(n))
    assert dev.uniform() == float(ref.random())
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(2):  # warm
        assert N.lib().pf_philox_normals_device(dev._h, n, ctypes.c_void_p(out.data_ptr()),
                                                ctypes.c_void_p(s.cuda_stream)) == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    reps = 5
    for _ in range(reps):
        N.lib().pf_philox_normals_device(dev._h, n, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s.cuda_stream))
    e1.record(s)
    e1.synchronize()
    rate = reps * n / (e0.elapsed_time(e1) * 1e-3)
    assert rate > 1e9, rate  # verdict bar: > 1e9 normals/s
    # and the values continued the stream exactly
    for _ in range(2 + reps - 1):
        ref.standard_normal(n)
    assert np.array_equal(out.cpu().numpy(), ref.standard_normal(n))
