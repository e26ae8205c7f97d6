"""GPU parity of the fused path (the product hot path) through the C ABI.

* bit-exact against oracle/fused.py (the CPU restatement of the same
  algorithm) in all three precisions;
* FP64 / FP32 within 1e-9 / 1e-4 relative of the REFERENCE trajectory with
  the same draws (goldens from the real halfpf run);
* FP16 stabilised within the reference FP16 error bound;
* results independent of threads-per-block and of batching tracks together.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import fused
from oracle import reference_port as rp
from oracle import rng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_2308_00763_b200 as pf

    return pf


def _err(traj, truth):
    return float(np.mean(np.hypot(*(traj - truth).T)))


def test_device_rng_matches_oracle(pf):
    from paper_2308_00763_b200 import _native as N

    for seed in (0, 42, 2**63 + 5):
        for pos, n in ((0, 20_000), (10**9 + 7, 5000), (2**40 + 3, 3000)):
            out = np.empty(n, dtype=np.float64)
            assert N.lib().pf_rng_normals(seed, pos, n, N.ptr(out), 0) == 0
            ref = rng.normals_from_lcg_words(rng.lcg_words(rng.lcg_seed_state(seed), pos, n))
            assert np.array_equal(out, ref), (seed, pos)
            uo = np.empty(64, dtype=np.float64)
            assert N.lib().pf_rng_uniforms(seed, pos, 64, N.ptr(uo), 0) == 0
            w = rng.lcg_words(rng.lcg_seed_state(seed), pos, 64)
            assert np.array_equal(uo, (w >> np.uint64(11)).astype(np.float64) * rng.TWO_M53)


def test_exp16_fast_path_equals_table_exhaustively(pf):
    # the fused FP16 kernel's exp16 (ex2.approx + midpoint guard + table
    # fallback) must equal RN16(exp(d)) for every binary16 d <= 0
    from paper_2308_00763_b200 import _native as N

    dev = np.empty(65536, dtype=np.uint16)
    tab = np.empty(65536, dtype=np.uint16)
    assert N.lib().pf_exp16_device(N.ptr(dev), 0) == 0
    assert N.lib().pf_exp16_table(N.ptr(tab)) == 0
    x = np.arange(65536, dtype=np.uint32).astype(np.uint16).view(np.float16).astype(np.float32)
    sel = (x <= 0) & ~np.isnan(x)
    assert np.array_equal(dev[sel], tab[sel])


def test_device_rng_stream_class(pf):
    g = golden("lcg_stream.npz")
    s = pf.RngStream(42)
    assert np.array_equal(s.normals(4096), g["n_42"])
    assert np.array_equal(np.array([s.uniform() for _ in range(8)]), g["u_42"])


@pytest.mark.parametrize("mode", ["fp64", "fp32", "fp16", "fp16-packed"])
def test_fused_bitexact_vs_oracle_acceptance(pf, acceptance_video, mode):
    frames, truth = acceptance_video
    f = pf.Filter(128, mode, 128, 128, 42, start_hint=(64.0, 64.0))
    traj = f.run(frames)
    ref, tr = fused.run(frames, 128, mode, 42, start_hint=(64.0, 64.0))
    assert np.array_equal(traj, ref)
    xs, ys, c = f.state()
    assert np.array_equal(xs, tr.xs) and np.array_equal(ys, tr.ys)
    assert np.array_equal(c.view(np.uint8), tr.c.view(np.uint8))


@pytest.mark.parametrize("mode", ["fp64", "fp32", "fp16", "fp16-packed"])
@pytest.mark.parametrize("K", [2, 1023, 1025, 10_000, 40_961, 200_003])
def test_fused_bitexact_vs_oracle_sizes(pf, mode, K):
    if mode == "fp16-packed" and K % 2:
        pytest.skip("packed binary16 needs an even particle count (filter.py:137-143)")
    frames, _ = rp.generate_video(rp.Params(), 6, 96, 80, (40.0, 30.0), 17)
    traj = pf.Filter(K, mode, 96, 80, 5, start_hint=(40.0, 30.0)).run(frames)
    ref, _ = fused.run(frames, K, mode, 5, start_hint=(40.0, 30.0))
    assert np.array_equal(traj, ref)


def test_fused_bitexact_odd_params(pf):
    g = golden("odd_params.npz")
    P = pf.ModelParams(bg_mean=100.3, fg_mean=227.7, likelihood_scale=47.1, drift_x=0.7, std_x=4.3, disk_radius=4)
    PP = rp.Params(bg_mean=100.3, fg_mean=227.7, likelihood_scale=47.1, drift_x=0.7, std_x=4.3, disk_radius=4)
    for mode in ("fp64", "fp32", "fp16"):
        traj = pf.Filter(301, mode, 96, 80, 9, params=P).run(g["frames"])
        ref, _ = fused.run(g["frames"], 301, mode, 9, params=PP, offsets=rp.disk_offsets(4))
        assert np.array_equal(traj, ref), mode


@pytest.mark.parametrize("mode,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_fused_vs_reference_trajectory(pf, acceptance_video, c1_video, mode, tol):
    frames, _ = acceptance_video
    traj = pf.Filter(128, mode, 128, 128, 42, start_hint=(64.0, 64.0)).run(frames)
    ref = golden("acceptance_k128.npz")[f"{mode}_traj"]
    assert np.max(np.abs(traj - ref) / np.abs(ref)) <= tol
    frames1, _ = c1_video
    traj1 = pf.Filter(10_000, mode, 128, 128, 42).run(frames1)
    ref1 = golden("c1_k10000.npz")[f"{mode}_traj"]
    assert np.max(np.abs(traj1 - ref1) / np.abs(ref1)) <= tol


def test_fp16_within_reference_error_bound(pf, acceptance_video):
    frames, truth = acceptance_video
    e16 = _err(pf.Filter(128, "fp16", 128, 128, 42, start_hint=(64.0, 64.0)).run(frames), truth)
    e64 = _err(golden("acceptance_k128.npz")["fp64_traj"], truth)
    assert e16 <= 2.0 * e64 and e16 <= 2.0 * 1.255495438119523


@pytest.mark.parametrize("mode", ["fp64", "fp32", "fp16"])
def test_tpb_independence(pf, mode):
    frames, _ = rp.generate_video(rp.Params(), 5, 128, 128, (64.0, 64.0), 3)
    base = pf.Filter(5000, mode, 128, 128, 1, tpb=256).run(frames)
    for tpb in (32, 64, 128, 512, 1024):
        assert np.array_equal(pf.Filter(5000, mode, 128, 128, 1, tpb=tpb).run(frames), base), tpb


def test_batched_tracks_equal_independent_runs(pf):
    frames, _ = rp.generate_video(rp.Params(), 4, 64, 64, (32.0, 32.0), 8)
    frames2, _ = rp.generate_video(rp.Params(), 4, 64, 64, (20.0, 40.0), 9)
    vids = np.stack([frames, frames2])
    seeds = [3, 4, 5]
    b = pf.Filter(3000, "fp16", 64, 64, seeds=seeds, n_tracks=3, n_videos=2, start_hint=(30.0, 30.0))
    traj = b.run_frames(vids, 4)
    for i, s in enumerate(seeds):
        single = pf.Filter(3000, "fp16", 64, 64, s, start_hint=(30.0, 30.0)).run(vids[i % 2])
        assert np.array_equal(traj[i], single), i


def test_step_equals_run(pf):
    frames, _ = rp.generate_video(rp.Params(), 5, 64, 64, (32.0, 32.0), 2)
    whole = pf.Filter(2048, "fp32", 64, 64, 7).run(frames)
    f = pf.Filter(2048, "fp32", 64, 64, 7)
    steps = np.array([f.step(frames[t]) for t in range(5)])
    assert np.array_equal(whole, steps)


def test_ancestors_and_loglik_match_oracle(pf):
    frames, _ = rp.generate_video(rp.Params(), 3, 64, 64, (32.0, 32.0), 6)
    f = pf.Filter(3000, "fp64", 64, 64, 11)
    f.enable_debug()
    tr = fused.FusedTrack("fp64", 3000, 64, 64, 11, (32.0, 32.0))
    for t in range(3):
        f.step(frames[t])
        tr.step(tr.loglik_map(frames[t]))
        anc, L = f.debug()
        assert np.array_equal(anc, tr.last_ancestors), t
        assert np.array_equal(L, tr.last_loglik), t


def test_run_api_fused(pf, acceptance_video):
    frames, truth = acceptance_video
    video = pf.Video(frames=frames, truth=truth)
    res = pf.run(video, 128, pf.PrecisionMode.FP64, 42, start_hint=(64.0, 64.0))
    ref, _ = fused.run(frames, 128, "fp64", 42, start_hint=(64.0, 64.0))
    assert np.array_equal(res.trajectory, ref)
    assert set(res.stage_ms) == set(pf.STAGES)
    assert res.launches == 1 + 2 * 100


@pytest.mark.parametrize("tpb", [32, 128, 256, 1024])
def test_fp16_scalar_and_packed_kernels_identical(pf, tpb):
    """The naive-vs-optimised pair: "fp16" runs the scalar-lane
    kernels (one RN16 op per lane), "fp16-packed" the half2 kernels; values are
    identical (reference test_acceptance.py:233-248), only the pipes differ."""
    frames, _ = rp.generate_video(rp.Params(), 8, 128, 96, (64.0, 48.0), 21)
    a = pf.Filter(50_000, "fp16", 128, 96, 3, tpb=tpb)
    b = pf.Filter(50_000, "fp16-packed", 128, 96, 3, tpb=tpb)
    assert np.array_equal(a.run(frames), b.run(frames))
    assert np.array_equal(a.state()[2].view(np.uint16), b.state()[2].view(np.uint16))
    assert np.array_equal(a.likelihood_maps(frames[:2]).view(np.uint16), b.likelihood_maps(frames[:2]).view(np.uint16))


def test_c4_scale_batch_creates_and_steps(pf):
    # 8192 tracks x 64K particles (C4 on one GPU): one table CTA per track, no
    # cross-CTA co-residency requirement -- creation must not refuse it
    frames, _ = rp.generate_video(rp.Params(), 2, 128, 128, (64.0, 64.0), 42)
    f = pf.Filter(65536, "fp16-packed", 128, 128, seeds=list(range(8192)), n_tracks=8192)
    traj = f.run(frames)
    assert traj.shape == (8192, 2, 2) and np.isfinite(traj).all()
    f.close()


@pytest.mark.parametrize("mode", ["fp16", "fp16-packed", "fp32"])
def test_saturated_frame_stays_finite(pf, mode):
    # reference test_model.py:169-190: on an all-255 frame the direct FP16
    # likelihood overflows; the stabilised (log-domain, max-shifted) path stays
    # finite and never degenerates
    frames = np.full((5, 64, 64), 255, dtype=np.uint8)
    traj = pf.Filter(20_000, mode, 64, 64, 3).run(frames)
    assert np.isfinite(traj).all()
    L = pf.Filter(64, mode, 64, 64, 3).likelihood_maps(frames[:1])
    assert np.isfinite(np.asarray(L, dtype=np.float64)).all()
