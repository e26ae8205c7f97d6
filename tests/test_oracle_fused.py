"""The fused tile algorithm (oracle/fused.py) against the reference semantics.

This pins the product's algorithm on CPU: FP64/FP32 trajectories within the
north-star tolerances (1e-9 / 1e-4 relative) of the reference run with the
same draws, FP16 stabilised within the reference FP16 error bound."""

import numpy as np
import pytest

from conftest import golden
from oracle import fused, rng
from oracle import reference_port as rp


def _err(traj, truth):
    return float(np.mean(np.hypot(*(traj - truth).T)))


@pytest.mark.parametrize("mode,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_acceptance_within_tolerance(acceptance_video, mode, tol):
    frames, truth = acceptance_video
    g = golden("acceptance_k128.npz")
    traj, _ = fused.run(frames, 128, mode, 42, start_hint=(64.0, 64.0))
    ref = g[f"{mode}_traj"]
    assert np.max(np.abs(traj - ref) / np.abs(ref)) <= tol


@pytest.mark.parametrize("mode,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_c1_within_tolerance(c1_video, mode, tol):
    frames, _ = c1_video
    g = golden("c1_k10000.npz")
    traj, _ = fused.run(frames, 10_000, mode, 42)
    ref = g[f"{mode}_traj"]
    assert np.max(np.abs(traj - ref) / np.abs(ref)) <= tol


def test_fp16_error_bound(acceptance_video):
    # test_acceptance.py:144-146: FP16 mean err <= 2 x FP64 mean err (same draws),
    # and the reference's absolute bound 2 x 1.255495438119523
    frames, truth = acceptance_video
    g = golden("acceptance_k128.npz")
    t16, _ = fused.run(frames, 128, "fp16", 42, start_hint=(64.0, 64.0))
    e16 = _err(t16, truth)
    e64 = _err(g["fp64_traj"], truth)
    assert e16 <= 2.0 * e64
    assert e16 <= 2.0 * 1.255495438119523


def test_fp32_pixel_rounded_equals_fp64(acceptance_video):
    # test_acceptance.py:140 analogue on the fused path
    frames, _ = acceptance_video
    a, _ = fused.run(frames, 128, "fp64", 42, start_hint=(64.0, 64.0))
    b, _ = fused.run(frames, 128, "fp32", 42, start_hint=(64.0, 64.0))
    assert np.array_equal(np.rint(a), np.rint(b))


def test_odd_params_within_tolerance():
    g = golden("odd_params.npz")
    P = rp.Params(bg_mean=100.3, fg_mean=227.7, likelihood_scale=47.1, drift_x=0.7, std_x=4.3, disk_radius=4)
    for mode, tol in (("fp64", 1e-9), ("fp32", 1e-4)):
        traj, _ = fused.run(g["frames"], 301, mode, 9, params=P, offsets=rp.disk_offsets(4))
        assert np.max(np.abs(traj - g[f"{mode}_traj"]) / np.abs(g[f"{mode}_traj"])) <= tol, mode


def test_tile_structures():
    """Local CDF ends at exactly 1, is monotone; tile table offsets are exact."""
    frames, truth = rp.generate_video(rp.Params(), 3, 64, 64, (32.0, 32.0), 1)
    for mode in ("fp64", "fp32", "fp16"):
        tr = fused.FusedTrack(mode, 5000, 64, 64, 7, (32.0, 32.0))
        for t in range(3):
            tr.step(tr.loglik_map(frames[t]))
            c = tr.c.astype(np.float64)
            for b in range(tr.n):
                cb = c[b * fused.TILE:(b + 1) * fused.TILE]
                assert np.all(np.diff(cb) >= 0)
                assert cb[-1] == 1.0
            s, O, invM = tr.table
            assert s[0] == 0 and np.all(np.diff(s) >= 0) and s[-1] <= 5000
            if mode == "fp16":  # (phi_b, rho_b): tile-local coordinate offsets / scales
                assert np.all(invM >= 0) and np.all(np.abs(O) <= 2.0)
            else:
                assert O[0] == 0.0 and np.all(np.diff(O) >= 0)


def test_ancestors_match_flat_systematic_resampling():
    """Given the same normalised CDF, the hierarchical search returns exactly
    the flat reference ancestors (filter.py:248-255) -- exercised by building
    the flat CDF from the tile table."""
    frames, _ = rp.generate_video(rp.Params(), 2, 64, 64, (32.0, 32.0), 4)
    tr = fused.FusedTrack("fp64", 3000, 64, 64, 2, (32.0, 32.0))
    tr.step(tr.loglik_map(frames[0]))
    s, O, invM = tr.table
    M = np.where(invM > 0, 1.0 / np.where(invM > 0, invM, 1.0), 0.0)
    flat = np.concatenate([O[b] + M[b] * tr.c[b * fused.TILE:(b + 1) * fused.TILE] for b in range(tr.n)])
    tr.u = 0.3141592653589793
    anc = tr.ancestors()
    pts = fused.points("fp64", 3000, tr.u)
    ref = np.minimum(np.searchsorted(flat, pts, side="left"), 2999)
    # identical except where a point falls within rounding of a boundary
    assert np.mean(anc == ref) > 0.999
    bad = np.nonzero(anc != ref)[0]
    for k in bad:  # every disagreement: the point sits on a CDF step (to rounding)
        lo, hi = sorted((anc[k], ref[k]))
        assert np.all(np.abs(flat[lo:hi] - pts[k]) <= 1e-12 * max(1.0, pts[k])), k


@pytest.mark.parametrize("mode", ["fp64", "fp32"])
def test_ancestors_given_identical_weights_at_scale(mode):
    # the reference's resampling (filter.py:248-255: flat CDF = cumsum of the
    # normalised weights, searchsorted-left of (k+u)/K) vs the fused
    # hierarchical search on the SAME weights (the fused frame's exact tile
    # weights): equal except at points within rounding of a CDF step
    K = 200_000
    frames, _ = rp.generate_video(rp.Params(), 3, 128, 128, (64.0, 64.0), 4)
    tr = fused.FusedTrack(mode, K, 128, 128, 2, (64.0, 64.0))
    tr.step(tr.loglik_map(frames[0]))
    tr.step(tr.loglik_map(frames[1]))
    s, O, invM = tr.table
    M = np.where(invM > 0, 1.0 / np.where(invM > 0, invM, 1.0), 0.0)
    flat = np.concatenate([O[b] + M[b] * tr.c[b * fused.TILE:(b + 1) * fused.TILE].astype(np.float64)
                           for b in range(tr.n)])
    pts = fused.points(mode, K, tr.u)
    anc = tr.ancestors()
    ref = np.minimum(np.searchsorted(flat, pts, side="left"), K - 1)
    bad = np.nonzero(anc != ref)[0]
    assert len(bad) <= K * 1e-3
    tol = 1e-12 if mode == "fp64" else 2e-7
    for k in bad:
        lo, hi = sorted((anc[k], ref[k]))
        assert np.all(np.abs(flat[lo:hi] - pts[k]) <= tol), (k, anc[k], ref[k])
    # the reference's own flat CDF from the same normalised weights: w_hat_k =
    # w_q,k * (mass_b / S_b) / sum(mass); cdf = cumsum(w_hat) (sequential, f64)
    S_b = np.add.reduceat(np.concatenate([tr.last_wq, np.zeros(tr.n * fused.TILE - K, np.int64)]),
                          np.arange(0, tr.n * fused.TILE, fused.TILE))
    scale = np.where(S_b > 0, tr.last_mass / np.where(S_b > 0, S_b, 1), 0.0) / float(tr.last_mass.sum())
    w_hat = tr.last_wq * np.repeat(scale, fused.TILE)[:K]
    cdf = np.cumsum(w_hat)
    ref2 = np.minimum(np.searchsorted(cdf, pts, side="left"), K - 1)
    # bit-exact here: no point falls within the cumsum's rounding of a step
    assert np.array_equal(anc, ref2), int(np.sum(anc != ref2))


def test_oracle_set_state_reproduces_the_run():
    # pf_set_state semantics: the post-resample state entering frame t
    # (positions gathered through frame t's ancestors) + identity ancestors
    frames, _ = rp.generate_video(rp.Params(), 6, 128, 128, (64.0, 64.0), 42)
    for mode in ("fp64", "fp32", "fp16"):
        tr = fused.FusedTrack(mode, 5000, 128, 128, 42, (64.0, 64.0))
        for t in range(4):
            tr.step(tr.loglik_map(frames[t]))
        xs, ys = tr.xs.copy(), tr.ys.copy()
        e4 = tr.step(tr.loglik_map(frames[4]))
        anc4 = tr.last_ancestors  # frame 4's ancestors into frame 3's positions
        e5 = tr.step(tr.loglik_map(frames[5]))
        inj = fused.FusedTrack(mode, 5000, 128, 128, 42, (64.0, 64.0))
        inj.set_state(xs[anc4], ys[anc4], 4)
        assert inj.step(inj.loglik_map(frames[4])) == e4
        assert inj.step(inj.loglik_map(frames[5])) == e5


@pytest.mark.parametrize("mode,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_oracle_teacher_forced_per_frame(mode, tol):
    # the fused algorithm given the reference's state entering each frame
    # reproduces the reference's estimate of that frame (SURVEY 8d
    # "teacher-forced per frame"); the GPU version at C2/C3 sizes is
    # tests/test_gpu_teacher.py
    frames, _ = rp.generate_video(rp.Params(), 40, 128, 128, (64.0, 64.0), 42)
    K = 20_000
    eng = rp.make_engine(mode, rp.Params(), rp.disk_offsets(5))
    stream = rng.LcgStream(42)
    s = eng.init(K, (64.0, 64.0))
    worst = 0.0
    for t in range(40):
        xs_in, ys_in = s.xs[s.ancestors], s.ys[s.ancestors]
        eng.propagate(s, stream.normals(K))
        eng.likelihoods(s, frames[t])
        eng.normalize_and_scan(s, eng.weight_update(s, eng.max_loglik(s)))
        ref = np.array(eng.estimate(s))
        eng.resample(s, stream.uniform())
        tr = fused.FusedTrack(mode, K, 128, 128, 42, (64.0, 64.0))
        tr.set_state(xs_in, ys_in, t)
        est = np.array(tr.step(tr.loglik_map(frames[t])))
        worst = max(worst, float(np.max(np.abs(est - ref) / np.abs(ref))))
    assert worst <= tol, worst
