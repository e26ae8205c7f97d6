"""Generate tests/golden/*.npz by running the REAL reference in this container.

TEST INFRASTRUCTURE.  Imports `halfpf` from /root/reference/pkg/src (read-only;
nothing is copied), swaps `halfpf.filter.RngStream` (resolved at call time,
filter.py:611) for `oracle.rng.LcgStream` where the product stream is wanted,
and records trajectories, per-stage snapshots and resampling KATs.  The GPU box
has no /root/reference; its tests read these fixtures.

Usage:  PYTHONPATH=. python oracle/tools/make_golden.py
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import halfpf.filter as hf  # noqa: E402
from halfpf import halfnum  # noqa: E402
from halfpf.model import ModelParams, disk_template, generate_video  # noqa: E402

from oracle import rng  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")
MODES = ["fp64", "fp32", "fp16", "fp16-packed"]


def _raw(a):
    if isinstance(a, list):
        return np.array(a, dtype=np.uint16)
    return np.asarray(a).copy()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def acceptance():
    """Reference acceptance scenario (test_acceptance.py:32-79): 100 frames,
    128x128, K=128, seed 42, start (64,64), all modes, product (LCG) stream,
    with stage snapshots for frames 0..3; plus the reference's own Philox
    stream FP64 trajectory (FP64_MEAN_ERR)."""
    vid = generate_video(ModelParams(), 100, 128, 128, (64.0, 64.0), 42)
    out = {"frames_sha256": np.array(sha(vid.frames)), "truth": vid.truth}
    orig = hf.RngStream
    for mode in MODES:  # the reference's own stream (Generator(Philox(42)))
        out[f"philox_{mode}_traj"] = hf.run(vid, 128, hf.PrecisionMode.from_name(mode), 42,
                                             start_hint=(64.0, 64.0)).trajectory
    hf.RngStream = rng.LcgStream
    try:
        for mode in MODES:
            snaps = {}

            def hook(t, name, ps):
                if t < 4:
                    snaps[(t, name)] = ps.snapshot()

            res = hf.run(vid, 128, hf.PrecisionMode.from_name(mode), 42, start_hint=(64.0, 64.0), stage_hook=hook)
            out[f"{mode}_traj"] = res.trajectory
            for (t, name), s in snaps.items():
                for k, v in s.items():
                    out[f"{mode}_t{t}_{name}_{k}"] = _raw(v)
    finally:
        hf.RngStream = orig
    np.savez_compressed(os.path.join(OUT, "acceptance_k128.npz"), **out)


def c1():
    """BASELINE config 1: 128x128, 10 frames, K=10,000, seed 42 (FP64 + FP32),
    product stream; plus the Philox-stream FP64/FP32 trajectories."""
    vid = generate_video(ModelParams(), 10, 128, 128, (64.0, 64.0), 42)
    out = {"frames_sha256": np.array(sha(vid.frames)), "truth": vid.truth}
    for mode in ("fp64", "fp32"):
        out[f"philox_{mode}_traj"] = hf.run(vid, 10_000, hf.PrecisionMode.from_name(mode), 42).trajectory
    orig = hf.RngStream
    hf.RngStream = rng.LcgStream
    try:
        for mode in ("fp64", "fp32"):
            out[f"{mode}_traj"] = hf.run(vid, 10_000, hf.PrecisionMode.from_name(mode), 42).trajectory
    finally:
        hf.RngStream = orig
    np.savez_compressed(os.path.join(OUT, "c1_k10000.npz"), **out)


def odd_params():
    """Non-default params, odd K, non-square frame: exercises rounding of the
    per-pixel terms (pairwise sum order), odd-K lane tails, border clamping."""
    P = ModelParams(bg_mean=100.3, fg_mean=227.7, likelihood_scale=47.1, drift_x=0.7, std_x=4.3, disk_radius=4)
    vid = generate_video(P, 12, 96, 80, (30.0, 40.0), 3)
    out = {"frames": vid.frames, "truth": vid.truth}
    orig = hf.RngStream
    hf.RngStream = rng.LcgStream
    try:
        for mode in ("fp64", "fp32", "fp16"):
            out[f"{mode}_traj"] = hf.run(vid, 301, hf.PrecisionMode.from_name(mode), 9, params=P,
                                         template=disk_template(4)).trajectory
    finally:
        hf.RngStream = orig
    np.savez_compressed(os.path.join(OUT, "odd_params.npz"), **out)


def resample_kats():
    """systematic_ancestors KATs (test_filter.py:280-347, test_acceptance.py:182-230)."""
    g = np.random.default_rng(41)
    cdfs, us, ancs = [], [], []
    cases = [(np.array([0.5, 1.0, 1.0, 1.0]), 0.1), (np.array([0.0, 0.0, 1.0, 1.0]), 0.5)]
    for k in (8,):
        c = np.cumsum(np.full(k, 1.0 / k))
        cases += [(c, 0.25), (c, 0.3), (c, 0.999)]
    for _ in range(200):
        K = int(g.integers(2, 300))
        w = g.uniform(0, 1, K) * (g.uniform(0, 1, K) < 0.4)
        w[g.integers(0, K)] += 0.5
        w /= w.sum()
        cases.append((np.cumsum(w), float(g.random())))
    for c, u in cases:
        cdfs.append(c)
        us.append(u)
        ancs.append(hf.systematic_ancestors(c, u))
    lens = np.array([len(c) for c in cdfs])
    np.savez_compressed(os.path.join(OUT, "resample_kats.npz"), lens=lens, cdf=np.concatenate(cdfs),
                        u=np.array(us), anc=np.concatenate(ancs))


def half_resample_kats():
    """Binary16 engine resample on half CDFs (test_filter.py:314-337)."""
    g = np.random.default_rng(43)
    out = {}
    for i, K in enumerate((16, 17, 1000, 4096)):
        eng = hf.make_engine(hf.PrecisionMode.FP16_PACKED if K % 2 == 0 else hf.PrecisionMode.FP16_SCALAR,
                             template=disk_template(2))
        ps = eng.init(K, (0.0, 0.0))
        w16 = [halfnum.from_f64(float(v)) for v in g.uniform(0, 1, K)]
        ps.weights = w16
        total = float(sum(halfnum.to_f64(b) for b in w16))
        eng.normalize_and_scan(ps, total)
        out[f"w_{i}"] = np.array(w16, dtype=np.uint16)
        out[f"total_{i}"] = np.array(total)
        out[f"wn_{i}"] = np.array(ps.weights, dtype=np.uint16)
        out[f"cdf_{i}"] = np.array(ps.cdf, dtype=np.uint16)
        u = float(g.random())
        eng.resample(ps, u)
        out[f"u_{i}"] = np.array(u)
        out[f"anc_{i}"] = ps.ancestors.copy()
    np.savez_compressed(os.path.join(OUT, "half_stage_kats.npz"), **out)


def lcg_stream():
    """Pin the product stream itself: first draws of a few seeds + far positions."""
    out = {}
    for seed in (0, 1, 42, 2**63 + 5):
        s = rng.LcgStream(seed)
        out[f"n_{seed}"] = s.normals(4096)
        out[f"u_{seed}"] = np.array([s.uniform() for _ in range(8)])
    x0 = rng.lcg_seed_state(42)
    out["far_pos"] = np.array([10**6, 2**31 + 7, 10**12 + 3], dtype=np.uint64)
    out["far_words"] = np.array([rng.lcg_word(x0, int(p)) for p in out["far_pos"]], dtype=np.uint64)
    np.savez_compressed(os.path.join(OUT, "lcg_stream.npz"), **out)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    for fn in (lcg_stream, resample_kats, half_resample_kats, acceptance, c1, odd_params):
        fn()
        print("done", fn.__name__, flush=True)
