"""Reference-semantics oracle pinned against the reference's own outputs.

The goldens in tests/golden/ were produced by running the real `halfpf`
(/root/reference/pkg/src) with oracle/tools/make_golden.py.  Where the
reference is importable (build container) the oracle is also checked against
it live."""

import numpy as np
import pytest

from conftest import golden, have_reference
from oracle import reference_port as rp
from oracle import rng

MODES = ["fp64", "fp32", "fp16", "fp16-packed"]


def test_video_generator_restatement(acceptance_video):
    import hashlib

    frames, truth = acceptance_video
    g = golden("acceptance_k128.npz")
    assert hashlib.sha256(frames.tobytes()).hexdigest() == str(g["frames_sha256"])
    assert np.array_equal(truth, g["truth"])


def test_fp64_mean_err_golden(acceptance_video):
    # test_acceptance.py:40 FP64_MEAN_ERR = 1.255495438119523 (reference's own stream)
    frames, truth = acceptance_video
    traj = rp.run(frames, 128, "fp64", 42, rp.numpy_philox_stream, start_hint=(64.0, 64.0))
    g = golden("acceptance_k128.npz")
    assert np.array_equal(traj, g["philox_fp64_traj"])
    err = float(np.mean(np.hypot(*(traj - truth).T)))
    assert err == pytest.approx(1.255495438119523, rel=1e-12)


@pytest.mark.parametrize("mode", MODES)
def test_acceptance_trajectory_and_stages_bit_exact(acceptance_video, mode):
    frames, truth = acceptance_video
    g = golden("acceptance_k128.npz")
    snaps = {}

    def hook(t, name, s):
        if t < 4:
            snaps[(t, name)] = s.snapshot()

    traj = rp.run(frames, 128, mode, 42, rng.LcgStream, start_hint=(64.0, 64.0), stage_hook=hook)
    assert np.array_equal(traj, g[f"{mode}_traj"])
    for (t, name), s in snaps.items():
        for k, v in s.items():
            ref = g[f"{mode}_t{t}_{name}_{k}"]
            got = v.view(np.uint16) if v.dtype == np.float16 else v
            assert np.array_equal(got, ref), (t, name, k)


@pytest.mark.parametrize("mode", ["fp64", "fp32"])
def test_c1_trajectory_bit_exact(c1_video, mode):
    frames, _ = c1_video
    g = golden("c1_k10000.npz")
    assert np.array_equal(rp.run(frames, 10_000, mode, 42, rng.LcgStream), g[f"{mode}_traj"])


def test_odd_params_bit_exact():
    g = golden("odd_params.npz")
    P = rp.Params(bg_mean=100.3, fg_mean=227.7, likelihood_scale=47.1, drift_x=0.7, std_x=4.3, disk_radius=4)
    for mode in ("fp64", "fp32", "fp16"):
        traj = rp.run(g["frames"], 301, mode, 9, rng.LcgStream, params=P, offsets=rp.disk_offsets(4))
        assert np.array_equal(traj, g[f"{mode}_traj"]), mode


def test_resample_kats():
    g = golden("resample_kats.npz")
    lens, cdf, us, anc = g["lens"], g["cdf"], g["u"], g["anc"]
    o = 0
    for L, u in zip(lens, us):
        assert np.array_equal(rp.systematic_ancestors(cdf[o:o + L], float(u)), anc[o:o + L])
        o += L
    # test_filter.py:281-294 examples
    assert list(rp.systematic_ancestors(np.array([0.5, 1.0, 1.0, 1.0]), 0.1)) == [0, 0, 1, 1]
    assert list(rp.systematic_ancestors(np.array([0.0, 0.0, 1.0, 1.0]), 0.5)) == [2, 2, 2, 2]


def test_half_stage_kats():
    g = golden("half_stage_kats.npz")
    for i, K in enumerate((16, 17, 1000, 4096)):
        eng = rp.HalfEngine(rp.Params(), rp.disk_offsets(2))
        s = eng.init(K, (0.0, 0.0))
        s.weights = g[f"w_{i}"].view(np.float16)
        eng.normalize_and_scan(s, float(g[f"total_{i}"]))
        assert np.array_equal(s.weights.view(np.uint16), g[f"wn_{i}"])
        assert np.array_equal(s.cdf.view(np.uint16), g[f"cdf_{i}"])
        eng.resample(s, float(g[f"u_{i}"]))
        assert np.array_equal(s.ancestors, g[f"anc_{i}"])


def test_exp16_table_matches_halfnum_semantics():
    # halfnum.exp16 = RN16(math.exp(v)) (halfnum.py:254-263); spot-check vs numpy float16
    t = rp.exp16_table()
    x = np.arange(0x8000, 0xCC00, 7, dtype=np.uint32).astype(np.uint16).view(np.float16)
    assert np.array_equal(t[x.view(np.uint16)], np.exp(x.astype(np.float64)).astype(np.float16))


@pytest.mark.skipif(not have_reference(), reason="reference not mounted (GPU box)")
def test_live_against_reference_small():
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    import halfpf.filter as hf
    from halfpf.model import ModelParams, generate_video

    vid = generate_video(ModelParams(), 8, 64, 48, (20.0, 30.0), 11)
    orig = hf.RngStream
    hf.RngStream = rng.LcgStream
    try:
        for mode in MODES:
            a = hf.run(vid, 37 if mode != "fp16-packed" else 38, hf.PrecisionMode.from_name(mode), 3).trajectory
            b = rp.run(vid.frames, 37 if mode != "fp16-packed" else 38, mode, 3, rng.LcgStream)
            assert np.array_equal(a, b), mode
    finally:
        hf.RngStream = orig
