"""GPU parity of the reference-semantics stage engine (make_engine / stage_hook).

Draws are injected exactly as the reference allows (`RngStream` is resolved at
call time), so the staged engine is compared against the reference's own
goldens: binary16 bit-exact, FP64/FP32 within tolerance (the only deviation
is NumPy's SIMD exp vs the device's portable exp)."""

import numpy as np
import pytest

from conftest import golden
from oracle import reference_port as rp
from oracle import rng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import paper_2308_00763_b200 as pf

    return pf


def _video(pf, v):
    frames, truth = v
    return pf.Video(frames=frames, truth=truth)


@pytest.mark.parametrize("mode", ["fp16", "fp16-packed"])
def test_staged_binary16_bit_exact_vs_reference(pf, acceptance_video, mode):
    res = pf.run(_video(pf, acceptance_video), 128, mode, 42, start_hint=(64.0, 64.0), engine="staged")
    assert np.array_equal(res.trajectory, golden("acceptance_k128.npz")[f"{mode}_traj"])


@pytest.mark.parametrize("mode,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_staged_wide_vs_reference(pf, acceptance_video, mode, tol):
    res = pf.run(_video(pf, acceptance_video), 128, mode, 42, start_hint=(64.0, 64.0), engine="staged")
    ref = golden("acceptance_k128.npz")[f"{mode}_traj"]
    assert np.max(np.abs(res.trajectory - ref) / np.abs(ref)) <= tol


def test_staged_reference_stream_reproduces_fp64_mean_err(pf, acceptance_video, monkeypatch):
    # inject the reference's own Philox stream: FP64_MEAN_ERR (test_acceptance.py:40)
    import paper_2308_00763_b200.filter as F

    monkeypatch.setattr(F, "RngStream", rp.numpy_philox_stream)
    frames, truth = acceptance_video
    res = pf.run(_video(pf, acceptance_video), 128, "fp64", 42, start_hint=(64.0, 64.0), engine="staged")
    err = float(np.mean(np.hypot(*(res.trajectory - truth).T)))
    assert err == pytest.approx(1.255495438119523, rel=1e-9)


@pytest.mark.parametrize("mode", ["fp64", "fp32", "fp16"])
def test_stage_by_stage_vs_oracle(pf, acceptance_video, mode):
    frames, _ = acceptance_video
    P = rp.Params()
    eng = pf.make_engine(mode)
    ps = eng.init(500, (64.0, 64.0))
    oe = rp.make_engine(mode, P, rp.disk_offsets(5))
    os_ = oe.init(500, (64.0, 64.0))
    stream = rng.LcgStream(3)
    wide_tol = {"fp64": 1e-15, "fp32": 1e-6}
    wide_atol = {"fp64": 1e-300, "fp32": 1e-37}  # subnormal weights carry no relative precision
    for t in range(6):
        noise = stream.normals(500)
        eng.propagate(ps, noise)
        oe.propagate(os_, noise)
        assert np.array_equal(ps.xs, os_.xs) and np.array_equal(ps.ys, os_.ys)
        eng.likelihoods(ps, frames[t])
        oe.likelihoods(os_, frames[t])
        assert np.array_equal(ps.loglik, os_.loglik)
        m = eng.max_loglik(ps)
        assert float(m) == float(oe.max_loglik(os_))
        tot = eng.weight_update(ps, m)
        otot = oe.weight_update(os_, m)
        if mode == "fp16":
            assert np.array_equal(ps.weights, os_.weights) and tot == otot
        else:
            assert np.allclose(ps.weights, os_.weights, rtol=wide_tol[mode], atol=wide_atol[mode])
            os_.weights = ps.weights  # continue from identical weights
            otot = os_.weights.sum(dtype=os_.weights.dtype)
            assert tot == otot  # NumPy pairwise sum order reproduced bit-exactly
        eng.normalize_and_scan(ps, tot)
        oe.normalize_and_scan(os_, otot)
        assert np.array_equal(ps.weights, os_.weights) and np.array_equal(ps.cdf, os_.cdf)
        assert eng.estimate(ps) == oe.estimate(os_)
        u = stream.uniform()
        eng.resample(ps, u)
        oe.resample(os_, u)
        assert np.array_equal(ps.ancestors, os_.ancestors)
        assert np.array_equal(ps.weights, os_.weights)


def test_degeneracy_carries_frame(pf):
    # test_filter.py:386-398 sabotage via stage_hook
    frames, truth = rp.generate_video(rp.Params(), 3, 64, 64, (20.0, 20.0), 5)

    def sabotage(t, name, ps):
        if t == 1 and name == "max":
            ps.weights = np.zeros(ps.count)

    with pytest.raises(pf.DegeneracyError) as info:
        pf.run(pf.Video(frames, truth), 8, "fp64", 6, template=pf.disk_template(2), stage_hook=sabotage)
    assert info.value.frame == 1


def test_stage_hook_order(pf):
    frames, truth = rp.generate_video(rp.Params(), 2, 64, 64, (20.0, 20.0), 5)
    seen = []
    pf.run(pf.Video(frames, truth), 8, "fp64", 7, template=pf.disk_template(2),
           stage_hook=lambda t, name, ps: seen.append((t, name)))
    assert seen == [(t, s) for t in range(2) for s in pf.STAGES]


def test_half_degenerate_at_65536(pf):
    # reference FP16 semantics: fp16(65536) = inf -> 1/K = 0 -> DegeneracyError at frame 0
    frames, truth = rp.generate_video(rp.Params(), 2, 64, 64, (32.0, 32.0), 5)
    with pytest.raises(pf.DegeneracyError) as info:
        pf.run(pf.Video(frames, truth), 65536, "fp16", 1, engine="staged")
    assert info.value.frame == 0


def test_systematic_ancestors_kats(pf):
    g = golden("resample_kats.npz")
    o = 0
    for L, u in zip(g["lens"], g["u"]):
        assert np.array_equal(pf.systematic_ancestors(g["cdf"][o:o + L], float(u)), g["anc"][o:o + L])
        o += L


def test_resampling_criterion4_dense_oracle(pf):
    # test_acceptance.py:182-230 (subset of u values per weight vector)
    g = np.random.default_rng(42)
    us = (np.arange(500) + 0.5) / 500
    for k in range(2, 9):
        for w in [np.full(k, 1.0 / k)] + [g.uniform(0, 1, k) for _ in range(3)]:
            w = w / w.sum()
            cdf = np.cumsum(w)
            pts = (np.arange(k)[None, :] + us[:, None]) / k
            oracle = np.argmax(cdf[None, None, :] >= pts[:, :, None], axis=2)
            counts = np.zeros(k)
            for i, u in enumerate(us):
                a = pf.systematic_ancestors(cdf, float(u))
                assert np.array_equal(a, oracle[i])
                counts += np.bincount(a, minlength=k)
            assert np.all(np.abs(counts / len(us) - k * w) <= 1.0)


def test_half_stage_kats(pf):
    g = golden("half_stage_kats.npz")
    for i, K in enumerate((16, 17, 1000, 4096)):
        mode = "fp16-packed" if K % 2 == 0 else "fp16"
        eng = pf.make_engine(mode, template=pf.disk_template(2))
        ps = eng.init(K, (0.0, 0.0))
        ps.weights = [int(v) for v in g[f"w_{i}"]]
        eng.normalize_and_scan(ps, float(g[f"total_{i}"]))
        assert np.array_equal(ps.weights.view(np.uint16), g[f"wn_{i}"])
        assert np.array_equal(ps.cdf.view(np.uint16), g[f"cdf_{i}"])
        eng.resample(ps, float(g[f"u_{i}"]))
        assert np.array_equal(ps.ancestors, g[f"anc_{i}"])
