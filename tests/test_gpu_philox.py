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
