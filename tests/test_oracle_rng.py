"""Oracle RNG: pinned against NumPy's own Philox/ziggurat and the committed LCG goldens."""

import hashlib
import math

import numpy as np
import pytest

from conftest import golden
from oracle import rng


@pytest.mark.parametrize("seed", [7, 42, 12345])
def test_ziggurat_tables_reproduce_numpy_standard_normal(seed):
    # RngStream.normals = Generator(Philox(seed)).standard_normal (filter.py:76-79)
    n = 60_000
    ref = np.random.Generator(np.random.Philox(seed)).standard_normal(n)
    src = rng._WordSource(np.random.Philox(seed).random_raw(int(n * 1.05) + 200))
    got = np.array([rng.numpy_standard_normal(src) for _ in range(n)])
    assert np.array_equal(got, ref)


def test_philox_uniform_layout():
    # RngStream.uniform = random() = (word >> 11) * 2^-53 (filter.py:81-82)
    w = np.random.Philox(3).random_raw(5)
    ref = np.random.Generator(np.random.Philox(3)).random(5)
    assert np.array_equal((w >> np.uint64(11)).astype(np.float64) * rng.TWO_M53, ref)


def test_survey_rng_goldens():
    # SURVEY.md A.3 values of the reference stream
    s = np.random.Generator(np.random.Philox(42))
    assert s.standard_normal((2, 2)).tolist() == [[-1.1043995228921153, 0.1891281100736375],
                                                   [0.04600092882122236, -2.1076745327476445]]
    assert float(s.random()) == 0.17016452673096505


def test_lcg_stream_matches_committed_golden():
    g = golden("lcg_stream.npz")
    for seed in (0, 1, 42, 2**63 + 5):
        s = rng.LcgStream(seed)
        assert np.array_equal(s.normals(4096), g[f"n_{seed}"])
        assert np.array_equal(np.array([s.uniform() for _ in range(8)]), g[f"u_{seed}"])
    x0 = rng.lcg_seed_state(42)
    for p, w in zip(g["far_pos"], g["far_words"]):
        assert rng.lcg_word(x0, int(p)) == int(w)


def test_lcg_jump_equals_sequential():
    x0 = rng.lcg_seed_state(9)
    x = x0
    seq = []
    for _ in range(300):
        seq.append(x)
        x = (rng.LCG_A * x + rng.LCG_C) & rng.M64
    assert [int(v) for v in rng.lcg_words(x0, 0, 300)] == seq
    assert [int(v) for v in rng.lcg_words(x0, 37, 100)] == seq[37:137]


def test_frame_layout_matches_stream_consumption():
    # run() draws normals(K) then uniform() per frame -> positions t(2K+1)+...
    K = 33
    s = rng.LcgStream(5)
    for t in range(3):
        n, u = rng.frame_draws(5, K, t)
        assert np.array_equal(s.normals(K), n)
        assert s.uniform() == u


def test_lcg_normals_statistics():
    x = rng.normals_from_lcg_words(rng.lcg_words(rng.lcg_seed_state(1), 0, 400_000))
    assert abs(x.mean()) < 0.01
    assert abs(x.std() - 1.0) < 0.01
    assert abs((x**4).mean() - 3.0) < 0.06
    # tail region (ziggurat layer 0) is exercised
    assert (np.abs(x) > rng.ZIG_R).sum() > 0


def test_slow_path_fraction():
    w = rng.lcg_words(rng.lcg_seed_state(2), 0, 200_000)
    idx = (w >> np.uint64(56)).astype(np.int64)
    rabs = (w >> np.uint64(3)) & np.uint64(rng.MASK52)
    slow = ~(rabs < rng.KI_NP[idx])
    assert 0.005 < slow.mean() < 0.02


def test_portable_exp_log_accuracy():
    xs = np.linspace(-700, 700, 200_001)
    e = rng.exp64_np(xs)
    assert np.max(np.abs(e - np.exp(xs)) / np.exp(xs)) < 5e-16
    for v in np.linspace(-0.999999, 5, 2001):
        assert abs(rng.log1p64(float(v)) - math.log1p(v)) <= 4e-16 * max(1.0, abs(math.log1p(v)))
    x32 = np.linspace(-86, 0, 50_001).astype(np.float32)
    e32 = rng.exp32_np(x32).astype(np.float64)
    ref = np.exp(x32.astype(np.float64))
    assert np.max(np.abs(e32 - ref) / ref) < 3e-7


def test_scalar_and_vector_exp_identical():
    xs = np.random.default_rng(0).uniform(-720, 720, 5000)
    v = rng.exp64_np(xs)
    assert all(rng.exp64(float(a)) == b for a, b in zip(xs, v))


def test_glibc_log1p_restatement_matches_libm():
    # NumPy's ziggurat tail uses npy_log1p (glibc); the device restatement must
    # agree bit-for-bit on the tail domain (-1, 0]
    import math

    g = np.random.default_rng(5)
    xs = np.concatenate([-g.random(60_000), -g.random(20_000) ** 12, -(1 - g.random(20_000) * 1e-3)])
    w = g.integers(0, 2**63, 40_000, dtype=np.int64).astype(np.uint64)
    xs = np.concatenate([xs, -(w >> np.uint64(11)).astype(np.float64) * 2.0**-53])
    assert all(rng.log1p_glibc(float(v)) == math.log1p(float(v)) for v in xs)
