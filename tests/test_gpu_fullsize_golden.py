"""The CUDA fused path at full BASELINE sizes, bit-exact against committed
outputs of its CPU restatement (oracle/fused.py), which takes minutes per
precision at these sizes (fixtures: oracle/tools/make_fullsize_golden.py).

  C2 (BASELINE.json configs[1]): 128x128, 100 frames, 10^6 particles, FP64/FP32/FP16
  C3 slice (configs[2]):          1024x1024, first 3 frames, 2^24 particles, FP16

Compared: the whole trajectory (exact), and SHA-256 digests of the final
positions and local CDFs (every particle's state, bit for bit)."""

import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import reference_port as rp

pytestmark = pytest.mark.gpu

CASES = ["c2_fp64", "c2_fp32", "c2_fp16", "c3_fp16"]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", CASES)
def test_fullsize_bit_exact(name):
    import paper_2308_00763_b200 as pf

    path = os.path.join(GOLDEN, f"fullsize_{name}.npz")
    g = np.load(path)
    K, W, H, F, mode = int(g["K"]), int(g["W"]), int(g["H"]), int(g["F"]), str(g["mode"])
    frames, _ = rp.generate_video(rp.Params(), F, W, H, (W / 2.0, H / 2.0), 42)
    assert _sha(frames) == str(g["frames_sha256"])
    modes = ["fp16", "fp16-packed"] if mode == "fp16" else [mode]
    for m in modes:
        f = pf.Filter(K, m, W, H, 42)
        traj = f.run(frames)
        assert np.array_equal(traj, g["traj"]), (name, m, np.abs(traj - g["traj"]).max())
        xs, ys, cdf = f.state()
        assert _sha(xs) == str(g["xs_sha256"]) and _sha(ys) == str(g["ys_sha256"]), (name, m)
        assert _sha(cdf) == str(g["cdf_sha256"]), (name, m)
        f.close()
