"""Generate full-BASELINE-size goldens of the fused algorithm (oracle/fused.py).

ORACLE tooling (test infrastructure only).  The CUDA fused path must be
bit-exact against oracle/fused.py; at the BASELINE sizes the oracle takes
minutes per precision on a CPU, so its outputs are committed as fixtures and
tests/test_gpu_fullsize_golden.py asserts the GPU reproduces them exactly:

  C2 (BASELINE.json configs[1]): 128x128, 100 frames, K = 10^6, FP64 / FP32 / FP16
  C3 slice (configs[2]):          1024x1024, first 3 frames, K = 2^24, FP16

Each case stores the (F, 2) trajectory and SHA-256 digests of the final
positions (x, y) and the final local CDF (mode dtype bytes).  Inputs:
reference video model (oracle/reference_port.generate_video, seed 42,
start (W/2, H/2)), run seed 42, disk_template(5).

  python -m oracle.tools.make_fullsize_golden [c2_fp64 c2_fp32 c2_fp16 c3_fp16]
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import fused  # noqa: E402
from oracle import reference_port as rp  # noqa: E402

CASES = {
    "c2_fp64": dict(W=128, H=128, F=100, K=1_000_000, mode="fp64"),
    "c2_fp32": dict(W=128, H=128, F=100, K=1_000_000, mode="fp32"),
    "c2_fp16": dict(W=128, H=128, F=100, K=1_000_000, mode="fp16"),
    "c3_fp16": dict(W=1024, H=1024, F=3, K=1 << 24, mode="fp16"),
}
OUT_DIR = os.path.join(ROOT, "tests", "golden")


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make(name: str) -> None:
    c = CASES[name]
    frames, _ = rp.generate_video(rp.Params(), c["F"], c["W"], c["H"], (c["W"] / 2.0, c["H"] / 2.0), 42)
    t0 = time.time()
    traj, tr = fused.run(frames, c["K"], c["mode"], 42)
    dt = time.time() - t0
    out = os.path.join(OUT_DIR, f"fullsize_{name}.npz")
    np.savez(out, traj=traj, xs_sha256=np.array(digest(tr.xs)), ys_sha256=np.array(digest(tr.ys)),
             cdf_sha256=np.array(digest(tr.c)), K=c["K"], W=c["W"], H=c["H"], F=c["F"], mode=np.array(c["mode"]),
             frames_sha256=np.array(digest(frames)))
    print(f"{name}: {dt:.0f} s -> {out}", flush=True)


if __name__ == "__main__":
    for n in (sys.argv[1:] or list(CASES)):
        make(n)
