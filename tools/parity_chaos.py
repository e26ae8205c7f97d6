#!/usr/bin/env python
"""Whole-run divergence at C2 (128x128, 100 frames, K=10^6) with identical draws.

Measures, per frame, the max relative difference of the trajectories:
  fused FP64 vs reference FP64, fused FP32 vs reference FP32,
  reference FP32 vs reference FP64, fused FP16 vs reference FP64 (tracking)
(oracle/fused.py = the CUDA path bit for bit; oracle/reference_port.py =
halfpf bit for bit; both on the product LCG stream).  The FP32 whole-run
numbers are chaotic (a single CDF rounding moves a resampling decision), which
is why the FP32 acceptance bound is per frame, teacher-forced
(tests/test_gpu_teacher.py).  Output: profiles/round2/parity_chaos_c2.txt
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import fused, rng  # noqa: E402
from oracle import reference_port as rp  # noqa: E402

K, F = 1_000_000, 100
frames, truth = rp.generate_video(rp.Params(), F, 128, 128, (64.0, 64.0), 42)
ref64 = rp.run(frames, K, "fp64", 42, rng.LcgStream)
ref32 = rp.run(frames, K, "fp32", 42, rng.LcgStream)
fu64, _ = fused.run(frames, K, "fp64", 42)
fu32, _ = fused.run(frames, K, "fp32", 42)
fu16, _ = fused.run(frames, K, "fp16", 42)


def rel(a, b):
    return np.max(np.abs(a - b) / np.abs(b), axis=1)


def err(t):
    return float(np.mean(np.hypot(*(t - truth).T)))


rows = {"fused64_vs_ref64": rel(fu64, ref64), "fused32_vs_ref32": rel(fu32, ref32),
        "ref32_vs_ref64": rel(ref32, ref64), "fused32_vs_ref64": rel(fu32, ref64)}
out = [__doc__.strip(), ""]
for k, v in rows.items():
    onset = next((t for t in range(F) if v[t] > 1e-4), None)
    out.append(f"{k:20s} max rel {v.max():.3e}  first frame > 1e-4: {onset}  frame0 {v[0]:.2e}")
out.append(f"mean tracking error px: ref64 {err(ref64):.4f} ref32 {err(ref32):.4f} fused64 {err(fu64):.4f} "
           f"fused32 {err(fu32):.4f} fused16 {err(fu16):.4f}")
txt = "\n".join(out)
print(txt)
os.makedirs(os.path.join(ROOT, "profiles", "round2"), exist_ok=True)
open(os.path.join(ROOT, "profiles", "round2", "parity_chaos_c2.txt"), "w").write(txt + "\n")
