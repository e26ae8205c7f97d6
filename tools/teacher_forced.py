"""Teacher-forced per-frame parity numbers (what tests/test_gpu_teacher.py asserts).

  python tools/teacher_forced.py > profiles/round2/teacher_forced.txt

For every frame t of C2 (128x128, 100 frames, 10^6 particles) in FP64 and FP32
and a C3 slice (1024x1024, 6 frames, 2^24 particles, FP32): the reference
state entering frame t (oracle/reference_port.py on the LCG stream, pinned to
halfpf) is injected with pf_set_state, one fused frame runs, and its estimate
is compared with the reference's estimate of frame t (relative error, max
over x / y).  Prints the worst and median frame.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import paper_2308_00763_b200 as pf
    from oracle import reference_port as rp
    from test_gpu_teacher import TOL, teacher_forced

    cases = [("C2", 100, 128, 1_000_000, "fp64"), ("C2", 100, 128, 1_000_000, "fp32"),
             ("C3 slice", 6, 1024, 1 << 24, "fp32")]
    for name, F, W, K, mode in cases:
        frames, _ = rp.generate_video(rp.Params(), F, W, W, (W / 2.0, W / 2.0), 42)
        worst, per = teacher_forced(pf, frames, K, mode)
        print(f"{name:9s} {mode}: K={K} frames={F}  worst rel {worst:.3e} (frame {int(np.argmax(per))})  "
              f"median {np.median(per):.3e}  tolerance {TOL[mode]:g}", flush=True)


if __name__ == "__main__":
    main()
