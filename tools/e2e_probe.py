"""Per-step breakdown of the host-buffer (e2e) path: wall clock vs the
library's device-event stage timings.  python tools/e2e_probe.py --config c3"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--precision", default=None)
    ap.add_argument("--steps", type=int, default=6)
    args = ap.parse_args()
    import torch

    import bench
    import paper_2308_00763_b200 as pf

    cfg = dict(bench.CONFIGS[args.config])
    prec = args.precision or cfg["precision"]
    F, W, H, K = cfg["F"], cfg["W"], cfg["H"], cfg["K"]
    v = pf.generate_video(pf.ModelParams(), F, W, H, (W / 2.0, H / 2.0), 42)
    pinned = torch.from_numpy(v.frames).pin_memory()
    host = pinned.numpy()
    f = pf.Filter(K, prec, W, H, 42)
    for i in range(args.steps):
        torch.cuda.synchronize()
        f.reset()
        t0 = time.perf_counter()
        f.run_frames(host, F)
        wall = (time.perf_counter() - t0) * 1e3
        t = f.timings()
        print(f"step {i}: wall {wall:8.2f} ms  " + "  ".join(f"{k} {x:7.2f}" for k, x in t.items()))


if __name__ == "__main__":
    main()
