"""Per-frame device timeline of the fused path from %globaltimer stamps.

  python tools/trace_frames.py [--config c2] [--precision fp16] [--tpb 0]

Runs one warm step, then one traced step, and prints (median over frames,
microseconds, relative to the first fused CTA entry of the frame):
fused entry spread, draws done, release (predecessor done), window ready,
particles done, exit; table entry, release, end.  Per-frame period = the
difference between consecutive frames' first release.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _q(v):
    return f"{v.mean():.2f}/{np.percentile(v, 90):.2f}/{v.max():.2f}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--precision", default=None)
    ap.add_argument("--tpb", type=int, default=0)
    ap.add_argument("--frames", type=int, default=0)
    args = ap.parse_args()
    import bench
    import paper_2308_00763_b200 as pf
    from paper_2308_00763_b200 import _native as N
    from oracle import reference_port as rp

    cfg = dict(bench.CONFIGS[args.config])
    prec = args.precision or cfg["precision"]
    F = args.frames or cfg["F"]
    frames, _ = rp.generate_video(rp.Params(), F, cfg["W"], cfg["H"], (cfg["W"] / 2, cfg["H"] / 2), 42)
    f = pf.Filter(cfg["K"], prec, cfg["W"], cfg["H"], 42, tpb=args.tpb or None)
    import torch

    dev = torch.from_numpy(frames).cuda()
    f.run_frames(dev, F)
    L = N.lib()
    N.check(L.pf_set_trace(f._h, 1), f._err)
    f.reset()
    f.run_frames(dev, F)
    f.reset()
    f.run_frames(dev, F)
    nt = (cfg["K"] + 1023) // 1024
    nc = 1 if nt <= 1024 else (nt + 255) // 256
    per = (nt + nc) * 8
    buf = np.zeros(F * per, dtype=np.uint64)
    N.check(L.pf_get_trace(f._h, N.ptr(buf), buf.size), f._err)
    buf = buf.reshape(F, nt + nc, 8).astype(np.int64)
    rows = []
    for t in range(F):
        fu = buf[t, :nt]
        tb = buf[t, nt:]
        t0 = fu[:, 0].min()

        def rel(a):
            a = a[a > 0]
            if a.size == 0:
                return (float("nan"), float("nan"))
            return (a.min() - t0) / 1e3, (a.max() - t0) / 1e3

        rows.append(dict(
            entry=rel(fu[:, 0]), draws=rel(fu[:, 1]), release=rel(fu[:, 2]), window=rel(fu[:, 3]),
            parts=rel(fu[:, 4]), exit=rel(fu[:, 5]), t_entry=rel(tb[:, 0]), t_rel=rel(tb[:, 1]),
            t_max=rel(tb[:, 4]), t_scan=rel(tb[:, 6]), t_tab=rel(tb[:, 7]), t_win=rel(tb[:, 5]), t_tree=rel(tb[:, 2]), t_end=rel(tb[:, 3]) if (tb[:, 3] > 0).any() else (0, 0), t0=t0))
    print(f"{args.config} {prec} K={cfg['K']} tiles={nt} chunks={nc} frames={F}")
    keys = ["entry", "draws", "release", "window", "parts", "exit", "t_entry", "t_rel", "t_max", "t_scan", "t_tab", "t_win", "t_tree", "t_end"]
    med = {k: (np.median([r[k][0] for r in rows[1:]]), np.median([r[k][1] for r in rows[1:]])) for k in keys}
    for k in keys:
        print(f"  {k:8s} first {med[k][0]:8.2f} us   last {med[k][1]:8.2f} us")
    # mean per-CTA phase durations (frames 1..F-1)
    fu = buf[1:, :nt].reshape(-1, 8).astype(np.float64)
    ok = (fu[:, :6] > 0).all(axis=1)
    fu = fu[ok]
    names = ["draws", "wait", "window", "particles", "tail"]
    d = np.diff(fu[:, :6], axis=1) / 1e3
    print("  mean per-CTA phase (us): " + ", ".join(f"{n} {v:.2f}" for n, v in zip(names, d.mean(axis=0))) +
          f"  | lifetime {(fu[:, 5] - fu[:, 0]).mean() / 1e3:.2f}")
    # inside the particle phase (trace slots 6 / 7: window CDFs landed, thread 0's search done)
    fu = buf[1:, :nt].reshape(-1, 8).astype(np.float64)
    ok = (fu[:, :8] > 0).all(axis=1)
    if ok.any():
        g = fu[ok]
        print(f"  particle phase split (us, mean / p90 / max): "
              f"copy wait {_q((g[:, 6] - g[:, 3]) / 1e3)}, search {_q((g[:, 7] - g[:, 6]) / 1e3)}, "
              f"gather..max {_q((g[:, 4] - g[:, 7]) / 1e3)}")
    t0s = np.array([r["t0"] for r in rows])
    print(f"  period (fused entry to entry): median {np.median(np.diff(t0s))/1e3:.2f} us")
    rel0 = np.array([r["t0"] + r["release"][0] * 1e3 for r in rows])
    print(f"  period (first release): median {np.median(np.diff(rel0))/1e3:.2f} us")
    f.close()


if __name__ == "__main__":
    main()
