"""Per-frame API latency breakdown (Filter.step, filter.py:617-654 analogue).

  python tools/step_probe.py [--K 1000000] [--precision fp16-packed]

Prints wall-clock us per call for: Filter.step on a host frame, on a device
frame, the raw C call pf_step (no Python validation), the library's device
event timings of one step, and pipelined pf_step_async throughput (frames
enqueued back to back, one sync at the end)."""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", type=int, default=1_000_000)
    ap.add_argument("--precision", default="fp16-packed")
    ap.add_argument("--n", type=int, default=100)
    args = ap.parse_args()
    import torch

    import paper_2308_00763_b200 as pf
    from paper_2308_00763_b200 import _native as N

    v = pf.generate_video(pf.ModelParams(), args.n, 128, 128, (64.0, 64.0), 42)
    host = np.ascontiguousarray(v.frames)
    dev = torch.from_numpy(host).cuda()
    f = pf.Filter(args.K, args.precision, 128, 128, 42)
    L = N.lib()

    def timed(fn, label):
        f.reset()
        for t in range(5):
            fn(t)
        torch.cuda.synchronize()
        f.reset()
        t0 = time.perf_counter()
        for t in range(args.n):
            fn(t)
        torch.cuda.synchronize()
        us = 1e6 * (time.perf_counter() - t0) / args.n
        print(f"{label:40s} {us:8.1f} us/frame")
        return us

    timed(lambda t: f.step(host[t]), "Filter.step(host frame)")
    timed(lambda t: f.step(dev[t]), "Filter.step(device frame)")
    est = np.empty(2)
    timed(lambda t: L.pf_step(f._h, host[t].ctypes.data, 0, est.ctypes.data), "pf_step (C, host frame)")
    ptrs = [dev[t].data_ptr() for t in range(args.n)]
    timed(lambda t: L.pf_step(f._h, C.c_void_p(ptrs[t]), 1, est.ctypes.data), "pf_step (C, device frame)")
    tm = f.timings()
    print("device timings of the last step (ms):", {k: round(x, 4) for k, x in tm.items()})
    outs = torch.empty((args.n, 2), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def enq(t):
        L.pf_step_async(f._h, C.c_void_p(ptrs[t]), 1, C.c_void_p(outs[t].data_ptr()), C.c_void_p(s))
    f.reset()
    for t in range(5):
        enq(t)
    L.pf_sync(f._h)
    f.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for t in range(args.n):
        enq(t)
    t1 = time.perf_counter()
    e1.record()
    L.pf_sync(f._h)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{'pf_step_async pipelined (device frames)':40s} {1e6 * (t2 - t0) / args.n:8.1f} us/frame  "
          f"(host enqueue {1e6 * (t1 - t0) / args.n:.1f} us/frame, device {1e3 * e0.elapsed_time(e1) / args.n:.1f} "
          f"us/frame)")
    f.reset()
    ref = f.run(host)
    print("pipelined steps == run():", bool(np.array_equal(outs.cpu().numpy(), ref)))


if __name__ == "__main__":
    main()
