import sys, os, numpy as np, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2308_00763_b200 as pf
v = pf.generate_video(pf.ModelParams(), 30, 128, 128, (64.0, 64.0), 42)
host = np.ascontiguousarray(v.frames)
dev = torch.from_numpy(host).cuda()
for K in (1_000_000, 10_000):
    f = pf.Filter(K, "fp16-packed", 128, 128, 42)
    f.set_profiling(True)
    for t in range(10):
        f.step(dev[t])
    acc = {}
    for t in range(10, 30):
        f.step(dev[t])
        for k, x in f.timings().items():
            acc[k] = acc.get(k, 0) + x / 20
    print(K, "profiled step (ms):", {k: round(x, 4) for k, x in acc.items()})
    f.set_profiling(False)
    f.close()
