import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2308_00763_b200 as pf
from oracle import reference_port as rp
frames, _ = rp.generate_video(rp.Params(), 6, 128, 128, (64.0, 64.0), 42)
for mode in ("fp64", "fp32", "fp16", "fp16-packed"):
    f = pf.Filter(5000 if mode != "fp16-packed" else 5000, mode, 128, 128, 42)
    a = f.run(frames)
    f.reset()
    b = np.array([f.step(frames[t]) for t in range(6)])
    assert np.array_equal(a, b), mode
    f.close()
f = pf.Filter(3001, "fp32", 128, 128, 42, n_tracks=3)
f.run_frames(np.stack([frames]), 6)
f.close()
print("sanitizer run ok")
