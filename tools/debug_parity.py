"""Locate the first fused-path divergence from oracle/fused.py (GPU debug aid)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2308_00763_b200 as pf  # noqa: E402
from oracle import fused  # noqa: E402
from oracle import reference_port as rp  # noqa: E402


def main(K=40961, mode="fp16", frames=6, tpb=256, W=96, H=80, seed=5, start=(40.0, 30.0), vseed=17):
    vid, _ = rp.generate_video(rp.Params(), frames, W, H, start, vseed)
    f = pf.Filter(K, mode, W, H, seed, start_hint=start, tpb=tpb)
    f.enable_debug()
    tr = fused.FusedTrack(mode, K, W, H, seed, start)
    for t in range(frames):
        est = f.step(vid[t])
        ref = tr.step(tr.loglik_map(vid[t]))
        anc, L = f.debug()
        bad_a = np.nonzero(anc != tr.last_ancestors)[0]
        bad_l = np.nonzero(L.view(np.uint8 if L.dtype == np.uint8 else L.dtype) != tr.last_loglik)[0]
        xs, ys, c = f.state()
        bad_c = np.nonzero(c.view(np.uint16 if c.dtype == np.float16 else c.dtype) !=
                           tr.c.astype(c.dtype).view(np.uint16 if c.dtype == np.float16 else c.dtype))[0]
        print(f"t={t} est={est} ref={ref} anc_bad={len(bad_a)} L_bad={len(bad_l)} c_bad={len(bad_c)}")
        if len(bad_l):
            for k in bad_l[:4]:
                print("  L mismatch k", k, "x,y dev", xs[k], ys[k], "ref", tr.xs[k], tr.ys[k],
                      "L dev", L[k], "ref", tr.last_loglik[k], "anc", anc[k], tr.last_ancestors[k])
        if len(bad_a):
            k = bad_a[0]
            s, O, iM = tr.table_prev if hasattr(tr, "table_prev") else (None, None, None)
            print("  first bad k", k, "dev", anc[k], "ref", tr.last_ancestors[k], "tile", k // 1024,
                  "bad tiles", np.unique(bad_a // 1024)[:20])
        if len(bad_c):
            print("  first bad c", bad_c[:10], c[bad_c[:5]], tr.c[bad_c[:5]])
        if len(bad_a) or len(bad_l) or len(bad_c) or est != ref:
            break


if __name__ == "__main__":
    args = [int(a) if a.isdigit() else a for a in sys.argv[1:]]
    main(*args)
