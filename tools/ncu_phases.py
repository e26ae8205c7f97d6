"""Aggregate a tools/ncu_lines.py listing (top N lines, N large) into the
fused kernel's phases.  Phase boundaries are found from marker comments and
helper-function names in the CURRENT paper_2308_00763_b200/csrc/pf_kernels.cuh,
so the listing must come from a capture of this source.

  python tools/ncu_phases.py gpurun_out/<name>_lines.txt"""
import os
import re
import sys

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2308_00763_b200", "csrc",
                   "pf_kernels.cuh")


def ranges():
    lines = open(SRC).read().split("\n")

    def find(pat, start=0):
        for i in range(start, len(lines)):
            if re.search(pat, lines[i]):
                return i + 1
        raise SystemExit(f"marker not found: {pat}")

    k0 = find(r"pf_fused_frame\(FusedArgs a\) \{")
    draws = find(r"one particle's pair of normals|---- phase 0", k0)
    window = find(r"---- warp 0: wait for the previous kernels", k0)
    p1 = find(r"---- phase 1: resample", k0)
    gather = find(r"all VPT ancestor gathers first", p1)
    tmax = find(r"tile max \(exact\)", p1)
    p2 = find(r"---- phase 2: weights", p1)
    pref = find(r"prefix of this thread's segment", p2)
    rec = find(r"// tile record", p2)
    end = find(r"^}", rec)
    out = [(k0, draws - 1, "setup"), (draws, window - 1, "draws"), (window, p1 - 1, "window"), (p1, gather - 1, "search"),
           (gather, tmax - 1, "gather/prop/lookup"), (tmax, p2 - 1, "tile max"), (p2, pref - 1, "weights/scan/moments"),
           (pref, rec - 1, "prefix/cdf/store"), (rec, end, "record")]

    def func(name, phase):  # every definition of a helper (incl. specialisations): signature .. closing brace
        found = False
        for i, l in enumerate(lines):
            if "__device__" in l and re.search(r"\b" + name + r"\b\s*(<[^>]*>)?\s*\(", l) and not l.rstrip().endswith(";"):
                j = find(r"^}", i + 1)
                out.append((i + 1, j, phase))
                found = True
        if not found:
            raise SystemExit(name)

    for n, ph in [("lb_key", "search"), ("gallop_key", "search"), ("lb_branchless", "search"), ("lb_first", "search"),
                  ("advance_key", "search"), ("point_of", "search"), ("set_comp", "draws"), ("scale_noise", "draws"),
                  ("prop", "gather/prop/lookup"), ("prop_scalar", "gather/prop/lookup"), ("round_clamp", "gather/prop/lookup"),
                  ("weight_q", "weights/scan/moments"), ("exp16_fast", "weights/scan/moments"),
                  ("tree_vpt", "weights/scan/moments"), ("gt_real", "tile max"), ("hadd_s", "fp16 scalar ops"),
                  ("hmul_s", "fp16 scalar ops"), ("hsub_s", "fp16 scalar ops")]:
        try:
            func(n, ph)
        except SystemExit:
            pass
    return out


FILEMAP = {"pf_rng.cuh": "draws", "cuda_fp16.hpp": "fp16 intrinsics", "sm_30_intrinsics.hpp": "shuffles",
           "sm_32_intrinsics.hpp": "ldg/funnelshift", "device_atomic_functions.hpp": "atomics", "pf_math.cuh": "math"}


def main():
    R = ranges()
    tot = {}
    head = open(sys.argv[1]).readline()
    total_thread = float(re.search(r"thread inst (\d+)", head).group(1))
    seen = set()
    for line in open(sys.argv[1]):
        m = re.match(r"(\S+):\s*(\d+)\s+([\d.]+)%i", line)
        if not m or (m.group(1), m.group(2)) in seen:
            continue
        seen.add((m.group(1), m.group(2)))
        f, ln, pct = m.group(1), int(m.group(2)), float(m.group(3))
        ph = FILEMAP.get(f, "other")
        if f == "pf_kernels.cuh":
            ph = "other kernels.cuh"
            best = None
            for a, b, p in R:  # innermost (shortest) matching range
                if a <= ln <= b and (best is None or b - a < best[1] - best[0]):
                    best = (a, b, p)
            if best:
                ph = best[2]
        tot[ph] = tot.get(ph, 0.0) + pct
    for ph, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{ph:24s} {v:6.1f}%")
    print(f"{'sum':24s} {sum(tot.values()):6.1f}%   (thread inst {total_thread:.3g})")


if __name__ == "__main__":
    main()
