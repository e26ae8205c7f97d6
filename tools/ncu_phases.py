"""Aggregate a tools/ncu_lines.py listing (top N lines, N large) into the
fused kernel's phases by pf_kernels.cuh line ranges (edit RANGES to the
current source).  python tools/ncu_phases.py gpurun_out/<name>_lines.txt"""
import re
import sys

RANGES = [  # (first, last, phase) on pf_kernels.cuh
    (1120, 1223, "setup"), (1224, 1313, "draws"), (1314, 1439, "window"), (1440, 1540, "search"),
    (1541, 1613, "gather/prop/lookup"), (1614, 1628, "tile max"), (1629, 1705, "weights/scan/moments"),
    (1706, 1761, "prefix/cdf/store"), (1762, 1800, "record"),
    (1019, 1045, "search"), (913, 938, "search"), (886, 912, "search"), (615, 631, "search"),
    (1046, 1083, "draws"), (947, 991, "gather/prop/lookup"), (774, 788, "gather/prop/lookup"),
    (829, 873, "weights/scan/moments"), (939, 946, "tile max"), (1084, 1104, "weights/scan/moments"),
    (711, 743, "weights/scan/moments"), (60, 80, "weights/scan/moments"),
]
FILEMAP = {"pf_rng.cuh": "draws", "cuda_fp16.hpp": "fp16 intrinsics", "sm_30_intrinsics.hpp": "shuffles",
           "sm_32_intrinsics.hpp": "ldg/funnelshift", "device_atomic_functions.hpp": "atomics", "pf_math.cuh": "math"}
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
        for a, b, p in RANGES:
            if a <= ln <= b:
                ph = p
                break
    tot[ph] = tot.get(ph, 0.0) + pct
for ph, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{ph:24s} {v:6.1f}%")
print(f"{'sum':24s} {sum(tot.values()):6.1f}%   (thread inst {total_thread:.3g})")
