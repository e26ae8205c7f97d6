#!/usr/bin/env python
"""Capture per-pipe instruction counts of the product kernels with ncu and
write profiles/ncu_pipes.json (read by bench.py roofline.pipes).

Run on the GPU box (one GPU, never multi-rank):
  python tools/pipes_capture.py [c2 c3] > gpurun_out/pipes_capture.log

For every (config, precision) it profiles `bench.py --profile-only` (one
untimed step) and records, per kernel kind (fused frame kernel, tile table,
likelihood maps), the mean per-launch warp-instruction counts of each pipe
(sm__inst_executed_pipe_*), the total, and the cold serialised duration.
The fused kernel's frame-0 launch (identity ancestors: no resampling) is
excluded from the mean.
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "sm__inst_executed.sum": "total",
    "sm__inst_executed_pipe_fma_type_fp16.sum": "fp16",
    "sm__inst_executed_pipe_fma.sum": "fma",
    "sm__inst_executed_pipe_alu.sum": "alu",
    "sm__inst_executed_pipe_fp64.sum": "fp64",
    "sm__inst_executed_pipe_lsu.sum": "lsu",
    "sm__inst_executed_pipe_xu.sum": "xu",
    "gpu__time_duration.sum": "ns",
}
PRECISIONS = {"c2": ["fp16-packed", "fp16", "fp32", "fp64"], "c3": ["fp16-packed", "fp32", "fp64"]}


def kind(name: str) -> str:
    if "pf_fused_frame" in name:
        return "fused"
    if "pf_tile_table" in name or "pf_shard_" in name:
        return "table"
    if "pf_map" in name:
        return "maps"
    return ""


def capture(config: str, prec: str) -> dict:
    cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "--csv", "-k",
           "regex:pf_fused|pf_tile|pf_map", "--launch-count", "24", sys.executable, os.path.join(ROOT, "bench.py"),
           "--profile-only", "--config", config, "--precision", prec]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout
    rows = [r for r in csv.reader(io.StringIO(out[out.find('"ID"'):]))]
    hdr = rows[0]
    iid, iname, imet, ival = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    launches: dict = {}
    for r in rows[1:]:
        if len(r) < len(hdr) or r[imet] not in METRICS:
            continue
        k = kind(r[iname])
        if not k:
            continue
        d = launches.setdefault(int(r[iid]), {"kind": k, "name": r[iname]})
        d[METRICS[r[imet]]] = float(r[ival].replace(",", ""))
    res: dict = {}
    seen_fused = False
    for lid in sorted(launches):
        d = launches[lid]
        k = d["kind"]
        if k == "fused" and not seen_fused:
            seen_fused = True  # frame 0: identity ancestors
            continue
        acc = res.setdefault(k, {"kernel": d["name"], "n": 0})
        acc["n"] += 1
        for m in METRICS.values():
            acc[m] = acc.get(m, 0.0) + d.get(m, 0.0)
    for k, acc in res.items():
        n = acc.pop("n")
        for m in METRICS.values():
            acc[m] = acc[m] / n
        acc["launches_averaged"] = n
        if k == "maps":
            acc["launches_per_step"] = 1
    return res


def main():
    configs = sys.argv[1:] or ["c2", "c3"]
    path = os.path.join(ROOT, "profiles", "ncu_pipes.json")
    try:
        data = json.load(open(path))
    except Exception:
        data = {"configs": {}}
    for c in configs:
        for p in PRECISIONS[c]:
            t0 = time.time()
            data["configs"].setdefault(c, {})[p] = capture(c, p)
            print(c, p, f"{time.time() - t0:.0f} s", json.dumps(data["configs"][c][p])[:300], flush=True)
    data["how"] = ("ncu --metrics sm__inst_executed[_pipe_*].sum,gpu__time_duration.sum --clock-control none, "
                   "bench.py --profile-only (one untimed step); per-launch means, frame-0 fused launch excluded")
    data["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    os.makedirs(os.path.dirname(path), exist_ok=True)
    json.dump(data, open(path, "w"), indent=1)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(data, open(os.path.join(ROOT, "gpurun_out", "ncu_pipes.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
