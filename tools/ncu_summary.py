"""Summarise an ncu report (.ncu-rep) into a small markdown block for profiles/."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Executed Instructions", "Registers Per Thread", "Block Size", "Grid Size",
        "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block",
        "Waves Per SM", "Avg. Active Threads Per Warp"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    hdr = next(r)
    rows = [dict(zip(hdr, row)) for row in r]
    got = {}
    for d in rows:
        name = d.get("Metric Name", "")
        if name in KEYS and name not in got:
            got[name] = (d.get("Metric Value", ""), d.get("Metric Unit", ""))
    kernel = rows[0].get("Kernel Name", "") if rows else ""
    return kernel, got


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    return {k: (v, u) for k, u, v in zip(rows[0], rows[1], rows[2])}


def main(rep, title):
    kernel, got = details(rep)
    d = raw(rep)
    print(f"### {title}\n\n`{rep}` — kernel `{kernel}`\n")
    print("| metric | value |\n|---|---|")
    for k in KEYS:
        if k in got:
            print(f"| {k} | {got[k][0]} {got[k][1]} |")
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in d:
            print(f"| {k} | {d[k][0]} {d[k][1]} |")
    stalls = []
    for k, (v, _) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    top = ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:5])
    print(f"| top stalls (cycles/issued instr) | {top} |\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
