"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*.sum --csv):
per kernel: launches, mean/total duration, mean DRAM bytes, share of the step."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    per = defaultdict(dict)
    for r in rows[1:]:
        v = float(r[ix["Metric Value"]].replace(",", ""))
        u = r[ix["Metric Unit"]]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                 "Gbyte": 1e9}.get(u, 1.0)
        per[r[ix["ID"]]]["name"] = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        per[r[ix["ID"]]][r[ix["Metric Name"]]] = v * scale
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        a = agg[d["name"]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"| kernel | launches | mean us | total us | share | mean DRAM bytes |\n|---|---|---|---|---|---|")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t / n:.2f} | {t:.1f} | {100 * t / tot:.1f}% | {b / n:.4g} |")


if __name__ == "__main__":
    main(sys.argv[1])
