"""Per-source-line breakdown of one kernel in an ncu report (--import-source on).

  python tools/ncu_lines.py report.ncu-rep [top_n]

Aggregates the cuda,sass source page per CUDA line: warp instructions
executed, thread instructions, stall samples.  Prints the top lines by thread
instructions and by stall samples, plus per-line-range totals.
"""
import csv
import io
import subprocess
import sys


def _int(v):
    try:
        return int(v)
    except (TypeError, ValueError):
        return 0


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    cur = None
    agg = {}
    fname = ""
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0]:
            cur = (fname, int(r[0]), r[1].strip()[:90])
            continue
        if cur is None:
            continue
        d = dict(zip(hdr[2:], r[2:]))
        a = agg.setdefault(cur, [0, 0, 0, 0])
        a[0] += _int(d.get("Instructions Executed"))
        a[1] += _int(d.get("Thread Instructions Executed"))
        a[2] += _int(d.get("Warp Stall Sampling (All Samples)"))
        a[3] += 1
    tot = [sum(v[i] for v in agg.values()) for i in range(3)]
    print(f"total warp inst {tot[0]}, thread inst {tot[1]}, stall samples {tot[2]}")
    print("\n-- top by thread instructions --")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k[0]}:{k[1]:5d} {100*v[1]/max(tot[1],1):5.1f}%i {100*v[2]/max(tot[2],1):5.1f}%s sass={v[3]:3d} | {k[2]}")
    print("\n-- top by stall samples --")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
        print(f"{k[0]}:{k[1]:5d} {100*v[1]/max(tot[1],1):5.1f}%i {100*v[2]/max(tot[2],1):5.1f}%s sass={v[3]:3d} | {k[2]}")


if __name__ == "__main__":
    main()
