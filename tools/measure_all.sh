#!/bin/bash
# One B200: every BASELINE config that fits one GPU, all precisions, C3 TPB sweep.
# Writes gpurun_out/measure_all.jsonl (one bench JSON line per run) and prints a table.
out=gpurun_out/measure_all.jsonl
: > $out
run() { python bench.py --no-cpu-baseline --no-extra "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); d['args']='$*'; print(json.dumps(d))" >> $out; }
run --config c1 --precision fp64 --steps 20
for p in fp16-packed fp16 fp32 fp64; do run --config c2 --precision $p; done
for p in fp16-packed fp16 fp32 fp64; do run --config c3 --precision $p --steps 5; done
for t in 32 64 128 256 512 1024; do run --config c3 --tpb $t --steps 5; done
run --config c4 --steps 3
run --config c5 --steps 3
python - <<'PY'
import json
for l in open("gpurun_out/measure_all.jsonl"):
    d = json.loads(l)
    r = d.get("roofline") or {}
    print(f"{d['args']:40s} {d['value']/1e9:8.2f} G/s  e2e {d['e2e']['value']/1e9:8.2f}  ms/step {d['ms_per_step']:9.3f}  "
          f"frac {r.get('frac', float('nan')):.3f}  err {d['tracking']['mean_err_px']:.3f}")
PY
