#!/bin/bash
# C2 FP16 / FP32 A/B of library builds (same box): tools/ab_c2.sh lib1.so lib2.so ...
for lib in "$@"; do
  for p in fp16-packed fp32; do
    PF_B200_LIB=$lib python /root/repo/bench.py --config c2 --precision $p --no-cpu-baseline --no-extra --steps 10 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$(basename $lib)', 'c2', '$p', round(d['value']/1e9,2))"
  done
done
