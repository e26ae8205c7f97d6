#!/bin/bash
# A/B over precisions: tools/ab_all.sh lib1.so lib2.so ...
for lib in "$@"; do
  for c in "c2 fp16-packed" "c2 fp32" "c2 fp64" "c3 fp16-packed" "c3 fp32" "c3 fp64"; do
    set -- $c
    PF_B200_LIB=$lib python /root/repo/bench.py --config $1 --precision $2 --no-cpu-baseline --no-extra --steps 5 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$(basename $lib)', '$1', '$2', round(d['value']/1e9,2))"
  done
done
