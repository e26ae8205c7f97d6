#!/bin/bash
# Same-box A/B, interleaved: tools/ab_pair.sh CONFIGS PRECISION libA.so libB.so ...
#   e.g. tools/ab_pair.sh "c2 c3" fp16-packed lib/variants/head.so lib/libpf_b200.so
CFGS=$1; PREC=$2; shift 2
for i in 1 2; do
  for c in $CFGS; do
    for lib in "$@"; do
      PF_B200_LIB=$lib python bench.py --config $c --precision $PREC --no-cpu-baseline --no-extra --steps 5 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$(basename $lib)', '$c', '$PREC', round(d['value']/1e9,2), 'period_us', round(d['roofline']['avg_launch_ms']*1e3,2))"
    done
  done
done
