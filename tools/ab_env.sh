#!/bin/bash
# Same-box A/B of one environment knob: tools/ab_env.sh "VAR=value" [configs] [precisions]
#   e.g. tools/ab_env.sh PF_NO_DRAW_GATE=1 "c2 c3" "fp16-packed fp32 fp64"
knob=$1; cfgs=${2:-c2}; precs=${3:-fp16-packed}
for rep in 1 2; do
  for c in $cfgs; do
    for p in $precs; do
      for arm in base knob; do
        if [ $arm = knob ]; then envs="env $knob"; else envs="env"; fi
        $envs python bench.py --config $c --precision $p --no-cpu-baseline --no-extra --steps 10 2>/dev/null | \
          python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$arm', '$c', '$p', round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,2), 'period_us', round(d['roofline']['avg_launch_ms']*1e3,2))"
      done
    done
  done
done
