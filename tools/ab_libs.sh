#!/bin/bash
# Same-box A/B of library builds: tools/ab_libs.sh "c2 c3" "fp16-packed fp32" lib1.so lib2.so ...
# (build a baseline of HEAD: git worktree add .wt/base HEAD; make -C .wt/base/paper_2308_00763_b200/csrc -j9
#  OUT=$PWD/paper_2308_00763_b200/lib/variants/head.so OBJ=/tmp/obj_head <that OUT>)
cfgs=$1; precs=$2; shift 2
for rep in 1 2; do
  for c in $cfgs; do
    for p in $precs; do
      for lib in "$@"; do
        PF_B200_LIB=$lib python bench.py --config $c --precision $p --no-cpu-baseline --no-extra --steps 10 2>/dev/null | \
          python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$(basename $lib)', '$c', '$p', round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,2), 'period_us', round(d['roofline']['avg_launch_ms']*1e3,2))"
      done
    done
  done
done
