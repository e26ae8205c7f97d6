#!/bin/bash
# A/B the fused path across library variants: tools/ab.sh lib1.so lib2.so ...
# (same box only -- boxes differ by up to 5%).  A baseline build of HEAD:
#   git worktree add .wt/base HEAD && make -C .wt/base/paper_2308_00763_b200/csrc \
#     OUT=$PWD/paper_2308_00763_b200/lib/variants/head.so
# then gpurun 'tools/ab.sh paper_2308_00763_b200/lib/variants/head.so paper_2308_00763_b200/lib/libpf_b200.so'
for lib in "$@"; do
  for c in c2 c3; do
    PF_B200_LIB=$lib python bench.py --config $c --no-cpu-baseline --no-extra --steps 5 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$(basename $lib)', '$c', round(d['value']/1e9,2), round(d['e2e']['value']/1e9,2))"
  done
done
