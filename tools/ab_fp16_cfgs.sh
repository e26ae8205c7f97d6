for rep in 1 2; do
for lib in paper_2308_00763_b200/lib/variants/head.so paper_2308_00763_b200/lib/libpf_b200.so; do
  for cfg in "c2" "c3" "c3 --tpb 128" "c4"; do
    PF_B200_LIB=$lib python bench.py --config $cfg --precision fp16-packed --no-cpu-baseline --no-extra --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$(basename $lib)', '$cfg', round(d['value']/1e9,2))"
  done
done
done
