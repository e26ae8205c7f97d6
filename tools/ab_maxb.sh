for rep in 1 2; do
for mb in 0 6 7 8 9; do
  for p in fp16-packed fp32; do
    PF_FUSED_MAXB=$mb python bench.py --config c2 --precision $p --no-cpu-baseline --no-extra --steps 10 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('maxb $mb', '$p', round(d['value']/1e9,2), 'period_us', round(d['roofline']['avg_launch_ms']*1e3,2))"
  done
done
done
