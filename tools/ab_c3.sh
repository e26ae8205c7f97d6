for lib in "$@"; do
  for i in 1 2; do
  PF_B200_LIB=$lib python /root/repo/bench.py --config c3 --precision fp16-packed --no-cpu-baseline --no-extra --steps 5 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$(basename $lib)', 'c3', round(d['value']/1e9,2))"
  done
done
