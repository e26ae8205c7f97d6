#!/bin/bash
# Pipe mix of the FP16 kernels, scalar ("fp16") vs packed ("fp16-packed"): the
# naive-vs-optimised pair.  Usage: tools/pipes.sh c3 > out.csv
CFG=${1:-c3}
M=gpu__time_duration.sum,sm__inst_executed.sum,sm__inst_executed_pipe_fma_type_fp16.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_xu.sum
for p in fp16 fp16-packed; do
  ncu --metrics $M --clock-control none --csv -k regex:"pf_map|pf_fused" --launch-count 4 \
    python bench.py --profile-only --config $CFG --precision $p 2>/dev/null | grep -E "pf_map|pf_fused" | \
    awk -v p=$p -F'","' '{print p "," $5 "," $(NF-2) "," $NF}' | tr -d '"'
done
