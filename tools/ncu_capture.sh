#!/bin/bash
# ncu --set full capture of one kernel launch, summarised ON the GPU box (the
# .ncu-rep of this 12 MB library is ~40 MB; gpurun copies back <= 64 MiB):
#   tools/ncu_capture.sh <name> <kernel-regex> <launch-skip> <bench args...>
# writes gpurun_out/<name>.md (tools/ncu_summary.py) and gpurun_out/<name>_lines.txt
# (tools/ncu_lines.py); keeps the report only with KEEP_REP=1.
name=$1; kre=$2; skip=$3; shift 3
mkdir -p gpurun_out /tmp/ncu
timeout 400 ncu -k "regex:$kre" --launch-skip "$skip" --launch-count 1 --set full --import-source on \
  --clock-control none -f -o /tmp/ncu/$name python bench.py --profile-only "$@" > gpurun_out/$name.log 2>&1
python tools/ncu_summary.py /tmp/ncu/$name.ncu-rep "$name" > gpurun_out/$name.md 2>&1
python tools/ncu_lines.py /tmp/ncu/$name.ncu-rep ${NLINES:-60} > gpurun_out/${name}_lines.txt 2>&1
if [ "$KEEP_REP" = 1 ]; then cp /tmp/ncu/$name.ncu-rep gpurun_out/; fi
