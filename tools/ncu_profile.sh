#!/bin/bash
# ncu evidence for profiles/ (run under gpurun, one GPU):
#  1. the bench command once without ncu (must exit 0 first),
#  2. the launch list of the timed step (NVTX range "timed"), gpu__time_duration per launch,
#  3. one `--set full` capture per listed kernel regex (first matching launch after -s skips).
# usage: tools/ncu_profile.sh <tag> <regex>[:skip] ...
set -euo pipefail
tag=$1; shift
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/${tag}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/${tag}_launches.csv $CMD > gpurun_out/${tag}_ncu_launch.log 2>&1
for spec in "$@"; do
  rx=${spec%%:*}; skip=0
  [[ "$spec" == *:* ]] && skip=${spec##*:}
  name=$(echo "$rx" | tr -c 'a-zA-Z0-9_' '_')
  ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:"$rx" -s $skip -c 1 \
      -o gpurun_out/${tag}_${name} -f $CMD > gpurun_out/${tag}_ncu_${name}.log 2>&1 || echo "ncu full $rx failed"
done
echo ncu_profile done
