#!/bin/bash
# round-2 (deferred QRCP) ncu evidence (under gpurun, one GPU); the bench step (C4 full build + C5 product):
#  1. the plain run (must exit 0 first)
#  2. every qrcp launch of the timed step: DRAM bytes and duration (traffic of the dominant kernel)
#  3. one --set full capture of a level-3 qrcp launch and of the C5 k=64 kblock launch
#  4. the launch list of the timed step (gpu__time_duration per launch)
set -x
CMD="python bench.py --steps 1 --warmup 1 --minimal"
$CMD > gpurun_out/r02c_plain.log 2>&1 || exit 0
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --nvtx --nvtx-include "timed/" -k regex:qrcp_lazy --csv --log-file gpurun_out/r02c_qrcp_dram.csv \
    $CMD > gpurun_out/r02c_ncu_dram.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:qrcp_lazy \
    -s 20 -c 1 -o gpurun_out/r02c_qrcp -f $CMD > gpurun_out/r02c_ncu_qrcp.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:kblock_kernel \
    -s 20 -c 1 -o gpurun_out/r02c_kblock -f $CMD > gpurun_out/r02c_ncu_kblock.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/r02c_launches.csv $CMD > gpurun_out/r02c_ncu_launch.log 2>&1
exit 0
