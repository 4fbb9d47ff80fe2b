#!/bin/bash
# round-2f: the P = 8 host-comm test, then the ncu launch list of one timed bench step at HEAD
# (gpu__time_duration per launch, NVTX range "timed"; the plain run of the same command exited 0 in prof_r02f.sh)
mkdir -p gpurun_out
( time timeout 1200 python -m pytest tests/test_gpu_hostcomm.py -x -q -p no:cacheprovider -s ) > gpurun_out/f_hostcomm.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --minimal"
timeout 2700 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/r02f_launches.csv $CMD > gpurun_out/r02f_ncu_launch.log 2>&1
exit 0
