#!/bin/bash
# round-2f ncu evidence for the TMA-staged kblock (under gpurun, one GPU); the bench step (C4 full build + C5 product):
#  1. the plain run (must exit 0 first)
#  2. duration + DRAM bytes of every kblock launch of the timed step
#  3. one --set full capture of the largest Y^(k) kblock_tma launch (w = 160) of the C4 SPD-HSS build
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --minimal"
$CMD > gpurun_out/r02f_plain.log 2>&1 || exit 0
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none \
    --nvtx --nvtx-include "timed/" -k regex:kblock --csv --log-file gpurun_out/r02f_kblock_launches.csv \
    $CMD > gpurun_out/r02f_ncu_kb.log 2>&1
IDX=$(python - <<'PY'
import csv
rows = [r for r in csv.DictReader(l for l in open("gpurun_out/r02f_kblock_launches.csv") if l.startswith('"'))
        if r["Metric Name"] == "gpu__time_duration.sum" and "kblock_tma_kernel" in r["Kernel Name"]]
best = max(range(len(rows)), key=lambda i: float(rows[i]["Metric Value"].replace(",", ""))) if rows else 0
print(best)
PY
)
echo "longest kblock_tma launch of the timed step: index $IDX" > gpurun_out/r02f_idx.log
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:kblock_tma_kernel \
    -s ${IDX:-0} -c 1 -o gpurun_out/r02f_kblock_tma -f $CMD > gpurun_out/r02f_ncu_kbtma.log 2>&1
exit 0
