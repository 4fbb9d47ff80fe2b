set -x
SPD_QR_TRACE=1 python tools/h2_probe.py C4 > gpurun_out/qrtrace.log 2>&1
python bench.py --steps 1 --warmup 1 --minimal > gpurun_out/r02a_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/r02a_launches.csv python bench.py --steps 1 --warmup 1 --minimal > gpurun_out/r02a_ncu_launch.log 2>&1
python tools/h2_probe.py C4 > gpurun_out/h2p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qrcp_kernel -s 14 -c 1 -o gpurun_out/r02a_qrcp -f python tools/h2_probe.py C4 > gpurun_out/r02a_ncu_qrcp.log 2>&1
exit 0
