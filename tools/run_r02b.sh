python tools/h2_probe.py C4 > gpurun_out/r02b_np2.log 2>&1
SPD_QR_NP=4 python tools/h2_probe.py C4 > gpurun_out/r02b_np4.log 2>&1
SPD_QR_NP=3 python tools/h2_probe.py C4 > gpurun_out/r02b_np3.log 2>&1
python -m pytest tests/test_gpu_h2.py tests/test_gpu_parity_configs.py -x -q 2>&1 | tail -5 > gpurun_out/r02b_t.log
SPD_QR_NP=4 python -m pytest tests/test_gpu_parity_configs.py -x -q -k "C4p or C5p or C2p" 2>&1 | tail -5 > gpurun_out/r02b_t4.log
exit 0
