python tools/gemm_bench.py > gpurun_out/c_gemm.log 2>&1
python tools/h2_probe.py C4 > gpurun_out/c_h2.log 2>&1
python tools/mv_probe.py --cfg C5 --k 64 > gpurun_out/c_mv64.log 2>&1
python tools/mv_probe.py --cfg C5 --k 256 > gpurun_out/c_mv256.log 2>&1
python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_h2.py tests/test_gpu_dense.py -x -q 2>&1 | tail -4 > gpurun_out/c_t.log
python bench.py --steps 2 --warmup 2 --minimal > gpurun_out/c_b.log 2>&1
exit 0
