# round 2i: mostly-unaddressable kblock launches fall back to the register-staged kernel -- A/B of the bench step, HSS parity suites
mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 2 --minimal > gpurun_out/i_b.log 2>&1
SPD_KB_TMA_MINSHARE=0 timeout 600 python bench.py --steps 2 --warmup 2 --minimal > gpurun_out/i_b_mix.log 2>&1
( time timeout 1200 python -m pytest tests/test_gpu_hss.py tests/test_gpu_parity_configs.py tests/test_gpu_h2.py tests/test_gpu_edge.py -x -q -p no:cacheprovider ) > gpurun_out/i_t.log 2>&1
exit 0
