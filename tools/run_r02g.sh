# round 2g: constant-base Halton radical inverse in proxy_kernel -- proxies bit-exact (H2 parity suites), bench step
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests/test_gpu_h2.py tests/test_gpu_parity_configs.py tests/test_gpu_rpy.py tests/test_gpu_shard.py -x -q -p no:cacheprovider ) > gpurun_out/g_t.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 2 --minimal > gpurun_out/g_b.log 2>&1
SPD_STAGES=1 timeout 900 python bench.py --steps 1 --warmup 1 --minimal > gpurun_out/g_stages.log 2>&1
exit 0
