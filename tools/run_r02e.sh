# round 2e: TMA-staged kblock with padded x^/y^ workspaces -- A/B of the C5 products, parity suites, bench step
mkdir -p gpurun_out
for k in 16 64 256; do
  SPD_STORE_FRAC=0 SPD_KB_TMA=0 timeout 600 python tools/mv_probe.py --cfg C5 --k $k > gpurun_out/j_mv${k}_off.log 2>&1
  SPD_STORE_FRAC=0 SPD_KB_TMA_TRACE=1 timeout 600 python tools/mv_probe.py --cfg C5 --k $k > gpurun_out/j_mv${k}_on.log 2>&1
done
timeout 900 python bench.py --steps 2 --warmup 2 --minimal > gpurun_out/j_b.log 2>&1
SPD_KB_TMA=0 timeout 900 python bench.py --steps 2 --warmup 2 --minimal > gpurun_out/j_b_off.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_h2.py tests/test_gpu_parity_configs.py tests/test_gpu_hss.py tests/test_gpu_shard.py tests/test_gpu_hostcomm.py tests/test_gpu_edge.py -x -q -p no:cacheprovider > gpurun_out/j_t.log 2>&1
exit 0
