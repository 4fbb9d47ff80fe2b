# round 2d: TMA-staged kblock -- parity suites, then A/B of the C5 products and the bench step
mkdir -p gpurun_out
SPD_KB_TMA_TRACE=1 timeout 1500 python -m pytest tests/test_gpu_h2.py tests/test_gpu_parity_configs.py tests/test_gpu_hss.py -x -q -p no:cacheprovider > gpurun_out/d_t.log 2>&1
grep -c "TMA-staged" gpurun_out/d_t.log >> gpurun_out/d_t.log
for k in 16 64 256; do
  SPD_STORE_FRAC=0 SPD_KB_TMA=0 timeout 600 python tools/mv_probe.py --cfg C5 --k $k > gpurun_out/d_mv${k}_off.log 2>&1
  SPD_STORE_FRAC=0 SPD_KB_TMA_TRACE=1 timeout 600 python tools/mv_probe.py --cfg C5 --k $k > gpurun_out/d_mv${k}_on.log 2>&1
done
timeout 900 python bench.py --steps 2 --warmup 2 --minimal > gpurun_out/d_b.log 2>&1
exit 0
