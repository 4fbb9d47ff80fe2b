# round 2g: constant-base Halton radical inverse in proxy_kernel + shared-memory panel Cholesky:
# the dense unit tests first, then the whole GPU suite, then the bench step (A/B against the unblocked potrf)
mkdir -p gpurun_out
( time timeout 600 python -m pytest tests/test_gpu_dense.py -x -q -p no:cacheprovider ) > gpurun_out/g_dense.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 2 --minimal > gpurun_out/g_b.log 2>&1
SPD_POTRF_GLOBAL=1 timeout 600 python bench.py --steps 2 --warmup 2 --minimal > gpurun_out/g_b_potrf_global.log 2>&1
( time timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > gpurun_out/g_t.log 2>&1
( time timeout 900 python bench.py --no-pcg ) > gpurun_out/g_bfull.log 2>&1
exit 0
