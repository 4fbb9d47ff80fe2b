# round 2l: default path after making the panel Cholesky opt-in -- dense unit tests and the host-comm cases
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dense.py tests/test_gpu_hostcomm.py tests/test_gpu_hss.py -x -q -p no:cacheprovider > gpurun_out/l_t.log 2>&1
exit 0
