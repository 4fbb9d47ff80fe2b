# round 2k: flake check of the P = 4 host-comm case (PCG breakdown seen once in run j): 4 repetitions each with the
# panel Cholesky (default) and the unblocked kernel
mkdir -p gpurun_out
for i in 1 2 3 4; do
  timeout 400 python -m pytest "tests/test_gpu_hostcomm.py::test_sharded_build_with_real_exchanges[4-8192-64]" -x -q -p no:cacheprovider > gpurun_out/k_def_$i.log 2>&1; echo "default $i rc=$?" >> gpurun_out/k_summary.log
  SPD_POTRF_GLOBAL=1 timeout 400 python -m pytest "tests/test_gpu_hostcomm.py::test_sharded_build_with_real_exchanges[4-8192-64]" -x -q -p no:cacheprovider > gpurun_out/k_glob_$i.log 2>&1; echo "global $i rc=$?" >> gpurun_out/k_summary.log
done
exit 0
