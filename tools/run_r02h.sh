# round 2h: stage marks of the bench step at HEAD and the tensor-map trace of the kblock launches (reduced N)
mkdir -p gpurun_out
SPD_STAGES=1 timeout 900 python bench.py --steps 1 --warmup 1 --minimal > gpurun_out/h_stages.log 2>&1
SPD_KB_TMA_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 1 --minimal --n 131072 > gpurun_out/h_tma.log 2>&1
exit 0
