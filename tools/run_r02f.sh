# round 2f: end-of-round verification -- the whole GPU suite, smoke, the default bench line, the reference arm
mkdir -p gpurun_out
( time timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > gpurun_out/f_t.log 2>&1
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/f_smoke.log 2>&1
( time timeout 1200 python bench.py ) > gpurun_out/f_b.log 2>&1
( time timeout 900 python bench.py --impl reference ) > gpurun_out/f_ref.log 2>&1
exit 0
