# round 2j: final verification at HEAD -- whole GPU suite, smoke, default bench line (without the 150 s C4 PCG)
mkdir -p gpurun_out
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/j_smoke.log 2>&1
( time timeout 900 python bench.py --no-pcg ) > gpurun_out/j_b.log 2>&1
( time timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > gpurun_out/j_t.log 2>&1
exit 0
