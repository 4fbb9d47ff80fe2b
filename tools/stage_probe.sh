# per-stage wall times (SPD_STAGES=1, synchronizing) of the C4 H2 + SPD-HSS builds
SPD_STAGES=1 python - <<'PY' > gpurun_out/stages.log 2>&1
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_2011_07632_b200 as spd, synth
c = synth.C4
X = torch.tensor(synth.points(c), device="cuda")
for rep in range(2):
    print("rep", rep, flush=True)
    h = spd.h2_build(X, c.kernel, c.ell, c.shift, c.leaf, c.h2_tol)
    H = spd.spdhss_build(h, c.rank_cap, c.hss_tol, c.oversample, seed=1234)
    torch.cuda.synchronize()
    del H, h
PY
