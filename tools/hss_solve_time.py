"""Time the standalone single-vector hss_solve (diagnostic).  usage: python tools/hss_solve_time.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402

cfg = synth.C2
h = spd.h2_build(torch.tensor(synth.points(cfg), device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=3)
b = torch.tensor(synth.rhs(cfg), device="cuda")
for _ in range(3):
    x = spd.hss_solve(H, b, layout=1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    x = spd.hss_solve(H, b, layout=1)
e1.record()
torch.cuda.synchronize()
print(f"hss_solve k=1: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us; sum {float(x.sum()):.15e}")
