"""Symmetric k=1 product probe (diagonostic): stored vs evaluated kernel blocks.
usage: SPD_SYM_FRAC=f python tools/sym_probe.py [--cfg C2] [--n N]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402
from bench import prof_table  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C2")
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
cfg = synth.CONFIGS[a.cfg]
if a.n:
    cfg = cfg.scaled(a.n)
X = torch.tensor(synth.points(cfg), device="cuda")
h = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=1)
b = torch.tensor(synth.rhs(cfg), device="cuda")
spd.pcg_solve(h, H, b, tol=cfg.pcg_tol, maxit=2)          # builds the symmetric store
lib = spd.lib()
for r in range(3):
    if r == 2:
        lib.spd_prof_reset()
        lib.spd_prof_enable(1)
    y = spd.h2_matvec(h, b)
    torch.cuda.synchronize()
lib.spd_prof_enable(0)
for k, v in sorted(prof_table(lib).items(), key=lambda kv: -kv[1]["ms"]):
    print(f"   {k:16s} {int(v['launches']):5d} {v['ms']:9.3f} ms  flops {v['flops']:.3e}  bytes {v['bytes']:.3e}")
