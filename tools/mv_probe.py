"""H2 multi-vector probe (diagnostic): time h2_matvec of width k on a config recipe,
report useful GFLOP/s (bench.py's F(k)) and the kblock share.
usage: python tools/mv_probe.py [--cfg C2] [--k 64] [--reps 3]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402
from bench import h2_useful_flops, prof_table  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C2")
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
cfg = synth.CONFIGS[a.cfg]
if a.n:
    cfg = cfg.scaled(a.n)
X = torch.tensor(synth.points(cfg), device="cuda")
h = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
V = torch.tensor(np.asfortranarray(synth.multivec(cfg.n, a.k)).T.copy(), device="cuda").t()
fl, counts = h2_useful_flops(h, a.k)
lib = spd.lib()
for r in range(a.reps):
    if r == a.reps - 1:
        lib.spd_prof_reset()
        lib.spd_prof_enable(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    spd.h2_matvec(h, V)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{a.cfg} k={a.k}: {ms:.2f} ms  useful {fl/ms/1e9:.1f} TF/s", flush=True)
lib.spd_prof_enable(0)
for k, v in sorted(prof_table(lib).items(), key=lambda kv: -kv[1]["ms"]):
    print(f"   {k:14s} {int(v['launches']):5d} {v['ms']:9.2f} ms  {v['flops']/max(v['ms'],1e-9)/1e9:7.2f} TF/s")
print("counts", counts)
