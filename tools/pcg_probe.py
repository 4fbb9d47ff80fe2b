"""PCG probe (diagnostic): iterations to 1e-8 for a config recipe at several N, with the
SPD-HSS preconditioner and, for comparison, unpreconditioned CG (both capped at maxit).
usage: python tools/pcg_probe.py C4 65536 262144 [--maxit 20000] [--cap 150]"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("ns", type=int, nargs="+")
ap.add_argument("--maxit", type=int, default=20000)
ap.add_argument("--cap", type=int, default=0)
ap.add_argument("--noprec", action="store_true")
a = ap.parse_args()
for n in a.ns:
    cfg = synth.CONFIGS[a.cfg].scaled(n)
    if a.cap:
        cfg = cfg.scaled(n, rank_cap=a.cap)
    X = torch.tensor(synth.points(cfg), device="cuda")
    t0 = time.time()
    h = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    torch.cuda.synchronize()
    t1 = time.time()
    H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=11)
    torch.cuda.synchronize()
    t2 = time.time()
    b = torch.tensor(synth.rhs(cfg), device="cuda")
    x, rep = spd.pcg_solve(h, H, b, tol=cfg.pcg_tol, maxit=a.maxit)
    t3 = time.time()
    print(f"{a.cfg} N={n} cap={cfg.rank_cap}: h2 {t1-t0:.1f}s (rank max {h.ranks().max()}), hss {t2-t1:.1f}s, "
          f"PCG {rep.iters} its relres {rep.relres:.2e} conv {rep.converged} in {t3-t2:.1f}s", flush=True)
    if a.noprec:
        x, rep = spd.pcg_solve(h, None, b, tol=cfg.pcg_tol, maxit=min(a.maxit, 3000))
        print(f"   unpreconditioned: {rep.iters} its relres {rep.relres:.2e}", flush=True)
    del H, h
