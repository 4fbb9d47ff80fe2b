"""Phase probe (diagnostic, not part of the product): host wall clock and device
events around each public call of one bench step on the C2 workload, repeated.
Usage: python tools/phase_probe.py [--n N] [--reps R]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cfg", default="C2")
args = ap.parse_args()
cfg = synth.CONFIGS[args.cfg]
if args.n:
    cfg = cfg.scaled(args.n)
torch.cuda.set_device(0)
X = torch.tensor(synth.points(cfg), device="cuda")
b = torch.tensor(synth.rhs(cfg), device="cuda")
V = torch.tensor(np.asfortranarray(synth.multivec(cfg.n, 64)).T.copy(), device="cuda").t()
st = torch.cuda.current_stream()


def timed(name, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(st)
    out = fn()
    e1.record(st)
    w1 = time.perf_counter()
    e1.synchronize()
    w2 = time.perf_counter()
    print(f"  {name:14s} dev {e0.elapsed_time(e1):9.2f} ms   host-return {1e3*(w1-w0):9.2f} ms   "
          f"wall {1e3*(w2-w0):9.2f} ms", flush=True)
    return out


for r in range(args.reps):
    print(f"rep {r}", flush=True)
    h = timed("h2_build", lambda: spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol))
    print("   h2 timings", [round(v, 4) for v in h.timings()[:4]], "ranks max", int(h.ranks().max()))
    H = timed("spdhss_build", lambda: spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=1234))
    print("   hss timings", [round(v, 4) for v in H.timings()[:8]])
    out = timed("pcg_solve", lambda: spd.pcg_solve(h, H, b, tol=cfg.pcg_tol, maxit=cfg.maxit))
    print("   pcg", out[1].iters, out[1].relres)
    timed("hss_solve", lambda: spd.hss_solve(H, b))
    timed("h2_matvec k1", lambda: spd.h2_matvec(h, b))
    timed("h2_matvec k64", lambda: spd.h2_matvec(h, V))
    timed("h2_matvec k64b", lambda: spd.h2_matvec(h, V))
    del H, h
    timed("free", lambda: None)
