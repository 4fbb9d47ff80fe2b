"""C5 multi-vector sweep at full size (diagnostic): useful TF/s per k with kernel blocks
evaluated on the fly (SPD_STORE_FRAC=0), then again after the PCG path built the symmetric store.
usage: python tools/c5_sweep.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402
from bench import h2_useful_flops  # noqa: E402

cfg = synth.C5
h = spd.h2_build(torch.tensor(synth.points(cfg), device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)


def sweep(tag):
    for k in (16, 64, 256):
        V = torch.tensor(np.random.default_rng(k).standard_normal((k, cfg.n)), device="cuda").t()
        spd.h2_matvec(h, V)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        spd.h2_matvec(h, V)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        fl = h2_useful_flops(h, k)[0]
        print(f"{tag} k={k}: {ms:.1f} ms, useful {fl / ms / 1e9:.1f} TF/s", flush=True)
        del V


os.environ["SPD_STORE_FRAC"] = "0"         # the evaluated pass never builds a store
sweep("evaluated")
os.environ["SPD_STORE_FRAC"] = "0.25"
b = torch.tensor(np.random.default_rng(0).standard_normal(cfg.n), device="cuda")
spd.pcg_solve(h, None, b, tol=1e-300, maxit=1)   # the PCG path builds the symmetric k = 1 store
torch.cuda.synchronize()
print("store", h.sym_store(), flush=True)
sweep("stored")
