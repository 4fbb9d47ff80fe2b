"""Diagnostic: one h2_matvec of a test case through the TMA-staged kblock, checked against
the oracle.  python tools/tma_dbg.py <case> <k>"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402

from dataclasses import replace  # noqa: E402
cases = {"ragged": synth.C1.scaled(1000, leaf=50), "C1": synth.C1, "C2s": synth.C2.scaled(4096, leaf=64)}
cases["g3"] = replace(cases["C2s"], kernel=synth.C1.kernel, ell=0.2)
cases["m2"] = replace(synth.C1, kernel=synth.C2.kernel, ell=0.2)
cfg = cases[sys.argv[1]]
k = int(sys.argv[2])
X = synth.points(cfg)
h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
x = synth.multivec(cfg.n, k)
xt = torch.tensor(np.asfortranarray(x).T.copy(), device="cuda").t()
y = spd.h2_matvec(h, xt).cpu().numpy()
ho = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
perm = ho.tree.perm
yo = np.empty_like(x)
yo[perm] = oracle.h2_matvec(ho, x[perm])
print(sys.argv[1:], "rel err", np.linalg.norm(y - yo) / np.linalg.norm(yo), flush=True)
