"""RPY H2 build vs proxy count (diagnostic): time and sampled-row error at N = 4e4 (R1).
usage: python tools/rpy_proxy_probe.py n_proxy [n_proxy ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402
from oracle.kernels import dof_points, rpy_matrix  # noqa: E402  (diagnostic check only)

cfg = synth.R1
X = synth.points(cfg)
D = dof_points(X)
rows = np.random.default_rng(1).choice(cfg.dofs, 200, replace=False)
x = synth.multivec(cfg.dofs, 2)
ref = rpy_matrix(cfg.ell, D[rows], D) @ x
for npx in map(int, sys.argv[1:]):
    torch.cuda.synchronize()
    t0 = time.time()
    h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol, n_proxy=npx)
    torch.cuda.synchronize()
    t1 = time.time()
    xd = torch.tensor(x.T.copy(), device="cuda").t()
    y = spd.h2_matvec(h, xd).cpu().numpy()
    err = np.linalg.norm(y[rows] - ref) / np.linalg.norm(ref)
    print(f"n_proxy {npx}: h2 {t1 - t0:.2f} s, ranks max {h.ranks().max()}, sampled error {err:.2e}", flush=True)
    del h
