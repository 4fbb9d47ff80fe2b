"""Diagnostic: per-level QRCP shapes of the C4 H2 build (node count, candidates n_c,
ranks) and its stage marks (run with SPD_STAGES=1 SPD_QR_TRACE=1).
python tools/qrcp_probe.py [config] [n]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
if len(sys.argv) > 2:
    cfg = cfg.scaled(int(sys.argv[2]))
X = torch.tensor(synth.points(cfg), device="cuda")
for rep in range(2):
    torch.cuda.synchronize()
    t = time.time()
    h = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    torch.cuda.synchronize()
    print(f"rep {rep} {cfg.name} N={cfg.n} h2_build {time.time() - t:.3f} s", flush=True)
r = h.ranks()
nn = len(r)
L = int(np.log2(nn + 1))
tot = 0.0
for lev in range(1, L + 1):          # level 1 = leaves (heap numbering: depth L - lev)
    dep = L - lev
    ids = np.arange(2 ** dep - 1, 2 ** (dep + 1) - 1)
    if lev == 1:
        nc = np.full(len(ids), cfg.leaf)
    else:
        nc = r[2 * ids + 1] + r[2 * ids + 2]
    s = r[ids]
    # recomputed-norm QRCP entries touched: sum_t (nc - t)^2, t <= s
    ent = sum(float(((c - np.arange(0, min(k + 1, c))) ** 2).sum()) for c, k in zip(nc, s))
    tot += ent
    print(f"level {lev}: nodes {len(ids)}, n_c mean {nc.mean():.0f} max {nc.max()}, rank mean {s.mean():.0f} max {s.max()}, "
          f"qrcp entries {ent:.3e} ({8 * ent / 1e9:.1f} GB per pass)", flush=True)
print(f"total qrcp trailing entries {tot:.3e}: {8 * tot / 1e9:.0f} GB read once per step")
