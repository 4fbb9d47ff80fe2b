"""Diagnostic: C4 (or another config) H2 build timings, one line per run; stage marks
with SPD_STAGES=1.  python tools/h2_probe.py [config] [n]"""
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
    print(f"rep {rep} {cfg.name} N={cfg.n} h2_build {time.time() - t:.3f} s, timings {np.round(h.timings()[:2], 3)}, "
          f"max rank {h.ranks().max()}, env L2MB={os.environ.get('SPD_QRCP_L2MB')}", flush=True)
    del h
