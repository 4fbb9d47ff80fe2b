"""C4 PCG probe (diagnostic): which PCG path runs and how much of the symmetric k = 1
store fits.  usage: python tools/c4_probe.py [N]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1048576
cfg = synth.C4.scaled(n)
X = torch.tensor(synth.points(cfg), device="cuda")
h = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=11)
b = torch.tensor(synth.rhs(cfg), device="cuda")
torch.cuda.synchronize()
t0 = time.time()
x, rep = spd.pcg_solve(h, H, b, tol=cfg.pcg_tol, maxit=200)
torch.cuda.synchronize()
t1 = time.time()
print(f"N={n}: store {h.sym_store()} bytes/pieces; {rep.iters} its in {t1 - t0:.2f} s "
      f"({(t1 - t0) / max(1, rep.iters) * 1e3:.2f} ms/it); free {torch.cuda.mem_get_info()[0] / 1e9:.1f} GB", flush=True)
