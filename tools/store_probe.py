"""Diagnostic: the symmetric k = 1 block store of a full-size H2 (C4 or C5): free memory,
store size and k = 1 product time."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
h = spd.h2_build(torch.tensor(synth.points(cfg), device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
print("after build: free %.1f GB (torch reserved %.1f GB)" % (torch.cuda.mem_get_info()[0] / 1e9,
                                                               torch.cuda.memory_reserved() / 1e9), flush=True)
x = torch.randn(cfg.n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t = time.time()
_, rep_ = spd.pcg_solve(h, None, x, tol=1e-30, maxit=20)      # PCG builds the k = 1 store
torch.cuda.synchronize()
print(f"unpreconditioned CG, 20 iterations: {time.time() - t:.2f} s (incl. store build), store {h.sym_store()}, "
      f"free {torch.cuda.mem_get_info()[0] / 1e9:.1f} GB", flush=True)
torch.cuda.synchronize()
t = time.time()
_, rep_ = spd.pcg_solve(h, None, x, tol=1e-30, maxit=20)
torch.cuda.synchronize()
print(f"again: {1e3 * (time.time() - t) / 20:.2f} ms per iteration", flush=True)
for rep in range(3):
    torch.cuda.synchronize()
    t = time.time()
    spd.h2_matvec(h, x)
    torch.cuda.synchronize()
    print(f"k=1 product {1e3 * (time.time() - t):.1f} ms, store {h.sym_store()}, free "
          f"{torch.cuda.mem_get_info()[0] / 1e9:.1f} GB", flush=True)
