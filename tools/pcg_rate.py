"""Diagnostic: PCG time per iteration on a full config (default C4) for the two loop
implementations -- the per-iteration CUDA graph and the persistent kernel with the blocks
the store cannot hold evaluated in the kernel (SPD_PCG_PERSISTENT_EVAL=1).  A bounded
number of iterations each, after a first call that builds the symmetric block store.
python tools/pcg_rate.py [config] [iters]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
its = int(sys.argv[2]) if len(sys.argv) > 2 else 200
X = torch.tensor(synth.points(cfg), device="cuda")
h = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=1234)
b = torch.tensor(synth.rhs(cfg), device="cuda")
t = time.time()
spd.pcg_solve(h, H, b, tol=1e-300, maxit=2)                  # builds the store
torch.cuda.synchronize()
print(f"store build + 2 its: {time.time() - t:.2f} s, store {h.sym_store()[0] / 1e9:.1f} GB", flush=True)
for mode in ["graph", "persistent_eval", "graph", "persistent_eval"]:
    if mode == "persistent_eval":
        os.environ["SPD_PCG_PERSISTENT_EVAL"] = "1"
    else:
        os.environ.pop("SPD_PCG_PERSISTENT_EVAL", None)
    torch.cuda.synchronize()
    t = time.time()
    x, rep = spd.pcg_solve(h, H, b, tol=1e-300, maxit=its)
    torch.cuda.synchronize()
    dt = time.time() - t
    print(f"{mode}: {rep.iters} its in {dt:.2f} s = {1e3 * dt / max(1, rep.iters):.2f} ms/it, relres {rep.relres:.3e}",
          flush=True)
