import os, sys, subprocess, json
sys.path.insert(0, "/root/repo")
code = r'''
import sys, numpy as np, torch, hashlib
sys.path.insert(0, "/root/repo")
import paper_2011_07632_b200 as spd, synth
cfg = synth.C2
h = spd.h2_build(torch.tensor(synth.points(cfg), device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=3)
b = torch.tensor(synth.rhs(cfg), device="cuda")
x, rep = spd.pcg_solve(h, H, b, tol=cfg.pcg_tol, maxit=cfg.maxit)
print(rep.iters, hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest()[:16])
'''
for env in ({}, {"SPD_PCG_NOFUSE": "1"}):
    e = dict(os.environ); e.update(env)
    print(env, subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True).stdout.strip())
