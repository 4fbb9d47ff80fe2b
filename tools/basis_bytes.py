import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2011_07632_b200 as spd, synth
cfg = synth.C2
h = spd.h2_build(torch.tensor(synth.points(cfg), device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
r = h.ranks(); nodes = h.nodes(); L = h.levels
tot = 0
for k in range(1, L):
    first, cnt = (1 << (L - k)) - 1, 1 << (L - k)
    b = 0
    for i in range(first, first + cnt):
        s = int(r[i])
        if not s: continue
        nc = int(nodes[i,1]-nodes[i,0]) if k == 1 else int(r[2*i+1] + r[2*i+2])
        b += 8 * s * (nc - s)
    tot += b
    print(f"level {k}: T bytes {b/1e6:.1f} MB, max rank {r[first:first+cnt].max()}")
print("total T MB", tot/1e6)
H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=3)
print("HSS export doubles MB", H.export().size * 8 / 1e6)
