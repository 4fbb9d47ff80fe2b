"""SPD-HSS build probe (diagnostic): per-kernel-class profile of spdhss_build.
usage: python tools/hss_probe.py [--cfg C4] [--n N]"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402
from bench import prof_table  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C4")
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
cfg = synth.CONFIGS[a.cfg]
if a.n:
    cfg = cfg.scaled(a.n)
X = torch.tensor(synth.points(cfg), device="cuda")
t0 = time.time()
h = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
torch.cuda.synchronize()
print(f"h2_build {time.time() - t0:.2f} s", flush=True)
lib = spd.lib()
lib.spd_prof_reset()
lib.spd_prof_enable(1)
t0 = time.time()
H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=1)
torch.cuda.synchronize()
print(f"spdhss_build {time.time() - t0:.2f} s  timings {[round(x, 3) for x in H.timings()[:4]]}", flush=True)
lib.spd_prof_enable(0)
for k, v in sorted(prof_table(lib).items(), key=lambda kv: -kv[1]["ms"]):
    print(f"   {k:16s} {int(v['launches']):6d} {v['ms']:10.2f} ms  {v['flops'] / max(v['ms'], 1e-9) / 1e9:7.2f} TF/s")
