"""HSS single-vector solve micro-benchmark (diagnostic): time per hss_solve call on a
config, CTA items vs warp items (env SPD_HSS_CTA read per launch).
usage: python tools/hsolve_bench.py [C2] [n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = synth.CONFIGS[name]
if len(sys.argv) > 2:
    cfg = cfg.scaled(int(sys.argv[2]))
X = torch.tensor(synth.points(cfg), device="cuda")
h = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=3)
b = torch.tensor(synth.rhs(cfg), device="cuda")
xs = {}
for mode in ("warp", "cta", "warp", "cta"):
    if mode == "cta":
        os.environ["SPD_HSS_CTA"] = "1"
    else:
        os.environ.pop("SPD_HSS_CTA", None)
    for _ in range(3):
        x = spd.hss_solve(H, b, layout=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        x = spd.hss_solve(H, b, layout=1)
    e1.record()
    torch.cuda.synchronize()
    xs[mode] = x.clone()
    print(f"{mode}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per solve", flush=True)
print("max |warp - cta| / max|x|:", float((xs["warp"] - xs["cta"]).abs().max() / xs["cta"].abs().max()))
