#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the SPD-HSS-from-H2 hot path.

One STEP = one pass of the whole hot path of arXiv 2011.07632 on BASELINE.json
configs[1] (C2: N=32768 points uniform in [0,1]^3, Matern-3/2 l=0.2 + 1e-4 I,
leaf 128, H2 tol 1e-10, HSS cap 100 / tol 1e-3, p = 10, PCG to 1e-8):
    h2_build -> spdhss_build (Alg. 4) -> pcg_solve (H2 matvec + HSS solve)
    -> one H2 multi-vector product of width 64 (the "H2 multi-vector GFLOP/s" line)
`value` = seconds per step (max over ranks), lower is better.  Inputs are
resident in HBM when the timed region starts; L2 (126 MB) is flushed between
steps by writing a 256 MB buffer.  Multi-GPU (torchrun): independent replicas,
weak scaling; with --shard one problem whose H2 build, SPD-HSS build and H2 products
(PCG's included) are sharded by subtrees over NCCL, strong scaling.

--impl reference: the CPU oracle (test infrastructure) timed on a bounded
sample of the same workload; prints the same JSON line with "impl": "reference".
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "SPD-HSS build s & H2 multi-vector GFLOP/s (fp64) vs FP64 roofline"
CFG = synth.C2
WORKLOAD = ("C2 (BASELINE configs[1]): N=32768 uniform [0,1]^3, Matern-3/2 (1+sqrt3 r/0.2)exp(-sqrt3 r/0.2) "
            "+ 1e-4 I, KD leaf 128, H2 proxy-ID tol 1e-10, SPD-HSS cap 100 / tol 1e-3, p=10, PCG b~N(0,1) to 1e-8; "
            "step = h2_build + spdhss_build + pcg_solve + h2_matvec(k=64)")
MV_K = 64
# roofline class of each kernel family
TENSOR_BOUND = {"kblock_dmma", "gemm_dmma"}
REF_SAMPLE_N = 2048      # oracle sample (same kernel / leaf / cap / tolerances)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--n", type=int, default=0, help="override N (testing only)")
    ap.add_argument("--shard", action="store_true",
                    help="N>1: ONE problem, H2/HSS builds and all H2 products sharded by subtrees over NCCL "
                         "(strong scaling); "
                         "default: independent replicas (weak scaling)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    REASONS = ["clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
               "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            q = "clocks.sm,clocks.max.sm," + ",".join(self.REASONS)
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.index)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out = self.proc.communicate()[0]
        sm, mx, reasons = [], [], set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6 or not f[0].isdigit():
                continue
            sm.append(int(f[0]))
            mx.append(int(f[1]))
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], f[2:]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ helpers
def load_traffic(kernel):
    """DRAM traffic of the dominant kernel from the committed ncu capture (or None)."""
    path = os.path.join(ROOT, "profiles", "r01g_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


def load_peaks():
    peaks = {}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peaks.update(json.load(open(p)))
    f = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(f):
        peaks.update(json.load(open(f)))
    return peaks


def prof_table(lib):
    import ctypes
    out = {}
    name = ctypes.create_string_buffer(64)
    vals = (ctypes.c_double * 4)()
    for i in range(lib.spd_prof_count()):
        if lib.spd_prof_get(i, name, 64, vals) == 0:
            out[name.value.decode()] = {"launches": vals[0], "ms": vals[1], "flops": vals[2], "bytes": vals[3]}
    return out


def max_over_ranks(v, device="cuda"):
    """Max of a per-rank float over the process group (identity without one)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(v)
    t = torch.tensor([float(v)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_config(rank):
    """Replicas (weak scaling): every rank solves its own C2 problem.  All ranks
    use the same recipe and seeds, so every replica does identical work."""
    return CFG


def h2_useful_flops(h, k):
    """F(k) = 2k (E_near + E_far + E_basis): ordered near leaf
    blocks n_a n_b, ordered Type-3 skeleton blocks s_a s_b, and the basis applies
    (up + down) 2 (sum_leaf n_a s_a + sum_nonleaf s_i sum_c s_c).  Evaluations of
    the kernel are not counted."""
    nodes = h.nodes()
    size = nodes[:, 1] - nodes[:, 0]
    r = h.ranks().astype(np.float64)
    e_near = float(sum(size[a] * size[b] for a, b in h.near_pairs()))
    e_far = float(sum(r[i] * r[j] for _, i, j in h.type3()))
    L = h.levels
    e_basis = 0.0
    for i in range(len(size)):
        lvl = L - int(math.floor(math.log2(i + 1)))
        if r[i] == 0:
            continue
        e_basis += r[i] * (size[i] if lvl == 1 else r[2 * i + 1] + r[2 * i + 2])
    return 2.0 * k * (e_near + e_far + 2.0 * e_basis), {"E_near": e_near, "E_far": e_far, "E_basis": e_basis}


def oracle_step(n):
    """One oracle pass (h2_build + Alg. 4 + PCG) on the C2 recipe at size n."""
    import oracle
    cfg = CFG.scaled(n)
    X = synth.points(cfg)
    h = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    H = oracle.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, synth.omega(cfg), form="chol")
    b = synth.rhs(cfg)[h.tree.perm]
    _, it, conv, _ = oracle.pcg(lambda v: oracle.h2_matvec(h, v), lambda v: oracle.hss_solve(H, v),
                                b, cfg.pcg_tol, cfg.maxit)
    return it


def cpu_baseline(n_full):
    """The oracle timed on a bounded sample (N=REF_SAMPLE_N), extrapolated by N log N."""
    t0 = time.time()
    it = oracle_step(REF_SAMPLE_N)
    dt = time.time() - t0
    scale = (n_full * math.log2(n_full / CFG.leaf)) / (REF_SAMPLE_N * math.log2(REF_SAMPLE_N / CFG.leaf))
    return {"value": round(dt * scale, 3), "unit": "s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"oracle h2_build+spdhss_build+pcg on the C2 recipe at N={REF_SAMPLE_N} "
                      f"({dt:.2f} s, {it} PCG its), extrapolated x{scale:.1f} by N log N to N={n_full}; "
                      "the oracle's C QRCP uses OpenMP over the host cores"}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(args.warmup):
        oracle_step(1024)                       # small warm-up (imports, C build)
    times = []
    for _ in range(args.steps):
        t0 = time.time()
        oracle_step(REF_SAMPLE_N)
        times.append(time.time() - t0)
    scale = (CFG.n * math.log2(CFG.n / CFG.leaf)) / (REF_SAMPLE_N * math.log2(REF_SAMPLE_N / CFG.leaf))
    v = statistics.mean(times) * scale
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v * 1e3, 1), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "parallelism": "cpu oracle (rank 0 only)"},
            "cpu_baseline": {"value": round(v, 3), "unit": "s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": f"each step: oracle on the C2 recipe at N={REF_SAMPLE_N} "
                                       f"(mean {statistics.mean(times):.2f} s), x{scale:.1f} by N log N"},
            "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2011_07632_b200 as spd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    lib = spd.lib()
    comm = None
    if args.shard and world > 1:
        uid = [spd.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = spd.Comm(world, rank, uid[0])
    cfg = replica_config(rank) if not args.n else CFG.scaled(args.n)
    N = cfg.n
    X_h = synth.points(cfg)
    b_h = synth.rhs(cfg)
    V_h = synth.multivec(N, MV_K)
    pts = torch.tensor(X_h, device="cuda")
    b = torch.tensor(b_h, device="cuda")
    V = torch.tensor(np.asfortranarray(V_h).T.copy(), device="cuda").t()
    flush = torch.empty(256 << 20 >> 3, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    record_flops = {}

    def step(points, rhs, record=None):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(stream)
        h = spd.h2_build(points, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol, comm=comm)
        ev[1].record(stream)
        H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=1234)
        ev[2].record(stream)
        x, rep = spd.pcg_solve(h, H, rhs, tol=cfg.pcg_tol, maxit=cfg.maxit)
        ev[3].record(stream)
        spd.h2_matvec(h, V)
        ev[4].record(stream)
        ev[4].synchronize()
        t = [ev[i].elapsed_time(ev[i + 1]) * 1e-3 for i in range(4)]
        if record is not None and not record:
            record_flops.update(zip(("flops", "counts"), h2_useful_flops(h, MV_K)))
        if record is not None:
            record.append({"h2_build_s": t[0], "spdhss_build_s": t[1], "pcg_s": t[2], "h2_mv_s": t[3],
                           "pcg_iters": rep.iters, "pcg_relres": rep.relres, "converged": rep.converged,
                           "h2_ranks_max": int(h.ranks().max()), "hss_rank_max": int(H.ranks().max()),
                           "h2_timings": list(h.timings()[:2]), "hss_timings": list(H.timings()[:4])})
        return x, h, H

    for _ in range(args.warmup):
        step(pts, b)
        flush.fill_(1.0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # ---------------- timed region (device events, max over ranks; library profiler OFF)
    sampler = ClockSampler(local)
    sampler.start()
    l0 = lib.spd_launch_count()
    recs, step_s = [], []
    torch.cuda.nvtx.range_push("timed")
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        step(pts, b, recs)
        s1.record(stream)
        s1.synchronize()
        step_s.append(s0.elapsed_time(s1) * 1e-3)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    launches = lib.spd_launch_count() - l0
    clocks = sampler.stop()
    t_step = max_over_ranks(statistics.mean(step_s))
    # ---------------- end-to-end: host (pinned) inputs, H2D inside, result D2H inside
    pts_pin = torch.tensor(X_h).pin_memory()
    b_pin = torch.tensor(b_h).pin_memory()
    x_pin = torch.empty(N, dtype=torch.float64).pin_memory()
    e2e = []
    for _ in range(max(1, args.steps)):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        p_d = pts_pin.to("cuda", non_blocking=True)
        b_d = b_pin.to("cuda", non_blocking=True)
        x, _, _ = step(p_d, b_d)
        x_pin.copy_(x, non_blocking=True)
        e1.record(stream)
        e1.synchronize()
        e2e.append(e0.elapsed_time(e1) * 1e-3)
    # ---------------- H2 multi-vector sweep over BASELINE C5's widths k in {1, 16, 64, 256}
    # on this workload's H2 (after the timed region; 3 timed products per k after one warm-up)
    sweep = {}
    _, h_sw, H_sw = step(pts, b)
    fp64_pk = load_peaks().get("fp64_dgemm_tflops_sustained") or load_peaks().get("fp64_dgemm_tflops") or 35.5
    for kk in (1, 16, 64, 256):
        Vk = torch.tensor(np.asfortranarray(synth.multivec(N, kk)).T.copy(), device="cuda").t()
        spd.h2_matvec(h_sw, Vk)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            spd.h2_matvec(h_sw, Vk)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 3
        fl = h2_useful_flops(h_sw, kk)[0]
        sweep[str(kk)] = {"ms": round(ms, 3), "useful_tflops": round(fl / ms / 1e9, 2),
                          "frac_fp64_peak": round(fl / ms / 1e9 / fp64_pk, 3)}
        del Vk
    # HSS error metric (the paper's Fig. 5 quantity P:1196-1206): mean over 10
    # Gaussian probes of ||H x - A_h2 x|| / ||A_h2 x||, H the SPD-HSS matrix (hss_matvec)
    Pr = torch.tensor(np.asfortranarray(np.random.default_rng(4000).standard_normal((N, 10))).T.copy(),
                      device="cuda").t()
    Ax = spd.h2_matvec(h_sw, Pr)
    Hx = spd.hss_matvec(H_sw, Pr)
    hss_err = float(((Hx - Ax).norm(dim=0) / Ax.norm(dim=0)).mean())
    # single-vector HSS solve (the PCG preconditioner), algorithmic bytes = the factors read
    # once: sum over nodes of 8 (m^2/2 + m r) (leaf m = n_i, nonleaf m = r_c1 + r_c2)
    hr = H_sw.ranks().astype(np.int64)
    nodes = h_sw.nodes()
    Lh = h_sw.levels
    hb = 0.0
    for i in range(len(hr)):
        depth = int(np.floor(np.log2(i + 1)))
        lev = Lh - depth
        if lev == Lh:
            m = int(hr[1] + hr[2]) if len(hr) > 2 else int(nodes[0, 1] - nodes[0, 0])
            hb += 8.0 * m * m / 2
            continue
        m = int(nodes[i, 1] - nodes[i, 0]) if lev == 1 else int(hr[2 * i + 1] + hr[2 * i + 2])
        hb += 8.0 * (m * m / 2 + m * int(hr[i]))
    bt = b.clone()
    for _ in range(3):
        spd.hss_solve(H_sw, bt, layout=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(20):
        spd.hss_solve(H_sw, bt, layout=1)
    e1.record(stream)
    e1.synchronize()
    hs_us = e0.elapsed_time(e1) / 20 * 1e3
    hss_solve_info = {"us": round(hs_us, 1), "algorithmic_mb": round(hb / 1e6, 1),
                      "gbs": round(hb / hs_us / 1e3, 1),
                      "frac_hbm": round(hb / hs_us / 1e3 / load_peaks().get("hbm_gbs", 6546.2), 3),
                      "note": "standalone solve (one launch per level); inside PCG the same phases run in the persistent kernel"}
    del h_sw, H_sw, Pr, Ax, Hx
    # ---------------- profiled pass (same steps, per-kernel-class CUDA events on the
    # launching streams; kept out of the timed region because the per-launch event
    # pairs and their host-side drains perturb the step time)
    lib.spd_prof_reset()
    lib.spd_prof_enable(1)
    prof_s = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        step(pts, b)
        s1.record(stream)
        s1.synchronize()
        prof_s.append(s0.elapsed_time(s1) * 1e-3)
    torch.cuda.synchronize()
    lib.spd_prof_enable(0)
    prof = prof_table(lib)
    e2e_v = max_over_ranks(statistics.mean(e2e))
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    # ---------------- roofline of the dominant kernel class
    peaks = load_peaks()
    fp64 = peaks.get("fp64_dgemm_tflops_sustained") or peaks.get("fp64_dgemm_tflops")
    fp64_src = "measured cuBLAS DGEMM sustained (profiles/fp64_peak.json)" if fp64 else \
        "bf16 measured x nominal fp64/bf16 ratio (40/2250)"
    if not fp64:
        fp64 = peaks.get("bf16_tflops_sustained", 1345.0) * 40.0 / 2250.0
    top = max(prof.items(), key=lambda kv: kv[1]["ms"]) if prof else (None, None)
    roof = None
    if top[0]:
        nm, p = top
        avg_s = p["ms"] * 1e-3 / max(1.0, p["launches"])
        if nm in TENSOR_BOUND:
            ach = p["flops"] / max(1.0, p["launches"]) / avg_s / 1e12
            roof = {"kernel": nm, "bound": "tensor", "achieved": round(ach, 3), "peak": round(fp64, 2),
                    "unit": "TFLOP/s", "frac": round(ach / fp64, 4), "traffic": None, "peak_source": fp64_src}
        else:
            ach = p["bytes"] / max(1.0, p["launches"]) / avg_s / 1e9
            roof = {"kernel": nm, "bound": "hbm", "achieved": round(ach, 1), "peak": peaks.get("hbm_gbs", 6550.7),
                    "unit": "GB/s", "frac": round(ach / peaks.get("hbm_gbs", 6550.7), 4), "traffic": None,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        tr = load_traffic(nm)
        if tr and nm == "pcg_persistent":        # per launch: ncu's bytes per PCG iteration x this launch's iterations
            roof["traffic"] = round(tr["bytes_per_iteration"] * statistics.mean(r["pcg_iters"] for r in recs) / 1e9, 2)
            roof["traffic_unit"] = "GB per launch (ncu dram read+write, profiles/r01g_traffic.json)"
            roof["algorithmic_gb_per_launch"] = round(p["bytes"] / max(1.0, p["launches"]) / 1e9, 2)
        roof["share_of_step"] = round(p["ms"] * 1e-3 / sum(prof_s), 4)
        roof["measured_in"] = "profiled pass (same steps as the timed region)"
    mv = statistics.mean(r["h2_mv_s"] for r in recs)
    mv_flops = prof.get("kblock_dmma", {}).get("flops", 0)
    line = {
        "metric": METRIC, "value": round(t_step, 4), "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 2), "higher_is_better": False,
        "scaling": "strong" if comm is not None else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "l2_flush": "256 MB write between steps",
                   "parallelism": ("h2_build, spdhss_build and every H2 product (PCG's k=1 too) sharded by subtrees over NCCL; "
                                   "PCG vectors and HSS solve replicated"
                                   if comm is not None else "replicas") if world > 1 else "single GPU", "N": N},
        "breakdown": {k: round(statistics.mean(r[k] for r in recs), 4)
                      for k in ("h2_build_s", "spdhss_build_s", "pcg_s", "h2_mv_s")},
        "full_build_s": round(statistics.mean(r["h2_build_s"] + r["spdhss_build_s"] for r in recs), 4),
        "pcg_iters": recs[-1]["pcg_iters"], "pcg_converged": bool(recs[-1]["converged"]),
        "h2_rank_max": recs[-1]["h2_ranks_max"], "hss_rank_max": recs[-1]["hss_rank_max"],
        "kernels": {k: {"launches": int(v["launches"]), "ms": round(v["ms"], 2),
                        "tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 3)} for k, v in prof.items()},
        "roofline": roof,
        "h2_multivector_sweep": sweep,
        "hss_error_o11": round(hss_err, 6),
        "hss_solve": hss_solve_info,
        "h2_multivector": {"k": MV_K, "useful_gflop": round(record_flops["flops"] / 1e9, 2),
                           "gflops": round(record_flops["flops"] / mv / 1e9, 1),
                           "frac_fp64_peak": round(record_flops["flops"] / mv / 1e12 / fp64, 4),
                           "counts": record_flops["counts"]},
        "e2e": {"value": round(e2e_v, 4), "unit": "s", "h2d_bytes_per_step": int(8 * N * (CFG.d + 1)),
                "d2h_bytes_per_step": int(8 * N)},
        "gpu_launches": int(launches // max(1, args.steps)),
        "profiled_pass_s_per_step": round(statistics.mean(prof_s), 4),
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(N)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
