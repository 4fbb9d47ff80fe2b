#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the SPD-HSS-from-H2 hot path.

BASELINE.json's metric is "SPD-HSS build s & H2 multi-vector GFLOP/s (fp64)"; its
single-GPU configurations at N = 2^20 are C4 (full build) and C5 (multi-vector
product sweep).  One STEP = one pass of the hot path on those configs:
    h2_build(C4) -> spdhss_build(C4, Alg. 4)  +  h2_matvec(C5's H2, X of width 64)
(C5's H2 is built once before the timed region; its product evaluates the kernel
blocks on the fly).  `value` = seconds per step (max over ranks), lower is better.
Inputs are resident in HBM when the timed region starts; they are larger than L2
(126 MB) and L2 is also flushed between steps (256 MB write).  Outside the timed
region: the C5 sweep k in {1, 16, 64, 256} (evaluated, then with the symmetric block
store, whose build time is reported), C4 PCG time-to-1e-8 once, the HSS solve
bandwidth, the O11 HSS error, a profiled pass (per-kernel-class CUDA events) for the
roofline, and the end-to-end pass through host buffers.
Multi-GPU (torchrun): independent replicas (weak scaling); --shard: one problem whose
builds and products are sharded by subtrees over NCCL (strong scaling).

--impl reference: the CPU oracle (test infrastructure) timed on a bounded sample of
the same workload (the C4 and C5 recipes at N = 4096), not extrapolated.
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
CFG = synth.C4                 # the full build (BASELINE configs[3])
CFG_MV = synth.C5              # the multi-vector product (BASELINE configs[4])
MV_K = 64
WORKLOAD = ("C4 full build + C5 product at N=2^20 (BASELINE configs[3], configs[4]): "
            "h2_build + spdhss_build of C4 (N=1048576 uniform [0,1]^3, IMQ 1/sqrt(r^2+0.01) + 1e-2 I, KD leaf 256, "
            "H2 proxy-ID tol 1e-10, SPD-HSS cap 150 / tol 1e-3, p=10, device Philox Omega) + one k=64 H2 product "
            "on C5's H2 (N=1048576 uniform [0,1]^3, Gaussian exp(-r^2/0.2^2), leaf 256, tol 1e-10, X~N(0,1), "
            "kernel blocks evaluated on the fly; C5's H2 built once before the timed region)")
# roofline class of each kernel family: DMMA contractions against the FP64
# peak; the QRCP with recomputed norms (R4) streams its trailing matrix once per step
# (its algorithmic bytes, set exactly after the launch), HBM-bound
TENSOR_BOUND = {"kblock_dmma", "gemm_dmma"}
HBM_BOUND = {"qrcp", "pcg_persistent", "hss_solve_vec", "sym_gemv"}
REF_SAMPLE_N = 4096      # oracle sample per reference-arm step (C4 / C5 recipes, same leaf / cap / tolerances)
def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pcg", action="store_true", help="skip the C4 PCG time-to-tolerance measurement")
    ap.add_argument("--minimal", action="store_true",
                    help="only the warm-up and timed steps (for profiler runs); prints the timing keys only")
    ap.add_argument("--n", type=int, default=0, help="override N of both configs (testing only)")
    ap.add_argument("--shard", action="store_true",
                    help="N>1: ONE problem, H2/HSS builds and all H2 products sharded by subtrees over NCCL "
                         "(strong scaling); default: independent replicas (weak scaling)")
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
    path = os.path.join(ROOT, "profiles", "r02c_traffic.json")
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
    """Replicas (weak scaling): every rank solves its own C4 build + C5 product.  All
    ranks use the same recipe and seeds, so every replica does identical work."""
    return CFG, CFG_MV


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
    """One oracle pass of the step on the C4 / C5 recipes at size n: h2_build +
    spdhss_build (Alg. 4, Philox Omega of reading R29) of the C4 recipe and one k=64
    product on the C5 recipe's H2 (built outside the timed part, like the GPU arm).
    Returns (seconds of the timed part, phase seconds)."""
    import oracle
    from oracle.omega import philox_normal
    c4, c5 = CFG.scaled(n), CFG_MV.scaled(n)
    h5 = oracle.h2_build(synth.points(c5), c5.kernel, c5.ell, c5.shift, c5.leaf, c5.h2_tol)
    V = synth.multivec(n, MV_K)[h5.tree.perm]
    t0 = time.time()
    X = synth.points(c4)
    h = oracle.h2_build(X, c4.kernel, c4.ell, c4.shift, c4.leaf, c4.h2_tol)
    t1 = time.time()
    oracle.spdhss_build(h, c4.rank_cap, c4.hss_tol, philox_normal(n, c4.w, 1234), form="chol")
    t2 = time.time()
    h5.blocks.clear()                          # evaluated on the fly, like the GPU step
    oracle.h2_matvec(h5, V)
    t3 = time.time()
    return t3 - t0, {"h2_build_s": round(t1 - t0, 3), "spdhss_build_s": round(t2 - t1, 3),
                     "c5_mv_s": round(t3 - t2, 3)}


def cpu_baseline():
    """The oracle as it stands, timed once on a bounded sample of the step (no scaling)."""
    dt, ph = oracle_step(REF_SAMPLE_N)
    return {"value": round(dt, 3), "unit": "s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"one step of the workload at N={REF_SAMPLE_N} instead of 2^20 (C4 recipe h2_build + "
                      f"spdhss_build, C5 recipe k={MV_K} product; leaf 256, caps and tolerances as configured), "
                      f"not extrapolated; phases {ph}; numpy/OpenMP over the host cores",
            "points_per_s": round(REF_SAMPLE_N / dt, 1)}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(args.warmup):
        oracle_step(1024)                       # small warm-up (imports, C build)
    times, phases = [], None
    for _ in range(args.steps):
        dt, phases = oracle_step(REF_SAMPLE_N)
        times.append(dt)
    v = statistics.mean(times)
    sample = (f"each step: the workload at N={REF_SAMPLE_N} instead of 2^20 (C4 recipe h2_build + spdhss_build, "
              f"C5 recipe k={MV_K} product), mean {v:.2f} s, not extrapolated; last phases {phases}")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v * 1e3, 1), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "parallelism": "cpu oracle (rank 0 only)", "N": REF_SAMPLE_N},
            "cpu_baseline": {"value": round(v, 3), "unit": "s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def colmajor(a):
    import torch
    return torch.tensor(np.asfortranarray(a).T.copy(), device="cuda").t()


def timed_products(spd, h, V, reps=3):
    """ms per product (one warm-up, then `reps` products between two events)."""
    import torch
    stream = torch.cuda.current_stream()
    spd.h2_matvec(h, V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        spd.h2_matvec(h, V)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def hss_solve_bytes(h, H):
    """Algorithmic bytes of one single-vector HSS solve: the factors read once,
    sum over nodes of 8 (m^2/2 + m r) (leaf m = n_i, nonleaf m = r_c1 + r_c2, root m^2/2)."""
    hr = H.ranks().astype(np.int64)
    nodes = h.nodes()
    Lh = h.levels
    hb = 0.0
    for i in range(len(hr)):
        lev = Lh - int(np.floor(np.log2(i + 1)))
        if lev == Lh:
            m = int(hr[1] + hr[2]) if len(hr) > 2 else int(nodes[0, 1] - nodes[0, 0])
            hb += 8.0 * m * m / 2
            continue
        m = int(nodes[i, 1] - nodes[i, 0]) if lev == 1 else int(hr[2 * i + 1] + hr[2 * i + 2])
        hb += 8.0 * (m * m / 2 + m * int(hr[i]))
    return hb


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
    c4, c5 = replica_config(rank)
    if args.n:
        c4, c5 = c4.scaled(args.n), c5.scaled(args.n)
    N = c4.n
    X4_h, X5_h = synth.points(c4), synth.points(c5)
    V_h = synth.multivec(N, MV_K)
    pts4 = torch.tensor(X4_h, device="cuda")
    pts5 = torch.tensor(X5_h, device="cuda")
    V = colmajor(V_h)
    flush = torch.empty(256 << 20 >> 3, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    # C5's H2, once, outside the timed region
    t5 = time.time()
    h5 = spd.h2_build(pts5, c5.kernel, c5.ell, c5.shift, c5.leaf, c5.h2_tol, comm=comm)
    torch.cuda.synchronize()
    h5_build_s = time.time() - t5
    mv_flops, mv_counts = h2_useful_flops(h5, MV_K)

    def step(points, X, record=None):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        h = spd.h2_build(points, c4.kernel, c4.ell, c4.shift, c4.leaf, c4.h2_tol, comm=comm)
        ev[1].record(stream)
        H = spd.spdhss_build(h, c4.rank_cap, c4.hss_tol, c4.oversample, seed=1234)
        ev[2].record(stream)
        Y = spd.h2_matvec(h5, X)
        ev[3].record(stream)
        ev[3].synchronize()
        t = [ev[i].elapsed_time(ev[i + 1]) * 1e-3 for i in range(3)]
        if record is not None:
            record.append({"h2_build_s": t[0], "spdhss_build_s": t[1], "c5_mv_s": t[2],
                           "h2_rank_max": int(h.ranks().max()), "hss_rank_max": int(H.ranks().max()),
                           "h2_timings": list(h.timings()[:2]), "hss_timings": list(H.timings()[:4])})
        return h, H, Y

    os.environ["SPD_STORE_FRAC"] = "0"       # the step's product evaluates its kernel blocks (north star)
    for _ in range(args.warmup):
        out = step(pts4, V)
        out = None
        flush.fill_(1.0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # ---------------- timed region (device events, max over ranks; library profiler OFF)
    sampler = ClockSampler(local)
    sampler.start()
    l0 = lib.spd_launch_count()
    recs, step_s = [], []
    last = None
    torch.cuda.nvtx.range_push("timed")
    for _ in range(args.steps):
        last = None                          # free the previous step's H2 / HSS / product
        flush.fill_(1.0)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        last = step(pts4, V, recs)
        s1.record(stream)
        s1.synchronize()
        step_s.append(s0.elapsed_time(s1) * 1e-3)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    launches = lib.spd_launch_count() - l0
    clocks = sampler.stop()
    t_step = max_over_ranks(statistics.mean(step_s))
    h4, H4, _ = last
    last = None
    if args.minimal:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": round(t_step, 4), "unit": "s", "n_gpus": world,
                              "steps": args.steps, "warmup": args.warmup, "minimal": True,
                              "breakdown": {k: round(statistics.mean(r[k] for r in recs), 4)
                                            for k in ("h2_build_s", "spdhss_build_s", "c5_mv_s")},
                              "gpu_launches": int(launches // max(1, args.steps)), "clocks": clocks}), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    # ---------------- O11 HSS error and the standalone HSS solve on the last C4 build
    Pr = colmajor(np.random.default_rng(4000).standard_normal((N, 10)))
    Ax = spd.h2_matvec(h4, Pr)
    Hx = spd.hss_matvec(H4, Pr)
    hss_err = float(((Hx - Ax).norm(dim=0) / Ax.norm(dim=0)).mean())
    del Pr, Ax, Hx
    hb = hss_solve_bytes(h4, H4)
    b4 = torch.tensor(synth.rhs(c4), device="cuda")
    bt = b4.clone()
    for _ in range(3):
        spd.hss_solve(H4, bt, layout=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(20):
        spd.hss_solve(H4, bt, layout=1)
    e1.record(stream)
    e1.synchronize()
    hs_us = e0.elapsed_time(e1) / 20 * 1e3
    hss_solve_info = {"us": round(hs_us, 1), "algorithmic_mb": round(hb / 1e6, 1),
                      "gbs": round(hb / hs_us / 1e3, 1),
                      "frac_hbm": round(hb / hs_us / 1e3 / load_peaks().get("hbm_gbs", 6546.2), 3),
                      "note": "standalone C4 solve (one launch per level); inside PCG the same phases run in "
                              "the persistent kernel or the per-iteration graph"}
    h4 = H4 = bt = None                      # one C4 build alive at a time (memory-pool growth stalls)
    # ---------------- end-to-end: host (pinned) inputs, H2D inside, results D2H inside
    pts_pin = torch.tensor(X4_h).pin_memory()
    V_pin = torch.tensor(np.ascontiguousarray(V_h.T)).pin_memory()          # k x N = column-major N x k
    Y_pin = torch.empty((MV_K, N), dtype=torch.float64).pin_memory()
    e2e = []
    for _ in range(max(1, min(args.steps, 2))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        p_d = pts_pin.to("cuda", non_blocking=True)
        V_d = V_pin.to("cuda", non_blocking=True).t()
        h, H, Y = step(p_d, V_d)
        Y_pin.copy_(Y.t(), non_blocking=True)
        ranks = H.ranks()                    # the build's result read back (host query)
        e1.record(stream)
        e1.synchronize()
        e2e.append(e0.elapsed_time(e1) * 1e-3)
        h = H = Y = p_d = V_d = None
    e2e_v = max_over_ranks(statistics.mean(e2e))
    # ---------------- C5 multi-vector sweep k in {1, 16, 64, 256} (BASELINE configs[4])
    fp64_pk = load_peaks().get("fp64_dgemm_tflops_sustained") or load_peaks().get("fp64_dgemm_tflops") or 35.5
    sweep = {}
    for kk in (16, 64, 256, 1):
        Vk = colmajor(synth.multivec(N, kk))
        fl = h2_useful_flops(h5, kk)[0]
        ent = {}
        ms = timed_products(spd, h5, Vk)
        ent.update({"ms": round(ms, 3), "useful_tflops": round(fl / ms / 1e9, 2),
                    "frac_fp64_peak": round(fl / ms / 1e9 / fp64_pk, 3), "blocks": "evaluated on the fly"})
        sweep[str(kk)] = ent
        del Vk
    # the symmetric block store (f4): built by the first PCG-path k = 1 product (within the
    # free memory); timed: that first product including the store build, then k = 1, 64, 256
    # products reading the store
    stored = {}
    os.environ["SPD_STORE_FRAC"] = "0.25"
    b5 = torch.tensor(synth.rhs(c5), device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    spd.pcg_solve(h5, None, b5, tol=1e-300, maxit=1)          # one CG iteration = one stored k=1 product
    e1.record(stream)
    e1.synchronize()
    stored["first_k1_ms_incl_store_build"] = round(e0.elapsed_time(e1), 1)
    stored["store_gb"] = round(h5.sym_store()[0] / 1e9, 2)
    if h5.sym_store()[0] > 0:                 # products reading the store instead
        V1 = colmajor(synth.multivec(N, 1))[:, 0].contiguous()
        ms = timed_products(spd, h5, V1)
        fl = h2_useful_flops(h5, 1)[0]
        stored["1"] = {"ms": round(ms, 3), "useful_tflops": round(fl / ms / 1e9, 2)}
        for kk in (64, 256):
            Vk = colmajor(synth.multivec(N, kk))
            ms = timed_products(spd, h5, Vk)
            fl = h2_useful_flops(h5, kk)[0]
            stored[str(kk)] = {"ms": round(ms, 3), "useful_tflops": round(fl / ms / 1e9, 2),
                               "frac_fp64_peak": round(fl / ms / 1e9 / fp64_pk, 3)}
            del Vk
        stored["store_build_included_in"] = "first_k1_ms_incl_store_build"
    h5.release_store()
    os.environ["SPD_STORE_FRAC"] = "0"
    # ---------------- profiled pass (same step, per-kernel-class CUDA events on the
    # launching streams; kept out of the timed region because the per-launch event
    # pairs and their host-side drains perturb the step time)
    lib.spd_prof_reset()
    lib.spd_prof_enable(1)
    prof_s = []
    for _ in range(1):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        out = step(pts4, V)
        s1.record(stream)
        s1.synchronize()
        h4, H4, _ = out                       # kept for the PCG below
        out = None
        prof_s.append(s0.elapsed_time(s1) * 1e-3)
    torch.cuda.synchronize()
    lib.spd_prof_enable(0)
    prof = prof_table(lib)
    # ---------------- C4 PCG time-to-1e-8, once (maxit 10000, reading R25)
    pcg_info = None
    if not args.no_pcg:
        h5 = None                            # C5's H2 is not needed any more: room for C4's block store
        torch.cuda.synchronize()
        free_before = torch.cuda.mem_get_info()[0]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, rep = spd.pcg_solve(h4, H4, b4, tol=c4.pcg_tol, maxit=10000)
        e1.record(stream)
        e1.synchronize()
        pcg_info = {"s": round(e0.elapsed_time(e1) * 1e-3, 3), "iters": rep.iters, "converged": bool(rep.converged),
                    "relres_true": rep.relres_true, "ms_per_iter": round(e0.elapsed_time(e1) / max(1, rep.iters), 3),
                    "store_gb": round(h4.sym_store()[0] / 1e9, 2), "free_gb_before": round(free_before / 1e9, 1),
                    "note": "includes building the symmetric k=1 block store (as much as fits the free memory)"}
    h4 = H4 = b4 = bt = None
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": round(t_step, 4), "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 2), "higher_is_better": False,
        "scaling": "strong" if comm is not None else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "N": N, "l2_flush": "256 MB write between steps; inputs > L2",
                   "parallelism": ("h2_build, spdhss_build and every H2 product sharded by subtrees over NCCL"
                                   if comm is not None else "replicas") if world > 1 else "single GPU"},
        "breakdown": dict({k: round(statistics.mean(r[k] for r in recs), 4)
                           for k in ("h2_build_s", "spdhss_build_s", "c5_mv_s")},
                          h2_tree_lists_s=round(statistics.mean(r["h2_timings"][0] for r in recs), 4)),
        "full_build_s": round(statistics.mean(r["h2_build_s"] + r["spdhss_build_s"] for r in recs), 4),
        "h2_rank_max": recs[-1]["h2_rank_max"], "hss_rank_max": recs[-1]["hss_rank_max"],
        "c5_h2_build_s": round(h5_build_s, 3),
        "h2_multivector": {"k": MV_K, "useful_gflop": round(mv_flops / 1e9, 2),
                           "gflops": round(mv_flops / statistics.mean(r["c5_mv_s"] for r in recs) / 1e9, 1),
                           "frac_fp64_peak": round(mv_flops / statistics.mean(r["c5_mv_s"] for r in recs)
                                                   / 1e12 / fp64_pk, 4),
                           "counts": mv_counts},
        "h2_multivector_sweep": sweep,
        "h2_multivector_stored": stored,
        "pcg_c4": pcg_info,
        "hss_error_o11": round(hss_err, 6),
        "hss_solve": hss_solve_info,
        "kernels": {k: {"launches": int(v["launches"]), "ms": round(v["ms"], 2),
                        "tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 3),
                        "gbs": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)} for k, v in prof.items()},
        "roofline": roofline(prof, sum(prof_s)),
        "e2e": {"value": round(e2e_v, 4), "unit": "s",
                "h2d_bytes_per_step": int(8 * N * (c4.d + MV_K)), "d2h_bytes_per_step": int(8 * N * MV_K)},
        "gpu_launches": int(launches // max(1, args.steps)),
        "profiled_pass_s_per_step": round(statistics.mean(prof_s), 4),
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def roofline(prof, prof_total_s):
    """Roofline of the dominant kernel class of the profiled step: achieved = its
    algorithmic flops (tensor) or bytes (hbm) per launch / its mean launch duration."""
    peaks = load_peaks()
    fp64 = peaks.get("fp64_dgemm_tflops_sustained") or peaks.get("fp64_dgemm_tflops")
    fp64_src = "measured cuBLAS DGEMM sustained (profiles/fp64_peak.json)" if fp64 else \
        "bf16 measured x nominal fp64/bf16 ratio (40/2250)"
    if not fp64:
        fp64 = peaks.get("bf16_tflops_sustained", 1345.0) * 40.0 / 2250.0
    if not prof:
        return None
    nm, p = max(prof.items(), key=lambda kv: kv[1]["ms"])
    avg_s = p["ms"] * 1e-3 / max(1.0, p["launches"])
    if nm in TENSOR_BOUND or (nm not in HBM_BOUND and p["flops"] > 5.7 * max(p["bytes"], 1.0)):
        ach = p["flops"] / max(1.0, p["launches"]) / avg_s / 1e12
        roof = {"kernel": nm, "bound": "tensor", "achieved": round(ach, 3), "peak": round(fp64, 2),
                "unit": "TFLOP/s", "frac": round(ach / fp64, 4), "traffic": None, "peak_source": fp64_src}
    else:
        ach = p["bytes"] / max(1.0, p["launches"]) / avg_s / 1e9
        roof = {"kernel": nm, "bound": "hbm", "achieved": round(ach, 1), "peak": peaks.get("hbm_gbs", 6550.7),
                "unit": "GB/s", "frac": round(ach / peaks.get("hbm_gbs", 6550.7), 4), "traffic": None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    tr = load_traffic(nm)
    if tr:                                       # ncu DRAM bytes of every launch of this class in one step,
        tot = tr.get("dram_read_gb", 0.0) + tr.get("dram_write_gb", 0.0)       # averaged like `achieved`
        roof["traffic"] = round(tot / max(1.0, p["launches"]), 2) if tot else tr.get("gb_per_launch")
        roof["traffic_unit"] = f"GB per launch (ncu dram read+write, {tr.get('source')})"
    roof["algorithmic_per_launch"] = {"gflop": round(p["flops"] / max(1.0, p["launches"]) / 1e9, 3),
                                      "gb": round(p["bytes"] / max(1.0, p["launches"]) / 1e9, 4)}
    roof["launches"] = int(p["launches"])
    roof["share_of_step"] = round(p["ms"] * 1e-3 / prof_total_s, 4)
    roof["measured_in"] = "profiled pass (one step, per-launch CUDA events on the launching stream)"
    return roof


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
