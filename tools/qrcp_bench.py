"""Diagnostic: time the batched QRCP alone (spd_test_qrcp, no Q) on `batch` m x m
matrices with singular values logspace(0, -14) (rank ~0.7 m at tol 1e-10), the shape of
one H2 level's triangles.  python tools/qrcp_bench.py batch m [reps]; SPD_QRCP_EAGER=1
selects the eager kernel."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_07632_b200 as spd  # noqa: E402

batch, m = int(sys.argv[1]), int(sys.argv[2])
TRIFILE = os.environ.get("TRI_FILE")      # triangles dumped by SPD_DUMP_QRCP (h2 build): batch m ignored
if TRIFILE:
    import numpy as np
    raw = open(TRIFILE, "rb").read()
    hdr = np.frombuffer(raw[:12], np.int32)
    mats, off = [], 12
    for q in range(int(hdr[0])):
        mq = int(np.frombuffer(raw[off:off + 4], np.int32)[0]); off += 4
        mats.append(np.frombuffer(raw[off:off + 8 * mq * mq], np.float64).reshape(mq, mq)); off += 8 * mq * mq
    m = max(a.shape[0] for a in mats)           # smaller triangles zero-padded (zero rows / columns)
    batch = len(mats)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ld = int(sys.argv[4]) if len(sys.argv) > 4 else m        # leading dimension (the H2 build: n_p = 6144)
g = torch.Generator(device="cuda").manual_seed(7)
s = torch.logspace(0, -14, m, dtype=torch.float64, device="cuda")
A0 = torch.zeros(batch, m, ld, dtype=torch.float64, device="cuda")     # column j of b: A0[b, j, :m]
for b in range(0 if TRIFILE else batch):
    G1 = torch.randn(m, m, dtype=torch.float64, device="cuda", generator=g)
    G2 = torch.randn(m, m, dtype=torch.float64, device="cuda", generator=g)
    M = (G1 * s) @ G2.T
    if os.environ.get("TRI"):            # the H2 build's input: the R factor (upper triangular)
        M = torch.linalg.qr(M)[1]
    A0[b, :, :m] = M.T
if TRIFILE:
    for b in range(batch):
        mb = mats[b].shape[0]
        A0[b, :mb, :mb] = torch.tensor(mats[b], device="cuda")    # stored column-major = rows of mats[b]
piv = torch.zeros(batch * m, dtype=torch.int32, device="cuda")
rank = torch.zeros(batch, dtype=torch.int32, device="cuda")
keep = []
PRE = None
if os.environ.get("PRE_QR"):             # a blocked QR of the same shape right before (as in the H2 build)
    PRE = torch.randn(batch, m, 6144, dtype=torch.float64, device="cuda", generator=g)
for rep in range(reps):
    A = A0.clone()
    if PRE is not None:
        P = PRE.clone()
        assert spd.lib().spd_test_qr_unpivoted(batch, ctypes.c_void_p(P.data_ptr()), 6144, m, 6144, m * 6144,
                                               spd._stream()) == 0
        del P
    if os.environ.get("FRESH"):
        keep.append(A)          # every rep on newly allocated memory
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = spd.lib().spd_test_qrcp(batch, ctypes.c_void_p(A.data_ptr()), m, m, ld, m * ld, m, 1e-10,
                                 ctypes.c_void_p(piv.data_ptr()), ctypes.c_void_p(rank.data_ptr()),
                                 None, 0, spd._stream())
    e1.record()
    torch.cuda.synchronize()
    assert st == 0, spd.lib().spd_last_error()
    r = rank.cpu()
    ent = sum(float(((m - torch.arange(0, min(int(k) + 1, m), dtype=torch.float64)) ** 2).sum()) for k in r)
    ms = e0.elapsed_time(e1)
    print(f"batch {batch} m {m} rank mean {r.double().mean():.0f}: {ms:.1f} ms, "
          f"algorithmic {8 * ent / 1e9:.1f} GB -> {8 * ent / ms / 1e6:.0f} GB/s "
          f"({'eager' if os.environ.get('SPD_QRCP_EAGER') else 'deferred'})", flush=True)
