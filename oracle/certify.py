"""Certified-tie checks of pivot sequences (reading R19) -- TEST INFRASTRUCTURE ONLY.

Businger-Golub QRCP (Alg. 2 step 3; reading R4) takes at step t the
column of largest residual norm.  Two correct implementations that round differently
can take different columns when two norms are within rounding of each other, and
truncate one step apart when |R_tt| lies within rounding of tau |R_00|.  Reading R19
accepts another implementation's run iff, replayed step by step in the oracle
(`qrcp_trace` in follow mode: the oracle's own arithmetic, the other run's pivots):

  pivots   nu_max(t) - nu_taken(t) <= band                   for every step t < s
  rank     nu_max(t) >  tau nu_0 - band                       for every t < s (it went on)
           nu_max(s) <= tau nu_0 + band  (or nu_max(s) == 0)  if s < min(m, n, cap) (it stopped)
  band     = 16 sqrt(m) eps nu_0,  nu_0 = nu_max(0)  (m = rows of the factored matrix)

A run that agrees with the oracle's own pivots passes trivially (every difference 0).
"""
import numpy as np

from .linalg import qrcp_trace

EPS = np.finfo(np.float64).eps


def certify_pivots(A, pivots, rank, rel_tol, max_rank, band_factor=16.0):
    """Replay `pivots[:rank]` (original column indices of A) in the oracle's QRCP.

    Returns a dict: ok, own (the oracle's own pivots[:r0] and rank r0), ties (steps
    where the replayed pivot differs from the oracle's argmax), worst (largest
    (nu_max - nu_taken) / band over the steps), rank_ok, band."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    kmax = max(0, min(m, n, int(max_rank)))
    s = int(rank)
    _, own_piv, r0, _, _ = qrcp_trace(A, max_rank, rel_tol)
    out = {"own": own_piv[:r0].copy(), "own_rank": r0, "ties": [], "worst": 0.0, "rank_ok": True,
           "ok": True, "band": 0.0}
    if s == r0 and np.array_equal(np.asarray(pivots[:s]), own_piv[:s]):
        return out
    _, _, r, numax, nuf = qrcp_trace(A, max_rank, rel_tol, follow=np.asarray(pivots[:s]))
    if r < 0 or s > kmax:
        out["ok"] = out["rank_ok"] = False
        return out
    nu0 = numax[0] if kmax > 0 else 0.0
    band = band_factor * np.sqrt(m) * EPS * nu0
    out["band"] = band
    for t in range(s):
        gap = numax[t] - nuf[t]
        if gap > 0.0:
            out["ties"].append(t)
            out["worst"] = max(out["worst"], gap / band if band > 0 else np.inf)
        if not numax[t] > rel_tol * nu0 - band:
            out["rank_ok"] = False
    if s < kmax and not (numax[s] == 0.0 or numax[s] <= rel_tol * nu0 + band):
        out["rank_ok"] = False
    out["ok"] = out["rank_ok"] and out["worst"] <= 1.0
    return out


def hss_tie_records(H, rank_cap, rel_tol, w, band_factor=16.0):
    """Per-node records of an oracle SPD-HSS build made with keep_sketch=True, over the
    nodes sorted by heap index (levels 1..L-1): ranks (array over all nodes), the pivots
    [:r] concatenated, and per node and step t < r the gap between the largest and the
    runner-up residual norm and the runner-up's column (band units, reading R19), and
    the rank margins (how far |R_rr| stopped below tau |R_00|, how far |R_(r-1)(r-1)|
    was above it; band units, inf when not applicable)."""
    from .linalg import qrcp_trace
    nn = H.h2.tree.nnodes
    rank = np.zeros(nn, np.int32)
    pivs, gaps, idx2, margins = [], [], [], []
    for i in sorted(H.rank):
        r = H.rank[i]
        rank[i] = r
        pivs.append(np.asarray(H.piv[i][:r], np.int32))
        Lam = H.Lam[i]
        _, piv, r2, numax, _, nu2, i2 = qrcp_trace(Lam, rank_cap, rel_tol, runner_up=True)
        assert r2 == r and np.array_equal(piv[:r], H.piv[i][:r])
        band = band_factor * np.sqrt(max(Lam.shape[0], 1)) * EPS * (numax[0] if r else 0.0)
        g = np.full(w, np.inf)
        ii = np.full(w, -1, np.int64)
        lo = hi = np.inf
        if r and band > 0:
            g[:r] = (numax[:r] - nu2[:r]) / band
            ii[:r] = i2[:r]
            thr = rel_tol * numax[0]
            if r < min(Lam.shape[0], Lam.shape[1], rank_cap):
                lo = (thr - numax[r]) / band
            hi = (numax[r - 1] - thr) / band
        gaps.append(g)
        idx2.append(ii)
        margins.append((lo, hi))
    return (rank, np.concatenate(pivs) if pivs else np.zeros(0, np.int32), np.stack(gaps),
            np.stack(idx2).astype(np.int32), np.array(margins, dtype=np.float64).reshape(-1, 2))
