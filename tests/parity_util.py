"""Certified-tie checks of GPU skeleton and pivot sets against the oracle (reading
R19, SURVEY.md §8(c) parity protocol steps 2 and 4).  Test infrastructure.

certify_h2   every active node's skeleton sequence (pivot order) and rank must be a
             valid Businger-Golub run on the node's proxy matrix M^T in the oracle's
             arithmetic: identical to the oracle's own run, or -- replayed with the
             GPU's pivots (oracle/certify.py) -- every deviation a tie within the band
             16 sqrt(m) eps nu_0 and the rank within that band of the threshold.  The
             candidates of a nonleaf node are the GPU's own child skeletons.
certify_hss  the SPD-HSS QRCP pivots: identical to the oracle's, or the first deviation
             is the oracle's runner-up within the band (golden per-step gaps), or the
             rank differs by one within the band (golden rank margins).
"""
import numpy as np

import oracle
from oracle.certify import certify_pivots
from oracle.h2 import active_nodes, default_n_proxy, proxy_points
from oracle.kernels import dof_points, dofs_per_point, kernel_matrix
from oracle.tree import build_tree, expand_dofs, interaction_lists


class TreeInfo:
    """The oracle's tree, lists, tree-order points and active set for a point set."""

    def __init__(self, X, kid, leaf):
        m = dofs_per_point(kid)
        t = build_tree(X, leaf)
        lists = interaction_lists(t)
        self.tree = expand_dofs(t, m)
        self.lists = lists
        Xd = np.asarray(X, dtype=np.float64) if m == 1 else dof_points(X, m)
        self.Xt = Xd[self.tree.perm]
        self.active = active_nodes(self.tree, lists)
        self.m = m


def certify_h2(info, kid, ell, tol, gpu_rank, gpu_skel, oracle_skel=None, n_proxy=0):
    """Returns (nodes, identical, ties, failures) over the active nodes."""
    t = info.tree
    n_proxy = n_proxy or default_n_proxy(t.d)
    nodes = same = ties = 0
    fails = []
    ident = {}
    for k in range(1, t.L):
        for i in t.nodes_at(k):
            s = int(gpu_rank[i])
            gs = np.asarray(gpu_skel.get(i, np.zeros(0, np.int64)), np.int64)
            if not info.active[i]:
                if s != 0:
                    fails.append((i, "inactive node with a skeleton"))
                ident[i] = True
                continue
            nodes += 1
            if t.is_leaf(i):
                cand = np.arange(t.begin[i], t.end[i])
                kids_same = True
            else:
                c1, c2 = t.children(i)
                cand = np.concatenate([np.asarray(gpu_skel.get(c, np.zeros(0, np.int64)), np.int64)
                                       for c in (c1, c2)])
                kids_same = ident[c1] and ident[c2]
            if oracle_skel is not None and kids_same and np.array_equal(gs, np.asarray(oracle_skel[i])):
                same += 1
                ident[i] = True
                continue
            ident[i] = False
            Y = proxy_points(t, i, n_proxy)
            if info.m > 1:
                Y = dof_points(Y, info.m)
            M = kernel_matrix(kid, ell, info.Xt[cand], Y)
            pos = {int(c): a for a, c in enumerate(cand)}
            if any(int(g) not in pos for g in gs):
                fails.append((i, "skeleton not among the candidates"))
                continue
            piv = np.array([pos[int(g)] for g in gs], np.int64)
            c = certify_pivots(M.T, piv, s, tol, min(M.shape))
            if c["ok"]:
                ties += 1
            else:
                fails.append((i, f"not certified: ties {c['ties'][:4]} worst {c['worst']:.3g} band units, "
                                 f"rank {s} (oracle {c['own_rank']}) rank_ok {c['rank_ok']}"))
    return nodes, same, ties, fails


def certify_hss(gpu_piv, gpu_rank, nodes, o_rank, o_piv_flat, o_gap, o_idx2, o_margin):
    """nodes: the heap nodes in the golden's (sorted) order.  Returns (identical, ties, failures)."""
    same = ties = 0
    fails = []
    off = 0
    for a, i in enumerate(nodes):
        ro = int(o_rank[i])
        po = o_piv_flat[off:off + ro]
        off += ro
        rg = int(gpu_rank[i])
        pg = np.asarray(gpu_piv[i][:rg])
        n = min(ro, rg)
        diff = np.nonzero(pg[:n] != po[:n])[0]
        if rg == ro and diff.size == 0:
            same += 1
            continue
        if diff.size:
            t = int(diff[0])
            if o_gap[a, t] <= 1.0 and int(pg[t]) == int(o_idx2[a, t]):
                ties += 1
                continue
            fails.append((i, f"pivot {t}: gpu {pg[t]} oracle {po[t]} (runner-up {o_idx2[a, t]}, "
                             f"gap {o_gap[a, t]:.3g} band units)"))
            continue
        if rg == ro - 1 and o_margin[a, 1] <= 1.0 or rg == ro + 1 and o_margin[a, 0] <= 1.0:
            ties += 1
            continue
        fails.append((i, f"rank gpu {rg} oracle {ro} (margins {o_margin[a]})"))
    return same, ties, fails


def oracle_skel_dict(rank, flat):
    out, off = {}, 0
    for i, s in enumerate(rank):
        if s:
            out[i] = flat[off:off + int(s)].astype(np.int64)
            off += int(s)
    return out


def maxrel(a, b):
    """Largest elementwise difference relative to the largest entry of b."""
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
