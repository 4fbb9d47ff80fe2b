"""SPD HSS construction, HSS apply/solve and PCG (oracle O5-O11).
TEST INFRASTRUCTURE ONLY.

spdhss_build      Alg. 4 (alg:spdhss_h2) step by step.
                  form="eig": (I + B_ii)^{+-1/2} by eigendecomposition, exactly
                  as printed.  form="chol": the Cholesky variant of
                  reading R9 (F F^T = I + B_ii, F = (I+B)^{1/2} Q); R_i, B_ij
                  and Phi are identical in exact arithmetic, V-bar rotates by
                  Q^T.  Sketches via Alg. 3 (alg:spdhss_matvec P:866-884)
                  recomputed from the leaf level for every k, as printed.
                  Y^(k) by the literal masked H2 product (eqn:Yk).
alg1_generalized  Alg. 1 (alg:spdhss) on the dense matrix with
                  injected bases (quadratic; tiny N only; O7).
hss_matvec        HSS apply: leaf D_i, U_i; transfers R_i; sibling B_ij
                  (eqn:nested).
hss_solve         recursive solve of reading R12:
                  H^{-1} = S^{-T}[(I - V V^T) + V (I+H_2)^{-1} V^T] S^{-1}.
pcg               textbook PCG, x0 = 0, stop on ||r_k|| <= tol ||b|| (R15).
block_jacobi_solve  the BJ baseline preconditioner:
                  x_i = A_ii^{-1} b_i over the leaves, A_ii = K(X_i, X_i) + sigma I.
hss_error         Fig. 5 metric: mean over probes of
                  ||H_hss x - H_h2 x|| / ||H_h2 x||.
"""
from dataclasses import dataclass, field
import numpy as np
from scipy.linalg import solve_triangular

from .linalg import NotPD, cholesky, qrcp, sym_sqrt_pair
from .h2 import H2, h2_matvec


@dataclass
class HSS:
    """SPD HSS approximation plus the factors the solve needs."""
    h2: H2
    form: str
    rank: dict = field(default_factory=dict)     # node -> r_i (levels 1..L-1)
    D: dict = field(default_factory=dict)        # leaf A_ii
    S: dict = field(default_factory=dict)        # leaf Cholesky factor
    V: dict = field(default_factory=dict)        # leaf V_i / nonleaf V-bar_i
    U: dict = field(default_factory=dict)        # leaf U_i = S_i V_i
    R: dict = field(default_factory=dict)        # nonleaf R_i = F_i Vbar_i
    F: dict = field(default_factory=dict)        # nonleaf F_i with F F^T = I + B_ii (root too)
    Finv: dict = field(default_factory=dict)     # (I+B)^{-1/2} (eig) or F^{-1} (chol)
    B: dict = field(default_factory=dict)        # (i, j) -> B_ij for i < j, Type-1/3/siblings
    PhiU: dict = field(default_factory=dict)     # node -> Phi_i U_i^{H2}
    Phi_leaf: dict = field(default_factory=dict)
    piv: dict = field(default_factory=dict)
    Lam: dict = field(default_factory=dict)      # node -> the sketch QRCP factored (keep_sketch)
    sketch_widths: list = field(default_factory=list)   # instrumentation

    def Bij(self, i, j):
        if i < j:
            return self.B[(i, j)]
        return self.B[(j, i)].T

    def sibling_B(self, p):
        c1, c2 = self.h2.tree.children(p)
        return self.Bij(c1, c2)


def _bold(hss: HSS, i, j):
    """Bold B_ij: children blocks B_{i_a j_b}; diagonal blocks 0 if i == j."""
    t = hss.h2.tree
    ci, cj = t.children(i), t.children(j)
    rows = []
    for a in ci:
        row = []
        for b in cj:
            if a == b:
                row.append(np.zeros((hss.rank[a], hss.rank[b])))
            else:
                row.append(hss.Bij(a, b))
        rows.append(np.hstack(row))
    return np.vstack(rows)


def _pairs(lists, k):
    """Type-1 and Type-3 pairs (i < j) at level k."""
    t1 = [(i, j) for (i, j) in lists.type1[k] if i < j]
    t3 = [(i, j) for (i, j) in lists.type3[k] if i < j]
    return t1, t3


def _left_factor(hss, i):
    """The matrix applied to the stacked children quantities at node i:
    (I+B_ii)^{-1/2} (eig) or F_i^{-1} (chol, R9)."""
    return hss.Finv[i]


def special_products(hss: HSS, Yk, k):
    """Alg. 3: (I+B_ii)^{-1/2} diag(Phi_children) Y_i^(k) for i in lvl(k).

    Needs levels 1..k-1 of hss and the factors of level k.
    """
    t = hss.h2.tree
    T = {}
    for i in t.nodes_at(1):                            # T_i = V_i^T S_i^{-1} Y_i
        Ti = Yk[t.begin[i]:t.end[i]]
        Ti = solve_triangular(hss.S[i], Ti, lower=True) if Ti.shape[0] else Ti
        T[i] = hss.V[i].T @ Ti
    for l in range(2, k):                              # T_i = Vbar^T (I+B)^{-1/2} [T_c]
        for i in t.nodes_at(l):
            c1, c2 = t.children(i)
            T[i] = hss.V[i].T @ (_left_factor(hss, i) @ np.vstack([T[c1], T[c2]]))
    out = {}
    for i in t.nodes_at(k):
        c1, c2 = t.children(i)
        out[i] = _left_factor(hss, i) @ np.vstack([T[c1], T[c2]])
    return out


def spdhss_build(h2: H2, rank_cap, rel_tol, omega, form="eig", keep_sketch=False):
    """Alg. 4.  omega: N x (r+p) in tree order (one for all k, R8).
    keep_sketch: keep every node's sketch Lambda (the matrix its QRCP factors) in
    hss.Lam, for the certified-tie records of reading R19."""
    t, lists = h2.tree, h2.lists
    L = t.L
    hss = HSS(h2, form)
    if L == 1:                                          # single node: HSS = dense block
        r0 = np.arange(t.N)
        hss.D[0] = h2.K(r0, r0)
        hss.S[0] = cholesky(hss.D[0], where=(1, 0))
        return hss
    omega = np.asarray(omega, dtype=np.float64)
    # line 1: Y^(k) = (A - diag(A_ii, i in lvl(k))) Omega, k = 1..L-1
    Y = {k: h2_matvec(h2, omega, exclude_level=k) for k in range(1, L)}
    hss.sketch_widths = [omega.shape[1]] * (L - 1)

    # ---- leaf level
    for i in t.nodes_at(1):
        rows = np.arange(t.begin[i], t.end[i])
        hss.D[i] = h2.K(rows, rows)
        S = cholesky(hss.D[i], where=(1, i))           # A_ii = S_i S_i^T
        hss.S[i] = S
        Lam = solve_triangular(S, Y[1][rows], lower=True) if len(rows) else Y[1][rows]
        V, _, piv, r = qrcp(Lam, rank_cap, rel_tol)    # Alg. 2 step 3
        hss.V[i], hss.piv[i], hss.rank[i] = V, piv, r
        if keep_sketch:
            hss.Lam[i] = Lam
        Phi = solve_triangular(S, V, lower=True, trans='T').T if len(rows) else V.T   # V^T S^{-1}
        hss.Phi_leaf[i] = Phi
        if h2.active[i]:
            hss.PhiU[i] = Phi @ h2.E[i]                # Phi_i U_i^{H2}
        hss.U[i] = S @ V                               # U_i = S_i V_i
    t1, t3 = _pairs(lists, 1)
    for (i, j) in t1:                                  # V_i^T S_i^{-1} A_ij S_j^{-T} V_j (R10)
        ri = np.arange(t.begin[i], t.end[i])
        rj = np.arange(t.begin[j], t.end[j])
        hss.B[(i, j)] = hss.Phi_leaf[i] @ h2.K(ri, rj) @ hss.Phi_leaf[j].T
    for (i, j) in t3:                                  # (Phi U) B^{H2} (Phi U)^T
        hss.B[(i, j)] = hss.PhiU[i] @ h2.K(h2.skel[i], h2.skel[j], shift=False) @ hss.PhiU[j].T

    # ---- levels k = 2..L-1, then the root factor (R11)
    for k in range(2, L + 1):
        for i in t.nodes_at(k):
            Bii = _bold(hss, i, i)
            m = Bii.shape[0]
            if form == "eig":
                G, Gi = sym_sqrt_pair(Bii, where=(k, i))
                hss.F[i], hss.Finv[i] = G, Gi
            else:
                F = cholesky(np.eye(m) + Bii, where=(k, i))
                hss.F[i] = F
                hss.Finv[i] = solve_triangular(F, np.eye(m), lower=True) if m else F
        if k == L:
            break
        Lam = special_products(hss, Y[k], k)           # Alg. 3
        for i in t.nodes_at(k):
            Vb, _, piv, r = qrcp(Lam[i], rank_cap, rel_tol)
            hss.V[i], hss.piv[i], hss.rank[i] = Vb, piv, r
            if keep_sketch:
                hss.Lam[i] = Lam[i]
            left = Vb.T @ hss.Finv[i]                  # Vbar^T (I+B)^{-1/2}
            if h2.active[i]:
                c1, c2 = t.children(i)
                blk = np.zeros((hss.rank[c1] + hss.rank[c2], h2.rank[c1] + h2.rank[c2]))
                blk[:hss.rank[c1], :h2.rank[c1]] = hss.PhiU[c1]
                blk[hss.rank[c1]:, h2.rank[c1]:] = hss.PhiU[c2]
                hss.PhiU[i] = left @ blk @ h2.E[i]
            hss.R[i] = hss.F[i] @ Vb                   # R_i = (I+B)^{1/2} Vbar_i
        t1, t3 = _pairs(lists, k)
        for (i, j) in t1:                              # eqn:Mijk / P:1049
            li = hss.V[i].T @ hss.Finv[i]
            lj = hss.V[j].T @ hss.Finv[j]
            hss.B[(i, j)] = li @ _bold(hss, i, j) @ lj.T
        for (i, j) in t3:                              # eqn:type3_Mij / P:1051
            hss.B[(i, j)] = hss.PhiU[i] @ h2.K(h2.skel[i], h2.skel[j], shift=False) @ hss.PhiU[j].T
    return hss


# --------------------------------------------------------------------------- apply
def hss_matvec(hss: HSS, x):
    """y = H x with H = A^{(L-1)} (tree order)."""
    t = hss.h2.tree
    x = np.asarray(x, dtype=np.float64)
    vec = x.ndim == 1
    if vec:
        x = x[:, None]
    L = t.L
    y = np.zeros_like(x)
    if L == 1:
        y = hss.D[0] @ x
        return y[:, 0] if vec else y
    xh, yh = {}, {}
    for k in range(1, L):
        for i in t.nodes_at(k):
            if k == 1:
                xh[i] = hss.U[i].T @ x[t.begin[i]:t.end[i]]
            else:
                c1, c2 = t.children(i)
                xh[i] = hss.R[i].T @ np.vstack([xh[c1], xh[c2]])
            yh[i] = np.zeros_like(xh[i])
    for k in range(2, L + 1):                          # sibling couplings
        for p in t.nodes_at(k):
            c1, c2 = t.children(p)
            B = hss.Bij(c1, c2)
            yh[c1] += B @ xh[c2]
            yh[c2] += B.T @ xh[c1]
    for k in range(L - 1, 0, -1):
        for i in t.nodes_at(k):
            if k == 1:
                y[t.begin[i]:t.end[i]] = hss.D[i] @ x[t.begin[i]:t.end[i]] + hss.U[i] @ yh[i]
            else:
                c1, c2 = t.children(i)
                z = hss.R[i] @ yh[i]
                yh[c1] += z[:hss.rank[c1]]
                yh[c2] += z[hss.rank[c1]:]
    return y[:, 0] if vec else y


def hss_densify(hss: HSS):
    return hss_matvec(hss, np.eye(hss.h2.tree.N))


def hss_solve(hss: HSS, b):
    """x = H^{-1} b by the recursion of reading R12 (factors of Alg. 4)."""
    t = hss.h2.tree
    b = np.asarray(b, dtype=np.float64)
    vec = b.ndim == 1
    if vec:
        b = b[:, None]
    L = t.L
    if L == 1:
        S = hss.S[0]
        x = solve_triangular(S.T, solve_triangular(S, b, lower=True), lower=False)
        return x[:, 0] if vec else x
    z, zh, res = {}, {}, {}
    for i in t.nodes_at(1):                            # z = S^{-1} b, zh = V^T z
        bi = b[t.begin[i]:t.end[i]]
        z[i] = solve_triangular(hss.S[i], bi, lower=True) if bi.shape[0] else bi
        zh[i] = hss.V[i].T @ z[i]
        res[i] = z[i] - hss.V[i] @ zh[i]               # (I - V V^T) z
    u = {}
    for k in range(2, L):                              # u = F^{-1} [zh_c], zh = Vbar^T u
        for i in t.nodes_at(k):
            c1, c2 = t.children(i)
            u[i] = hss.Finv[i] @ np.vstack([zh[c1], zh[c2]])
            zh[i] = hss.V[i].T @ u[i]
            res[i] = u[i] - hss.V[i] @ zh[i]
    c1, c2 = t.children(0)                             # root: (F F^T)^{-1} [zh_c]
    g = hss.Finv[0] @ np.vstack([zh[c1], zh[c2]])
    xr = hss.Finv[0].T @ g
    xh = {c1: xr[:hss.rank[c1]], c2: xr[hss.rank[c1]:]}
    for k in range(L - 1, 1, -1):                      # out = F^{-T}[res + Vbar xh]
        for i in t.nodes_at(k):
            o = hss.Finv[i].T @ (res[i] + hss.V[i] @ xh[i])
            c1, c2 = t.children(i)
            xh[c1], xh[c2] = o[:hss.rank[c1]], o[hss.rank[c1]:]
    x = np.zeros_like(b)
    for i in t.nodes_at(1):                            # x = S^{-T}[res + V xh]
        v = res[i] + hss.V[i] @ xh[i]
        x[t.begin[i]:t.end[i]] = solve_triangular(hss.S[i].T, v, lower=False) if v.shape[0] else v
    return x[:, 0] if vec else x


def spdhss_build_adaptive(h2: H2, rel_tol, r0, r_max, omega_full, p=10, form="chol"):
    """Threshold-driven SPD HSS, restart form (reading R27): cap = r0,
    2 r0, ... <= r_max until every rank stops on |R_tt| <= tol |R_00| below the cap;
    Omega = the leading cap + p columns of omega_full.  Returns (HSS, cap)."""
    cap = r0
    while True:
        H = spdhss_build(h2, cap, rel_tol, omega_full[:, :cap + p], form=form)
        if max(H.rank.values(), default=0) < cap or cap >= r_max:
            return H, cap
        cap = min(2 * cap, r_max)


def block_jacobi_solve(h2: H2, b):
    """Block-Jacobi preconditioner: x_i = A_ii^{-1} b_i for every leaf i, by the
    Cholesky factor of A_ii (SPD-HSS = BJ's diagonal blocks + off-diagonal
    approximations).  b, x in tree order."""
    t = h2.tree
    b = np.asarray(b, dtype=np.float64)
    x = np.empty_like(b)
    for i in t.nodes_at(1):
        rows = np.arange(t.begin[i], t.end[i])
        S = cholesky(h2.K(rows, rows), where=f"leaf {i}")
        x[rows] = solve_triangular(S, solve_triangular(S, b[rows], lower=True), lower=True, trans="T")
    return x


def pcg(apply_A, apply_M, b, tol, maxit):
    """Preconditioned CG (R15).  Returns (x, iters, converged, relres_hist)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return x, 0, True, [0.0]
    r = b.copy()
    z = apply_M(r)
    p = z.copy()
    rz = r @ z
    hist = [1.0]
    for it in range(1, maxit + 1):
        q = apply_A(p)
        pq = p @ q
        if not pq > 0.0:
            raise NotPD(f"PCG breakdown: p^T A p = {pq:.3e}", it, pq)
        alpha = rz / pq
        x += alpha * p
        r -= alpha * q
        rel = np.linalg.norm(r) / nb
        hist.append(rel)
        if rel <= tol:
            return x, it, True, hist
        z = apply_M(r)
        rz_new = r @ z
        if not rz_new > 0.0:
            raise NotPD(f"PCG breakdown: r^T M r = {rz_new:.3e}", it, rz_new)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, maxit, False, hist


def hss_error(hss: HSS, probes):
    """Fig. 5 metric: mean_j ||H_hss x_j - H_h2 x_j|| / ||H_h2 x_j||."""
    errs = []
    for x in probes.T:
        ref = h2_matvec(hss.h2, x)
        errs.append(np.linalg.norm(hss_matvec(hss, x) - ref) / np.linalg.norm(ref))
    return float(np.mean(errs))


# --------------------------------------------------------------------------- Alg. 1
def alg1_generalized(A, tree, V_leaf, Vbar):
    """Alg. 1 on a dense SPD matrix A (tree order) with injected
    bases V_i (leaf) and Vbar_i (nonleaf, eig form).  Computes B_ij for ALL
    same-level pairs i != j and R_i.  Returns dicts B[(i,j)], R[i]."""
    L = tree.L
    S, B, R, Gi, G = {}, {}, {}, {}, {}
    lv1 = tree.nodes_at(1)
    for i in lv1:
        ri = slice(tree.begin[i], tree.end[i])
        S[i] = cholesky(A[ri, ri])
    for i in lv1:
        for j in lv1:
            if i == j:
                continue
            ri = slice(tree.begin[i], tree.end[i])
            rj = slice(tree.begin[j], tree.end[j])
            C = solve_triangular(S[i], solve_triangular(S[j], A[ri, rj].T, lower=True).T, lower=True)
            B[(i, j)] = V_leaf[i].T @ C @ V_leaf[j]    # B_ij = V_i^T C_ij V_j
    rank = {i: V_leaf[i].shape[1] for i in lv1}
    for k in range(2, L):
        lvk = tree.nodes_at(k)
        for i in lvk:
            c1, c2 = tree.children(i)
            Bii = np.block([[np.zeros((rank[c1], rank[c1])), B[(c1, c2)]],
                            [B[(c2, c1)], np.zeros((rank[c2], rank[c2]))]])
            G[i], Gi[i] = sym_sqrt_pair(Bii)
            rank[i] = Vbar[i].shape[1]
        for i in lvk:
            for j in lvk:
                if i == j:
                    continue
                ci, cj = tree.children(i), tree.children(j)
                Bij = np.block([[B[(a, b)] for b in cj] for a in ci])
                B[(i, j)] = Vbar[i].T @ Gi[i] @ Bij @ Gi[j] @ Vbar[j]
        for i in lvk:
            R[i] = G[i] @ Vbar[i]
    return B, R
