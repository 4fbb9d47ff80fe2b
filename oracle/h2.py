"""H2 representation by proxy-point interpolative decomposition (oracle O3/O4).
TEST INFRASTRUCTURE ONLY.

Structure (§5.1, eqn:uniformbasis_h2 P:667-671):
  A_ij = U_i B_ij U_j^T for Type-3 pairs, dense near leaf blocks,
  nested bases U_i = blockdiag(U_children) R_i (eqn:nested P:218-226).
Construction: the paper delegates to H2Pack's "proxy point method"
 and gives no algorithm; this follows readings R3/R4:

R3  proxies for node i: a Halton sequence (bases 2,3[,5]; index k = 1, 2, ...;
    radical inverse computed as an exact integer ratio), n_p/2 points mapped
    into the local shell box  c_i +- 3 max(e_i)  and n_p - n_p/2 points mapped
    into the root bbox expanded by 10% of its largest extent; a point is
    rejected if it lies strictly inside the inner box [lo_i - ehat_i,
    hi_i + ehat_i] (which R2 guarantees to hold no far-field point).  The
    domain group scans at most 64 n_p indices; any shortfall is filled by
    continuing the shell sequence.  Only nodes that have a Type-3 partner at
    their own or an ancestor level ("active" nodes) are compressed.
R4  row ID of M = K(X_cand, Y_proxy) by QRCP of M^T with rel tol tau:
    skeleton J = cand[piv[:s]], interpolation E (n_c x s) with
    E[piv[:s]] = I and E[piv[s+k]] = (R11^{-1} R12)[:, k]^T, so M ~= E M[J].

All index sets are TREE POSITIONS (rows of X[perm]).
"""
from dataclasses import dataclass, field
import numpy as np
from scipy.linalg import solve_triangular

from .kernels import kernel_matrix, dofs_per_point, dof_points
from .linalg import qrcp
from .tree import Tree, Lists, build_tree, interaction_lists, expand_dofs

HALTON_BASES = (2, 3, 5)


def halton(k: int, base: int) -> float:
    """Radical inverse of k in `base` as an exact integer ratio num/den."""
    num, den = 0, 1
    while k > 0:
        den *= base
        num = num * base + (k % base)
        k //= base
    return num / den


def _map(box_lo, box_hi, k, d):
    width = [box_hi[a] - box_lo[a] for a in range(d)]
    return [box_lo[a] + halton(k, HALTON_BASES[a]) * width[a] for a in range(d)]


def _inside(p, ilo, ihi, d):
    return all(ilo[a] < p[a] < ihi[a] for a in range(d))


def proxy_points(tree: Tree, i: int, n_proxy: int):
    """Proxy point set of node i (reading R3)."""
    d = tree.d
    lo, hi = tree.lo[i], tree.hi[i]
    e = [0.5 * (hi[a] - lo[a]) for a in range(d)]
    emax = max(e)
    ehat = [max(e[a], 0.25 * emax) for a in range(d)]
    ilo = [lo[a] - ehat[a] for a in range(d)]
    ihi = [hi[a] + ehat[a] for a in range(d)]
    c = [0.5 * (lo[a] + hi[a]) for a in range(d)]
    t3 = 3.0 * emax
    slo = [c[a] - t3 for a in range(d)]
    shi = [c[a] + t3 for a in range(d)]
    rlo, rhi = tree.lo[0], tree.hi[0]
    ext = 0.1 * max(rhi[a] - rlo[a] for a in range(d))
    dlo = [rlo[a] - ext for a in range(d)]
    dhi = [rhi[a] + ext for a in range(d)]

    n_shell = n_proxy // 2
    n_dom = n_proxy - n_shell
    pts = []
    k = 0
    while len(pts) < n_shell:
        k += 1
        p = _map(slo, shi, k, d)
        if not _inside(p, ilo, ihi, d):
            pts.append(p)
    k_shell = k
    got = 0
    for kk in range(1, 64 * n_proxy + 1):
        if got == n_dom:
            break
        p = _map(dlo, dhi, kk, d)
        if not _inside(p, ilo, ihi, d):
            pts.append(p)
            got += 1
    k = k_shell
    while got < n_dom:                 # shortfall: continue the shell sequence
        k += 1
        p = _map(slo, shi, k, d)
        if not _inside(p, ilo, ihi, d):
            pts.append(p)
            got += 1
    return np.array(pts, dtype=np.float64)


@dataclass
class H2:
    tree: Tree
    lists: Lists
    Xt: np.ndarray          # points in tree order
    kid: int
    ell: float
    shift: float
    tol: float
    n_proxy: int
    active: np.ndarray      # bool per node
    skel: dict = field(default_factory=dict)   # node -> tree positions (skeleton J_i)
    E: dict = field(default_factory=dict)      # node -> leaf U_i or nonleaf R_i
    piv: dict = field(default_factory=dict)    # node -> QRCP pivots over candidates
    rank: dict = field(default_factory=dict)
    blocks: dict = field(default_factory=dict)  # cache of evaluated near / coupling blocks (R21)

    def block(self, key, rows, cols, shift=True):
        """K(rows, cols) of a near block (key ("n", a, b)) or coupling (("c", i, j)),
        evaluated once and kept: reading R21 lets the oracle store what the device
        evaluates on the fly; the entries are the same function of the same points."""
        B = self.blocks.get(key)
        if B is None:
            B = self.K(rows, cols, shift)
            self.blocks[key] = B
        return B

    def K(self, rows, cols, shift=True):
        return kernel_matrix(self.kid, self.ell, self.Xt[rows], self.Xt[cols],
                             self.shift if shift else 0.0, rows, cols)

    def candidates(self, i):
        t = self.tree
        if t.is_leaf(i):
            return np.arange(t.begin[i], t.end[i])
        c1, c2 = t.children(i)
        return np.concatenate([self.skel[c1], self.skel[c2]])


def active_nodes(tree: Tree, lists: Lists):
    """Nodes with a Type-3 partner at their own or an ancestor level."""
    act = np.zeros(tree.nnodes, bool)
    for k in range(1, tree.L + 1):
        for (i, j) in lists.type3[k]:
            act[i] = True
    for i in range(1, tree.nnodes):          # heap order: parents first
        if act[(i - 1) // 2]:
            act[i] = True
    act[0] = False
    return act


def default_n_proxy(d):
    return 4096 if d == 2 else 6144


def h2_build(X, kid, ell, shift, leaf, tol, n_proxy=0):
    """H2 by proxy-point ID, bottom-up (R3, R4).  Tensor kernels (RPY, R28): the tree
    is built on the points (leaf = points per leaf), then every index set, proxy set
    and skeleton is over degrees of freedom (dof rows (x, y, z, c))."""
    m = dofs_per_point(kid)
    tree = build_tree(X, leaf)
    lists = interaction_lists(tree)
    tree = expand_dofs(tree, m)
    Xd = np.asarray(X, dtype=np.float64) if m == 1 else dof_points(X, m)
    Xt = Xd[tree.perm]
    n_proxy = n_proxy or default_n_proxy(tree.d)
    h = H2(tree, lists, Xt, kid, ell, shift, tol, n_proxy, active_nodes(tree, lists))
    for k in range(1, tree.L):
        for i in tree.nodes_at(k):
            if not h.active[i]:
                h.skel[i] = np.zeros(0, np.int64)
                continue
            cand = h.candidates(i)
            Y = proxy_points(tree, i, n_proxy)
            if m > 1:
                Y = dof_points(Y, m)                        # proxy dofs (R28)
            M = kernel_matrix(kid, ell, Xt[cand], Y)       # n_c x n_p, no shift
            _, R, piv, s = qrcp(M.T, min(M.shape), tol, want_q=False)
            T = solve_triangular(R[:s, :s], R[:s, s:]) if s > 0 else np.zeros((0, len(cand) - s))
            E = np.zeros((len(cand), s))
            E[piv[:s], np.arange(s)] = 1.0
            E[piv[s:], :] = T.T
            h.skel[i] = cand[piv[:s]]
            h.E[i] = E
            h.piv[i] = piv
            h.rank[i] = s
    return h


def h2_matvec(h: H2, x, exclude_level=0, reverse=False, shuffle=None):
    """y = A x for the H2 matrix A (tree order), x: (N, w).

    exclude_level = k > 0 gives the literal Y^(k) = (A - blockdiag_k(A)) x of
    eqn:Yk: every H2 block whose row and column sets share a
    level-k ancestor (LCA level <= k) is skipped, "just neglecting the block
    diagonal parts during multiplication".
    Up pass / coupling / down pass follow eqn:uniformbasis_h2 + eqn:nested.
    reverse=True accumulates the near blocks and the couplings in the reverse list
    order, shuffle=<seed> in a seeded random order: the same sum in another order
    (the drift evidence of reading R24).
    """
    t, lists = h.tree, h.lists
    x = np.asarray(x, dtype=np.float64)
    vec = x.ndim == 1
    if vec:
        x = x[:, None]
    w = x.shape[1]
    y = np.zeros_like(x)
    keep = (lambda i, j: True) if exclude_level <= 0 else \
        (lambda i, j: lists.lca[(i, j)] > exclude_level)
    # near field (dense leaf blocks, shift on the diagonal)
    def order(lst):
        if shuffle is not None:
            return [lst[q] for q in np.random.default_rng(shuffle).permutation(len(lst))]
        return reversed(lst) if reverse else lst

    for (a, b) in order(lists.near):
        if keep(a, b):
            ra = np.arange(t.begin[a], t.end[a])
            rb = np.arange(t.begin[b], t.end[b])
            y[ra] += h.block(("n", a, b), ra, rb) @ x[rb]
    # up pass: xh_i = U_i^T x_i (leaf), R_i^T [xh_c1; xh_c2] (nonleaf)
    xh = {}
    for k in range(1, t.L):
        for i in t.nodes_at(k):
            if not h.active[i]:
                continue
            if k == 1:
                xh[i] = h.E[i].T @ x[t.begin[i]:t.end[i]]
            else:
                c1, c2 = t.children(i)
                xh[i] = h.E[i].T @ np.vstack([xh[c1], xh[c2]])
    # coupling: yh_i += K(J_i, J_j) xh_j over Type-3 pairs
    yh = {i: np.zeros((h.rank[i], w)) for i in xh}
    for k in range(1, t.L):
        for (i, j) in order(lists.type3[k]):
            if keep(i, j):
                yh[i] += h.block(("c", i, j), h.skel[i], h.skel[j], shift=False) @ xh[j]
    # down pass
    for k in range(t.L - 1, 0, -1):
        for i in t.nodes_at(k):
            if not h.active[i]:
                continue
            if k == 1:
                y[t.begin[i]:t.end[i]] += h.E[i] @ yh[i]
            else:
                c1, c2 = t.children(i)
                z = h.E[i] @ yh[i]
                s1 = h.rank[c1]
                yh[c1] += z[:s1]
                yh[c2] += z[s1:]
    return y[:, 0] if vec else y


def h2_densify(h: H2, exclude_level=0):
    return h2_matvec(h, np.eye(h.tree.N), exclude_level)
