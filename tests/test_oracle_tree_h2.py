"""Pins of the oracle's tree, lists and H2 (O2-O4) by invariants, brute force
and the dense kernel matrix.  CPU only."""
import itertools

import numpy as np
import pytest

import oracle
import synth
from oracle.kernels import kernel_matrix
from oracle.tree import far


def _pts(n, d, seed=0, sphere=False):
    rng = np.random.default_rng(seed)
    if sphere:
        g = rng.standard_normal((n, 3))
        return g / np.linalg.norm(g, axis=1, keepdims=True)
    return rng.random((n, d))


@pytest.mark.parametrize("n,d,leaf,sphere", [(256, 2, 16, False), (300, 3, 16, False),
                                             (512, 3, 32, True), (37, 2, 8, False), (10, 2, 16, False)])
def test_tree_invariants(n, d, leaf, sphere):
    X = _pts(n, d, 1, sphere)
    t = oracle.build_tree(X, leaf)
    assert sorted(t.perm.tolist()) == list(range(n))
    assert t.L == (1 if n <= leaf else int(np.ceil(np.log2(n / leaf))) + 1)
    leaves = t.nodes_at(1)
    assert t.begin[leaves[0]] == 0 and t.end[leaves[-1]] == n
    for a, b in zip(leaves[:-1], leaves[1:]):
        assert t.end[a] == t.begin[b]
    assert all(0 < t.size(i) <= leaf for i in leaves)
    for i in range(t.nnodes):
        P = X[t.perm[t.begin[i]:t.end[i]]]
        np.testing.assert_array_equal(P.min(0), t.lo[i])       # tight boxes
        np.testing.assert_array_equal(P.max(0), t.hi[i])
        if not t.is_leaf(i):
            c1, c2 = t.children(i)
            assert t.begin[c1] == t.begin[i] and t.end[c2] == t.end[i] and t.end[c1] == t.begin[c2]
            assert t.size(c1) - t.size(c2) in (0, 1)              # left takes ceil(n/2)
            sd = int(np.argmax(t.hi[i] - t.lo[i]))
            assert X[t.perm[t.begin[c1]:t.end[c1]], sd].max() <= X[t.perm[t.begin[c2]:t.end[c2]], sd].min()


@pytest.mark.parametrize("n,d,leaf,sphere", [(256, 2, 16, False), (384, 3, 12, False), (512, 3, 16, True)])
def test_lists_cover_every_entry_exactly_once(n, d, leaf, sphere):
    X = _pts(n, d, 2, sphere)
    t = oracle.build_tree(X, leaf)
    li = oracle.interaction_lists(t)
    cover = np.zeros((n, n), np.int32)
    for (a, b) in li.near:
        cover[t.begin[a]:t.end[a], t.begin[b]:t.end[b]] += 1
    for k in range(1, t.L + 1):
        for (i, j) in li.type3[k]:
            cover[t.begin[i]:t.end[i], t.begin[j]:t.end[j]] += 1
            assert far(t, i, j) and not far(t, t.parent(i), t.parent(j))
    assert (cover == 1).all()
    # symmetry of every list
    assert set(li.near) == {(b, a) for (a, b) in li.near}
    for k in li.type3:
        assert set(li.type3[k]) == {(j, i) for (i, j) in li.type3[k]}
        assert set(li.type1[k]) == {(j, i) for (i, j) in li.type1[k]}


def test_admissibility_symmetric_monotone_and_separating():
    X = _pts(512, 3, 3)
    t = oracle.build_tree(X, 16)
    for k in range(1, t.L):
        nodes = t.nodes_at(k)
        for i, j in itertools.combinations(nodes, 2):
            fij = far(t, i, j)
            assert fij == far(t, j, i)
            if fij and k > 1:                     # far parents -> far children
                for a in t.children(i):
                    for b in t.children(j):
                        assert far(t, a, b)
            if fij:                               # every point of j outside i's inner box (R2, R3)
                e = 0.5 * (t.hi[i] - t.lo[i])
                eh = np.maximum(e, 0.25 * e.max())
                P = X[t.perm[t.begin[j]:t.end[j]]]
                inside = ((P > t.lo[i] - eh) & (P < t.hi[i] + eh)).all(axis=1)
                assert not inside.any()


def test_lca_levels_by_ancestor_sets():
    t = oracle.build_tree(_pts(256, 2, 4), 16)
    def anc(i):
        out = [i]
        while i > 0:
            i = (i - 1) // 2
            out.append(i)
        return out
    for i, j in itertools.product(t.nodes_at(1), repeat=2):
        common = [a for a in anc(i) if a in anc(j)][0]
        assert t.lca_level(i, j) == t.level(common)


# ---------------------------------------------------------------- H2 (O3, O4)
def _small_h2(cfgname="C1", n=512, leaf=None, tol=1e-10):
    cfg = synth.CONFIGS[cfgname].scaled(n, **({"leaf": leaf} if leaf else {}))
    X = synth.points(cfg)
    return cfg, oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, tol)


def _dense(h):
    r = np.arange(h.tree.N)
    return kernel_matrix(h.kid, h.ell, h.Xt, h.Xt, h.shift, r, r)


def test_proxies_avoid_inner_box():
    cfg, h = _small_h2("C2", 1024, leaf=32)
    t = h.tree
    for i in [1, 5, 20, 40]:
        Y = oracle.proxy_points(t, i, 512)
        assert Y.shape == (512, 3)
        e = 0.5 * (t.hi[i] - t.lo[i])
        eh = np.maximum(e, 0.25 * e.max())
        inside = ((Y > t.lo[i] - eh) & (Y < t.hi[i] + eh)).all(axis=1)
        assert not inside.any()


def _expanded_U(h, i):
    """Dense |I_i| x s_i basis from the nested transfers (eqn:nested)."""
    t = h.tree
    if t.is_leaf(i):
        return h.E[i]
    c1, c2 = t.children(i)
    U1, U2 = _expanded_U(h, c1), _expanded_U(h, c2)
    blk = np.zeros((U1.shape[0] + U2.shape[0], U1.shape[1] + U2.shape[1]))
    blk[:U1.shape[0], :U1.shape[1]] = U1
    blk[U1.shape[0]:, U1.shape[1]:] = U2
    return blk @ h.E[i]


@pytest.mark.parametrize("cfgname,n,leaf", [("C1", 1024, 64), ("C2", 2048, 64), ("C3", 2048, 64)])
def test_h2_accuracy_and_block_assembly(cfgname, n, leaf):
    cfg, h = _small_h2(cfgname, n, leaf)
    t = h.tree
    A = _dense(h)
    Ah = oracle.h2_densify(h)
    # H2 error against the dense kernel matrix <= 10 tol
    assert np.linalg.norm(Ah - A) <= 10 * cfg.h2_tol * np.linalg.norm(A)
    # independent assembly: near blocks + expanded U_i B_ij U_j^T over Type-3 pairs
    B = np.zeros_like(A)
    for (a, b) in h.lists.near:
        ra, rb = slice(t.begin[a], t.end[a]), slice(t.begin[b], t.end[b])
        B[ra, rb] = A[ra, rb]
    for k in range(1, t.L):
        for (i, j) in h.lists.type3[k]:
            Ui, Uj = _expanded_U(h, i), _expanded_U(h, j)
            Bij = kernel_matrix(h.kid, h.ell, h.Xt[h.skel[i]], h.Xt[h.skel[j]])
            B[t.begin[i]:t.end[i], t.begin[j]:t.end[j]] = Ui @ Bij @ Uj.T
    np.testing.assert_allclose(Ah, B, atol=1e-13 * np.abs(A).max())
    # interpolation structure: identity rows at the skeleton, nested skeletons
    for i, E in h.E.items():
        s = h.rank[i]
        np.testing.assert_array_equal(E[h.piv[i][:s]], np.eye(s))
        if not t.is_leaf(i):
            c1, c2 = t.children(i)
            assert set(h.skel[i]) <= set(h.skel[c1]) | set(h.skel[c2])


def test_level_excluded_products_match_dense_masking():
    cfg, h = _small_h2("C1", 1024, 32)
    t = h.tree
    Ah = oracle.h2_densify(h)
    Om = synth.omega(cfg, w=7)
    assert t.L >= 4
    for k in range(1, t.L):
        D = np.zeros_like(Ah)
        for i in t.nodes_at(k):
            r = slice(t.begin[i], t.end[i])
            D[r, r] = Ah[r, r]
        Yk = oracle.h2_matvec(h, Om, exclude_level=k)
        np.testing.assert_allclose(Yk, (Ah - D) @ Om, atol=1e-12 * np.abs(Ah @ Om).max())
