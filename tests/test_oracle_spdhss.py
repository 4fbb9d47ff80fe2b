"""Pins of the oracle's Alg. 4 construction, HSS solve and PCG (O5-O12)
against the paper's identities, Alg. 1, special cases and dense algebra."""
import numpy as np
import pytest
from scipy.linalg import solve_triangular

import oracle
import synth
from oracle.kernels import kernel_matrix


def _build(cfgname="C1", n=512, leaf=None, cap=None, tol=None, w=None, form="eig", ell=None):
    kw = {}
    if leaf:
        kw["leaf"] = leaf
    if cap:
        kw["rank_cap"] = cap
    if tol is not None:
        kw["hss_tol"] = tol
    if ell is not None:
        kw["ell"] = ell
    cfg = synth.CONFIGS[cfgname].scaled(n, **kw)
    X = synth.points(cfg)
    h = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    om = synth.omega(cfg, w=w or cfg.w)
    H = oracle.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, om, form=form)
    return cfg, h, om, H


@pytest.fixture(scope="module")
def c1small():
    return _build("C1", 1024, leaf=32, cap=20)


def _phi_dense(H, i):
    """Phi_i materialized by eqn:phi: leaf V^T S^{-1},
    nonleaf Vbar^T (I+B)^{-1/2} blockdiag(Phi_c)."""
    t = H.h2.tree
    if t.is_leaf(i):
        return H.V[i].T @ np.linalg.inv(H.S[i])
    c1, c2 = t.children(i)
    P1, P2 = _phi_dense(H, c1), _phi_dense(H, c2)
    blk = np.zeros((P1.shape[0] + P2.shape[0], P1.shape[1] + P2.shape[1]))
    blk[:P1.shape[0], :P1.shape[1]] = P1
    blk[P1.shape[0]:, P1.shape[1]:] = P2
    return H.V[i].T @ H.Finv[i] @ blk


def test_spd_and_symmetric(c1small):
    cfg, h, om, H = c1small
    Hd = oracle.hss_densify(H)
    assert np.abs(Hd - Hd.T).max() <= 1e-13 * np.abs(Hd).max()
    np.linalg.cholesky(0.5 * (Hd + Hd.T))
    assert np.linalg.eigvalsh(0.5 * (Hd + Hd.T)).min() > 0
    assert H.sketch_widths == [cfg.w] * (h.tree.L - 1)      # exactly L-1 groups of r+p


def test_bij_equals_phi_A_phi(c1small):
    """B_ij = Phi_i A_ij Phi_j^T (eqn:bij_hss) for every Type-1 and
    Type-3 pair at every level, A = the H2 matrix."""
    cfg, h, om, H = c1small
    t = h.tree
    A = oracle.h2_densify(h)
    n_checked = 0
    for k in range(1, t.L):
        for (i, j) in h.lists.type1[k] + h.lists.type3[k]:
            if i >= j:
                continue
            Pi, Pj = _phi_dense(H, i), _phi_dense(H, j)
            want = Pi @ A[t.begin[i]:t.end[i], t.begin[j]:t.end[j]] @ Pj.T
            np.testing.assert_allclose(H.B[(i, j)], want, atol=1e-10 * max(1, np.abs(want).max()))
            n_checked += 1
    assert n_checked > 50


def test_sketches_are_lambda_times_omega(c1small):
    """Alg. 3 output = Lambda_{ii^c} Omega_{i^c}: leaf S^{-1} A_{ii^c} Omega,
    nonleaf (I+B)^{-1/2} blockdiag(Phi_c) A_{ii^c} Omega, with dense A and Phi."""
    cfg, h, om, H = c1small
    t = h.tree
    A = oracle.h2_densify(h)
    for k in range(2, t.L):
        Yk = oracle.h2_matvec(h, om, exclude_level=k)
        lam = oracle.special_products(H, Yk, k)
        for i in t.nodes_at(k):
            r = slice(t.begin[i], t.end[i])
            Ao = A[r] @ om - A[r, r] @ om[r]
            c1, c2 = t.children(i)
            P1, P2 = _phi_dense(H, c1), _phi_dense(H, c2)
            blk = np.zeros((P1.shape[0] + P2.shape[0], P1.shape[1] + P2.shape[1]))
            blk[:P1.shape[0], :P1.shape[1]] = P1
            blk[P1.shape[0]:, P1.shape[1]:] = P2
            np.testing.assert_allclose(lam[i], H.Finv[i] @ blk @ Ao, atol=1e-10 * np.abs(lam[i]).max())


def test_alg1_with_injected_bases_equals_alg4(c1small):
    """Alg. 1 (quadratic, dense) fed the bases Alg. 4 chose reproduces Alg. 4's
    sibling B_ij and R_i."""
    cfg, h, om, H = c1small
    t = h.tree
    A = oracle.h2_densify(h)
    Vleaf = {i: H.V[i] for i in t.nodes_at(1)}
    Vbar = {i: H.V[i] for k in range(2, t.L) for i in t.nodes_at(k)}
    B1, R1 = oracle.alg1_generalized(A, t, Vleaf, Vbar)
    for k in range(2, t.L + 1):
        for p in t.nodes_at(k):
            c1, c2 = t.children(p)
            want = B1[(c1, c2)]
            np.testing.assert_allclose(H.Bij(c1, c2), want, atol=1e-10 * max(1, np.abs(want).max()))
    for i, R in R1.items():
        np.testing.assert_allclose(H.R[i], R, atol=1e-10)


def test_eig_and_cholesky_forms_agree():
    """Reading R9: R_i, B_ij and the HSS matrix are identical (to rounding)."""
    _, h, om, He = _build("C1", 512, leaf=32, cap=20, form="eig")
    _, _, _, Hc = _build("C1", 512, leaf=32, cap=20, form="chol")
    assert He.rank == Hc.rank
    for key in He.B:
        np.testing.assert_allclose(Hc.B[key], He.B[key], atol=1e-11)
    for key in He.R:
        np.testing.assert_allclose(Hc.R[key], He.R[key], atol=1e-11)
    np.testing.assert_allclose(oracle.hss_densify(Hc), oracle.hss_densify(He), atol=1e-12)


def test_level_two_spd_formula():
    """For L = 2, A^(1) = diag(U W) A diag(U W)^T + diag(S (I - V V^T) S^T)
    with W_i = V_i^T S_i^{-1}."""
    cfg, h, om, H = _build("C1", 128, leaf=64, cap=20)
    t = h.tree
    assert t.L == 2
    A = oracle.h2_densify(h)
    UW = np.zeros_like(A)
    Dg = np.zeros_like(A)
    for i in t.nodes_at(1):
        r = slice(t.begin[i], t.end[i])
        W = H.V[i].T @ np.linalg.inv(H.S[i])
        UW[r, r] = H.U[i] @ W
        Dg[r, r] = H.S[i] @ (np.eye(t.size(i)) - H.V[i] @ H.V[i].T) @ H.S[i].T
    np.testing.assert_allclose(oracle.hss_densify(H), UW @ A @ UW.T + Dg, atol=1e-12 * np.abs(A).max())


def test_no_truncation_reproduces_h2_and_solve_is_inverse():
    """Textbook special case: full ranks (cap >= sizes, tol 0, w = N) make the
    HSS equal to the H2 matrix; the solve is then A^{-1} (LAPACK)."""
    cfg, h, om, H = _build("C1", 128, leaf=16, cap=128, tol=0.0, w=128)
    A = oracle.h2_densify(h)
    Hd = oracle.hss_densify(H)
    np.testing.assert_allclose(Hd, A, atol=1e-12 * np.abs(A).max())
    b = synth.rhs(cfg)
    np.testing.assert_allclose(oracle.hss_solve(H, b), np.linalg.solve(A, b), rtol=1e-8)
    # PCG with the exact preconditioner converges in 1-2 iterations
    x, it, conv, _ = oracle.pcg(lambda v: A @ v, lambda v: oracle.hss_solve(H, v), b, 1e-8, 100)
    assert conv and it <= 2


def test_identity_like_kernel_gives_rank_zero():
    """l -> 0: off-diagonal kernel entries underflow to 0, so every sketch is
    zero, all ranks are 0 and the HSS is (1+sigma) I exactly."""
    cfg, h, om, H = _build("C1", 256, leaf=32, cap=20, ell=1e-6)
    assert all(r == 0 for r in H.rank.values())
    np.testing.assert_array_equal(oracle.hss_densify(H), (1 + cfg.shift) * np.eye(256))


def test_hss_solve_residual_symmetry_positivity(c1small):
    cfg, h, om, H = c1small
    rng = np.random.default_rng(9)
    b = rng.standard_normal(h.tree.N)
    x = oracle.hss_solve(H, b)
    assert np.linalg.norm(oracle.hss_matvec(H, x) - b) <= 1e-10 * np.linalg.norm(b)
    y = rng.standard_normal(h.tree.N)
    sx, sy = oracle.hss_solve(H, y), x
    assert abs(b @ sx - y @ sy) <= 1e-10 * abs(b @ sx)
    for _ in range(5):
        v = rng.standard_normal(h.tree.N)
        assert v @ oracle.hss_solve(H, v) > 0
    # block version equals column-by-column
    Bm = rng.standard_normal((h.tree.N, 3))
    np.testing.assert_allclose(oracle.hss_solve(H, Bm)[:, 1], oracle.hss_solve(H, Bm[:, 1]), rtol=0, atol=1e-12 * np.abs(sx).max())


def test_pcg_textbook_cases():
    b = np.random.default_rng(3).standard_normal(10)
    x, it, conv, _ = oracle.pcg(lambda v: v, lambda v: v, b, 1e-12, 10)
    assert it == 1 and conv
    D = np.arange(1.0, 11.0)
    x, it, conv, _ = oracle.pcg(lambda v: D * v, lambda v: v / D, b, 1e-12, 10)
    assert it == 1 and conv
    rng = np.random.default_rng(4)
    Q, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    A = (Q * np.linspace(1, 50, 30)) @ Q.T
    x, it, conv, _ = oracle.pcg(lambda v: A @ v, lambda v: v, b := rng.standard_normal(30), 1e-12, 200)
    assert conv and it <= 60
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-9)


def test_spdhss_preconditions_better_than_none(c1small):
    cfg, h, om, H = c1small
    b = synth.rhs(cfg.scaled(h.tree.N))
    _, it_p, cp, _ = oracle.pcg(lambda v: oracle.h2_matvec(h, v), lambda v: oracle.hss_solve(H, v), b, 1e-8, 3000)
    _, it_n, cn, _ = oracle.pcg(lambda v: oracle.h2_matvec(h, v), lambda v: v, b, 1e-8, 3000)
    assert cp and it_p < it_n
    err = oracle.hss_error(H, synth.multivec(h.tree.N, 10, seed=5))
    assert 0 < err < 0.5


def test_block_jacobi_pins(c1small):
    """BJ baseline: on a block-diagonal matrix it is the exact
    inverse; it equals the SPD-HSS solve with all off-diagonal ranks forced to 0
    (identity-like kernel); and the paper's ordering none > BJ > SPD-HSS in
    iterations holds (Table 1 rows "Unpreconditioned", "BJ", "SPDHSS")."""
    cfg, h, om, H = c1small
    t = h.tree
    rng = np.random.default_rng(12)
    x = rng.standard_normal(t.N)
    # block-diagonal A: blocks A_ii of the leaves, applied densely
    Ax = np.zeros_like(x)
    for i in t.nodes_at(1):
        r = np.arange(t.begin[i], t.end[i])
        Ax[r] = h.K(r, r) @ x[r]
    np.testing.assert_allclose(oracle.block_jacobi_solve(h, Ax), x, rtol=0, atol=1e-9 * np.abs(x).max())
    # identity-like kernel: HSS ranks are 0, so SPD-HSS == BJ
    cfg2, h2, om2, H2 = _build("C1", 256, leaf=32, cap=20, ell=1e-6)
    b2 = rng.standard_normal(256)
    np.testing.assert_allclose(oracle.block_jacobi_solve(h2, b2), oracle.hss_solve(H2, b2), rtol=1e-13)
    b = synth.rhs(cfg.scaled(t.N))
    A = lambda v: oracle.h2_matvec(h, v)
    _, it_h, ch, _ = oracle.pcg(A, lambda v: oracle.hss_solve(H, v), b, 1e-8, 3000)
    _, it_b, cb, _ = oracle.pcg(A, lambda v: oracle.block_jacobi_solve(h, v), b, 1e-8, 3000)
    _, it_n, cn, _ = oracle.pcg(A, lambda v: v, b, 1e-8, 3000)
    assert ch and cb and it_h < it_b < it_n


def test_adaptive_threshold_build():
    """P:998-999 (restart form, R27): the chosen cap is the first in r0, 2 r0, ...
    at which every sketch compression stops on the threshold; the previous cap did
    not; the error metric does not increase; and a threshold below
    rounding with a cap above the node sizes reproduces the H2 exactly."""
    cfg = synth.C1.scaled(512, leaf=32)
    X = synth.points(cfg)
    h = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    om = synth.omega(cfg, w=64 + 10)
    H, cap = oracle.spdhss_build_adaptive(h, 1e-3, 4, 64, om)
    assert max(H.rank.values()) < cap and cap > 4
    Hprev = oracle.spdhss_build(h, cap // 2, 1e-3, om[:, :cap // 2 + 10], form="chol")
    assert max(Hprev.rank.values()) == cap // 2
    probes = synth.multivec(512, 6, seed=3)
    assert oracle.hss_error(H, probes) <= oracle.hss_error(Hprev, probes)
    # no truncation: tol below rounding, cap above every node's rows -> HSS == H2
    cfg2 = synth.C1.scaled(128, leaf=32)
    X2 = synth.points(cfg2)
    h2 = oracle.h2_build(X2, cfg2.kernel, cfg2.ell, cfg2.shift, cfg2.leaf, 1e-14)
    om2 = synth.omega(cfg2, w=128 + 10)
    H2, cap2 = oracle.spdhss_build_adaptive(h2, 1e-15, 8, 128, om2)
    Ad = oracle.h2_densify(h2)
    np.testing.assert_allclose(oracle.hss_densify(H2), Ad, atol=1e-11 * np.abs(Ad).max())
