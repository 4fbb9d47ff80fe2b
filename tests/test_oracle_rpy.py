"""Pins of the oracle's RPY tensor kernel and its degree-of-freedom expansion
(reading R28).  CPU only.

The RPY tensor is pinned by closed forms and known properties, not by re-typing
its formula: hand-evaluated entries on each branch, K(0) = I/a, continuity at
|r| = 2a (fails for the printed near branch unless a = 1: reading R28), the
Oseen far-field limit 3/(4r)(I + rhat rhat^T), rotation equivariance
K(Qr) = Q K(r) Q^T, and positive definiteness of the mobility matrix.  The
vectorised dof-level rpy_matrix is pinned to the per-pair tensors; the dof tree
to the point tree; the H2 / SPD-HSS / PCG oracle on RPY by the same invariants
as the scalar kernels (H2 error against the dense matrix, SPD, solve residual).
"""
import numpy as np
import pytest

import oracle
import synth
from oracle.kernels import RPY, dof_points, rpy_matrix, rpy_tensor
from oracle.tree import build_tree, expand_dofs


def test_rpy_hand_values():
    # far branch, a = 0.5, r = (2, 0, 0): 3/8 (I + e1 e1^T) + 3/64 (I/3 - e1 e1^T)
    K = rpy_tensor(0.5, np.array([2.0, 0.0, 0.0]))
    np.testing.assert_allclose(K, np.diag([0.71875, 0.390625, 0.390625]), rtol=0, atol=1e-15)
    # near branch, a = 0.5, r = (0.5, 0, 0), |r|/a = 1: 2 [(23/32) I + (3/32) e1 e1^T]
    K = rpy_tensor(0.5, np.array([0.5, 0.0, 0.0]))
    np.testing.assert_allclose(K, np.diag([1.625, 1.4375, 1.4375]), rtol=0, atol=1e-15)
    # off-diagonal: r along (1, 1, 0)/sqrt2 at |r| = 3, a = 1: rr^T entry 1/2 times
    # (3/(4*3) - 3/(2*27)) = 1/4 - 1/18
    r = 3.0 * np.array([1.0, 1.0, 0.0]) / np.sqrt(2.0)
    K = rpy_tensor(1.0, r)
    assert abs(K[0, 1] - 0.5 * (0.25 - 1.0 / 18.0)) < 1e-15
    assert K[0, 2] == 0.0 and K[1, 2] == 0.0


@pytest.mark.parametrize("a", [0.29, 0.42, 1.0, 2.5])
def test_rpy_zero_continuity_and_far_limit(a):
    np.testing.assert_array_equal(rpy_tensor(a, np.zeros(3)), np.eye(3) / a)
    rng = np.random.default_rng(7)
    u = rng.standard_normal(3)
    u /= np.linalg.norm(u)
    eps = 1e-9
    Kin = rpy_tensor(a, 2 * a * (1 - eps) * u)
    Kout = rpy_tensor(a, 2 * a * (1 + eps) * u)
    assert np.abs(Kin - Kout).max() <= 10 * eps / a          # continuous at |r| = 2a (R28)
    # near r -> 0: K -> I/a continuously
    assert np.abs(rpy_tensor(a, 1e-9 * a * u) - np.eye(3) / a).max() <= 1e-8 / a
    # Oseen limit: |K - 3/(4r)(I + uu^T)| = O(a^2 / r^3)
    R = 1e3 * a
    oseen = 3.0 / (4.0 * R) * (np.eye(3) + np.outer(u, u))
    assert np.abs(rpy_tensor(a, R * u) - oseen).max() <= 2.0 * a * a / R ** 3


def test_rpy_rotation_equivariance_and_symmetry():
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    for rad in (0.1, 0.5, 0.9, 3.0):
        r = rad * rng.standard_normal(3)
        K = rpy_tensor(0.42, r)
        np.testing.assert_allclose(rpy_tensor(0.42, Q @ r), Q @ K @ Q.T, atol=1e-14)
        np.testing.assert_allclose(K, K.T, atol=0)
        np.testing.assert_allclose(rpy_tensor(0.42, -r), K, atol=0)       # even in r


def test_rpy_matrix_is_assembled_tensors_and_spd():
    cfg = synth.R2.scaled(200)
    P = synth.points(cfg)
    D = dof_points(P)
    K = rpy_matrix(cfg.ell, D, D)
    B = np.zeros_like(K)
    for p in range(len(P)):
        for q in range(len(P)):
            B[3 * p:3 * p + 3, 3 * q:3 * q + 3] = rpy_tensor(cfg.ell, P[p] - P[q])
    np.testing.assert_allclose(K, B, rtol=0, atol=1e-15)
    # the RPY mobility matrix is symmetric positive definite for any configuration
    np.testing.assert_array_equal(K, K.T)
    assert np.linalg.eigvalsh(K).min() > 0.0
    # and the kernel_matrix entry point routes kid 4 to it
    np.testing.assert_array_equal(oracle.kernel_matrix(RPY, cfg.ell, D[:30], D[:45]), K[:30, :45])


def test_dof_tree_expands_point_tree():
    cfg = synth.R1.scaled(500, leaf=32)
    P = synth.points(cfg)
    t = build_tree(P, cfg.leaf)
    td = expand_dofs(t, 3)
    assert td.N == 3 * t.N and td.L == t.L
    np.testing.assert_array_equal(td.begin, 3 * t.begin)
    Xt = dof_points(P)[td.perm]
    for pos in (0, 1, 2, 100, 3 * t.N - 1):
        p, c = divmod(pos, 3)
        np.testing.assert_array_equal(Xt[pos, :3], P[t.perm[p]])
        assert Xt[pos, 3] == c


def test_ball_points_density():
    cfg = synth.R1.scaled(20000)
    P = synth.points(cfg)
    rad = (3 * cfg.n / (4 * np.pi)) ** (1 / 3)
    rn = np.linalg.norm(P, axis=1)
    assert rn.max() <= rad
    # uniform in the ball: P(|x| <= rad/2) = 1/8
    assert abs(np.mean(rn <= rad / 2) - 0.125) < 0.01


@pytest.fixture(scope="module")
def rpy_small():
    # 16 leaves of 50 points (150 dofs); tol 1e-4 so the IDs really truncate
    cfg = synth.R1.scaled(800, leaf=64, rank_cap=30, h2_tol=1e-4)
    X = synth.points(cfg)
    h = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol, n_proxy=512)
    return cfg, X, h


def test_rpy_h2_accuracy(rpy_small):
    cfg, X, h = rpy_small
    assert h.tree.N == 3 * cfg.n and h.tree.L >= 4
    D = dof_points(X)
    A = rpy_matrix(cfg.ell, D, D)[np.ix_(h.tree.perm, h.tree.perm)]
    Ah = oracle.h2_densify(h)
    err = np.linalg.norm(Ah - A) / np.linalg.norm(A)
    assert 0.0 < err <= 10 * cfg.h2_tol                   # SPEC S:259 bound, and compression happened
    t = h.tree
    assert any(h.rank[i] < t.size(i) for i in t.nodes_at(1) if h.active[i])


def test_rpy_spdhss_spd_and_preconditions(rpy_small):
    cfg, X, h = rpy_small
    om = synth.omega(cfg, w=cfg.w)
    H = oracle.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, om, form="chol")
    M = oracle.hss_densify(H)
    np.testing.assert_allclose(M, M.T, atol=1e-12 * np.abs(M).max())
    assert np.linalg.eigvalsh(0.5 * (M + M.T)).min() > 0.0
    b = synth.rhs(cfg)[h.tree.perm]
    x = oracle.hss_solve(H, b)
    assert np.linalg.norm(M @ x - b) <= 1e-10 * np.linalg.norm(b)
    A = lambda v: oracle.h2_matvec(h, v)
    _, it_p, conv_p, _ = oracle.pcg(A, lambda v: oracle.hss_solve(H, v), b, cfg.pcg_tol, 500)
    _, it_n, conv_n, _ = oracle.pcg(A, lambda v: v, b, cfg.pcg_tol, 500)
    assert conv_p and conv_n and it_p < it_n
