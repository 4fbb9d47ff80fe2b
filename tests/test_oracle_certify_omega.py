"""Pins of the round-2 oracle pieces (CPU only):

* oracle/omega.py -- the counter-based Gaussian sketch (Alg. 2 step 1, R8,
  reading R29): Random123 known-answer vectors of Philox4x32-10, N(0,1) moments and
  Kolmogorov-Smirnov distance, column independence, counter = column-major index.
* oracle/linalg.qrcp_trace + oracle/certify.py -- the certified-tie rule (reading
  R19): the trace reproduces the plain QRCP, numax(t) = R_tt, exact ties certify,
  non-ties and off-threshold ranks do not, near-threshold ranks do.
* oracle.hss_error (Fig. 5 metric) against an independent dense route.
* kernel_matrix's pairwise distances against exact integer geometry and
  scipy.spatial.distance.cdist.
"""
import numpy as np
import pytest
from scipy import stats
from scipy.spatial.distance import cdist

import oracle
import synth
from oracle.certify import certify_pivots
from oracle.kernels import kernel_matrix, sqdist
from oracle.linalg import qrcp, qrcp_trace
from oracle.omega import philox4x32_10, philox_normal


# ---------------------------------------------------------------- Philox Omega
@pytest.mark.parametrize("ctr,key,want", [
    # Random123 kat_vectors, philox4x32 with 10 rounds
    ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
])
def test_philox_known_answers(ctr, key, want):
    out = philox4x32_10([np.array([c], dtype=np.uint64) for c in ctr], key)
    assert tuple(int(o[0]) for o in out) == want


def test_philox_normal_distribution():
    z = philox_normal(1 << 17, 10, seed=1234)          # 1.3e6 samples
    x = z.ravel()
    n = x.size
    assert abs(x.mean()) < 5 / np.sqrt(n)
    assert abs(x.var() - 1.0) < 5 * np.sqrt(2.0 / n)
    assert abs(stats.skew(x)) < 5 * np.sqrt(6.0 / n)
    assert abs(stats.kurtosis(x)) < 5 * np.sqrt(24.0 / n)
    ks = stats.kstest(x, "norm")
    assert ks.statistic < 1.63 / np.sqrt(n)             # 1 % critical value
    C = np.corrcoef(z.T)
    off = C[~np.eye(10, dtype=bool)]
    assert np.abs(off).max() < 5 / np.sqrt(z.shape[0])  # columns uncorrelated
    # lag-1 correlation along a column (consecutive counters)
    assert abs(np.corrcoef(z[:-1, 0], z[1:, 0])[0, 1]) < 5 / np.sqrt(z.shape[0])


def test_philox_counter_is_column_major_element_index():
    a = philox_normal(100, 7, seed=99)
    b = philox_normal(700, 1, seed=99)[:, 0]            # same counters, one column
    np.testing.assert_array_equal(a.ravel(order="F"), b)
    assert not np.array_equal(philox_normal(10, 2, seed=1), philox_normal(10, 2, seed=2))
    # the adaptive build's prefix property (R27): leading columns coincide
    np.testing.assert_array_equal(philox_normal(50, 8, 5)[:, :3], philox_normal(50, 3, 5))


# ---------------------------------------------------------------- certified ties
def test_qrcp_trace_reproduces_qrcp():
    A = np.random.default_rng(0).standard_normal((60, 35))
    _, R, piv, r = qrcp(A, 35, 1e-6)
    R2, piv2, r2, numax, nuf = qrcp_trace(A, 35, 1e-6)
    assert r == r2 and np.array_equal(piv, piv2) and np.array_equal(R, R2)
    np.testing.assert_allclose(numax[:r], np.diag(R)[:r], rtol=1e-12)   # |R_tt| = max norm
    np.testing.assert_array_equal(numax[:r], nuf[:r])
    # following the oracle's own pivots is the oracle's run
    R3, piv3, r3, _, _ = qrcp_trace(A, 35, 1e-6, follow=piv[:r])
    assert r3 == r and np.array_equal(piv3, piv) and np.array_equal(R3, R)


def test_certify_accepts_own_and_exact_ties_rejects_others():
    A = np.random.default_rng(1).standard_normal((50, 30))
    _, _, piv, r = qrcp(A, 30, 1e-8, want_q=False)
    assert certify_pivots(A, piv, r, 1e-8, 30)["ok"]
    B = A.copy()
    B[:, 5] = B[:, 2]                                   # exact duplicate: a true tie
    _, _, pb, rb = qrcp(B, 30, 1e-8, want_q=False)
    alt = pb.copy()
    i, j = list(alt).index(2), list(alt).index(5)
    alt[i], alt[j] = alt[j], alt[i]
    c = certify_pivots(B, alt, rb, 1e-8, 30)
    assert c["ok"] and c["rank_ok"]
    swapped = pb.copy()
    swapped[[0, 1]] = swapped[[1, 0]]                   # distinct norms: not a tie
    c = certify_pivots(B, swapped, rb, 1e-8, 30)
    assert not c["ok"] and c["ties"][0] == 0
    assert not certify_pivots(A, piv, r - 1, 1e-8, 30)["ok"]     # stopped far above tau
    assert not certify_pivots(A, np.r_[piv[:r], 0], r + 1, 1e-8, 30)["ok"] or r == 30


def test_certify_rank_band_at_the_threshold():
    # diagonal matrix: residual norms are the diagonal; |R_22| = tau (1 + 4 eps)
    tau = 1e-3
    eps = np.finfo(float).eps
    A = np.diag([1.0, 0.5, tau * (1 + 4 * eps), 1e-9])
    _, _, piv, r = qrcp(A, 4, tau, want_q=False)
    assert r == 3
    assert certify_pivots(A, piv, 2, tau, 4)["ok"]      # stopping one step early is a tie
    A2 = np.diag([1.0, 0.5, 2 * tau, 1e-9])
    assert not certify_pivots(A2, piv, 2, tau, 4)["ok"]


# ---------------------------------------------------------------- hss_error (Fig. 5)
def test_hss_error_against_dense_block_diagonal():
    """With rel_tol >= 1 every HSS rank is 0 (|R_00| <= tol |R_00|), so the SPD-HSS
    matrix is blockdiag(A_ii) exactly (Alg. 4 with empty bases) and the Fig. 5 metric is
    ||(A - blockdiag A) x|| / ||A x|| -- evaluated here on the dense H2 matrix."""
    cfg = synth.C1.scaled(256, leaf=32)
    X = synth.points(cfg)
    h = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    H = oracle.spdhss_build(h, 20, 1.0, synth.omega(cfg, w=30), form="chol")
    assert all(r == 0 for r in H.rank.values())
    A = oracle.h2_densify(h)
    D = np.zeros_like(A)
    t = h.tree
    for i in t.nodes_at(1):
        s = slice(t.begin[i], t.end[i])
        D[s, s] = A[s, s]
    P = synth.multivec(256, 7, seed=4)
    want = np.mean([np.linalg.norm((A - D) @ p) / np.linalg.norm(A @ p) for p in P.T])
    assert oracle.hss_error(H, P) == pytest.approx(want, rel=1e-10)
    assert want > 0.05                                   # the off-diagonal part is not small


# ---------------------------------------------------------------- distances (O1)
def test_sqdist_exact_integer_geometry():
    # Pythagorean quadruples: |(1,2,2)| = 3, |(2,3,6)| = 7, |(1,4,8)| = 9, |(2,6,9)| = 11
    X = np.array([[0.0, 0.0, 0.0], [1.0, 2.0, 2.0], [2.0, 3.0, 6.0]])
    Y = np.array([[1.0, 4.0, 8.0], [-2.0, -6.0, -9.0], [0.0, 0.0, 0.0]])
    want = np.array([[81.0, 121.0, 0.0], [0 + 4 + 36, 9 + 64 + 121, 9.0], [1 + 1 + 4, 16 + 81 + 225, 49.0]])
    np.testing.assert_array_equal(sqdist(X, Y), want)
    # the kernels at those distances (closed forms), shift only where labels coincide
    K = kernel_matrix(3, 0.1, X, Y, 0.25, np.array([0, 1, 2]), np.array([5, 6, 0]))
    np.testing.assert_allclose(K[0, 0], 1.0 / np.sqrt(81.0 + 0.01), rtol=1e-15)
    np.testing.assert_allclose(K[1, 2], 1.0 / np.sqrt(9.0 + 0.01), rtol=1e-15)
    np.testing.assert_allclose(K[0, 2], 1.0 / 0.1 + 0.25, rtol=1e-15)
    np.testing.assert_allclose(kernel_matrix(2, 0.5, X[1:2], Y[2:3]), [[np.exp(-3.0 / 0.5)]], rtol=1e-15)


def test_sqdist_matches_cdist():
    rng = np.random.default_rng(7)
    for d in (2, 3):
        X, Y = rng.random((40, d)), rng.random((33, d))
        np.testing.assert_allclose(sqdist(X, Y), cdist(X, Y, "sqeuclidean"), rtol=1e-13, atol=1e-16)
        K = kernel_matrix(1, 0.2, X, Y)
        r = cdist(X, Y)
        np.testing.assert_allclose(K, (1 + np.sqrt(3) * r / 0.2) * np.exp(-np.sqrt(3) * r / 0.2), rtol=1e-13)
