"""Pins of the oracle's primitives against closed forms, textbook special
cases and brute force (DESIGN.md §Oracle pins).  CPU only."""
import math
import os

import numpy as np
import pytest
from scipy.special import gamma, kv

import oracle
from oracle.kernels import kernel_matrix, kernel_value
from oracle.linalg import NotPD, cholesky, house, qrcp, sym_sqrt_pair

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].strip()
        if line:
            yield line


# ---------------------------------------------------------------- kernels (O1)
def test_kernel_special_values_golden():
    n = 0
    for line in _golden_rows("kernel_special_values.txt"):
        kid, ell, r, want = line.split()
        got = float(kernel_value(int(kid), float(ell), float(r) ** 2))
        assert got == pytest.approx(float(want), rel=2e-15, abs=0), line
        n += 1
    assert n >= 10


def test_matern32_is_bessel_matern_nu_1p5():
    # general Matern: 2^{1-nu}/Gamma(nu) (sqrt(2nu) r/l)^nu K_nu(sqrt(2nu) r/l), nu = 3/2
    nu, ell = 1.5, 0.2
    for r in [0.01, 0.1, 0.37, 1.3]:
        z = math.sqrt(2 * nu) * r / ell
        want = 2 ** (1 - nu) / gamma(nu) * z ** nu * kv(nu, z)
        assert float(kernel_value(1, ell, r * r)) == pytest.approx(want, rel=1e-12)


def test_kernel_matrix_symmetry_and_shift_only_on_diagonal():
    rng = np.random.default_rng(0)
    X = rng.random((30, 3))
    idx = np.arange(30)
    for kid in range(4):
        K = kernel_matrix(kid, 0.3, X, X, 0.5, idx, idx)
        K0 = kernel_matrix(kid, 0.3, X, X)
        assert np.array_equal(K, K.T)
        D = K - K0
        assert np.array_equal(D, 0.5 * np.eye(30))
        # off-diagonal blocks between distinct index sets get no shift
        Kb = kernel_matrix(kid, 0.3, X[:10], X[10:], 0.5, idx[:10], idx[10:])
        assert np.array_equal(Kb, K0[:10, 10:])


# ---------------------------------------------------------------- linalg
def test_spec_linalg_examples_golden():
    rows = list(_golden_rows("spec_linalg_examples.txt"))
    a = [float(v) for v in rows[0].split("->")[0].split()[1:]]
    want = [float(v) for v in rows[0].split("->")[1].split()]
    np.testing.assert_allclose(cholesky(np.array(a).reshape(2, 2)), np.array(want).reshape(2, 2), rtol=1e-15)
    with pytest.raises(NotPD):
        cholesky(np.array([float(v) for v in rows[1].split()[1:]]).reshape(2, 2))
    B = np.array([float(v) for v in rows[2].split("->")[0].split()[1:]]).reshape(2, 2)
    P, M = sym_sqrt_pair(B)
    wp, wm = rows[2].split("->")[1].split("|")
    np.testing.assert_allclose(P, np.array([float(v) for v in wp.split()]).reshape(2, 2), atol=1e-15)
    np.testing.assert_allclose(M, np.array([float(v) for v in wm.split()]).reshape(2, 2), atol=1e-15)


def test_sym_sqrt_pair_random():
    rng = np.random.default_rng(1)
    Q, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    B = (Q * rng.uniform(-0.5, 0.5, 12)) @ Q.T
    P, M = sym_sqrt_pair(B)
    np.testing.assert_allclose(P @ P, np.eye(12) + B, atol=1e-13)
    np.testing.assert_allclose(P @ M, np.eye(12), atol=1e-13)
    np.testing.assert_allclose(M @ (np.eye(12) + B) @ M, np.eye(12), atol=1e-13)
    with pytest.raises(NotPD):
        sym_sqrt_pair(np.diag([-2.0, 0.0]))


def test_house_maps_to_positive_multiple_of_e1():
    rng = np.random.default_rng(2)
    for x in [rng.standard_normal(7), -np.abs(rng.standard_normal(7)), np.array([-3.0, 0, 0]),
              np.array([2.0, 0.0]), np.array([1e-300, 1.0])]:
        v, beta = house(x)
        y = x - beta * v * (v @ x)
        np.testing.assert_allclose(y[0], np.linalg.norm(x), rtol=1e-14)
        assert np.abs(y[1:]).max() <= 1e-14 * np.linalg.norm(x)


def _greedy_pivots(A, r):
    """Brute force: at each step pick the column farthest from the span of the
    columns already chosen (least-squares residual), lowest index on ties."""
    chosen = []
    for _ in range(r):
        best, bestd = None, -1.0
        for j in range(A.shape[1]):
            if j in chosen:
                continue
            if chosen:
                C = A[:, chosen]
                coef = np.linalg.lstsq(C, A[:, j], rcond=None)[0]
                d = np.linalg.norm(A[:, j] - C @ coef)
            else:
                d = np.linalg.norm(A[:, j])
            if d > bestd * (1 + 1e-12):
                best, bestd = j, d
        chosen.append(best)
    return chosen


@pytest.mark.parametrize("m,n,seed", [(9, 6, 0), (6, 9, 1), (20, 20, 2), (40, 12, 3)])
def test_qrcp_factorization_and_greedy_pivots(m, n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) * rng.uniform(0.1, 3.0, n)
    Q, R, piv, r = qrcp(A, min(m, n), 0.0)
    assert r == min(m, n)
    np.testing.assert_allclose(Q.T @ Q, np.eye(r), atol=1e-13)
    np.testing.assert_allclose(Q @ R, A[:, piv], atol=1e-12 * np.abs(A).max())
    d = np.diag(R)
    assert np.all(d >= 0) and np.all(np.diff(d) <= 1e-12 * d[0])
    assert list(piv[:r]) == _greedy_pivots(A, r)


def test_qrcp_ties_lowest_index_and_rank_rules():
    v = np.array([1.0, 2.0, 2.0])
    A = np.stack([v, 2 * v, 2 * v, v], axis=1)      # rank 1, duplicated max column
    Q, R, piv, r = qrcp(A, 4, 1e-10)
    assert r == 1 and piv[0] == 1                   # columns 1 and 2 tie: lowest index
    np.testing.assert_allclose(np.abs(Q[:, 0]), v / np.linalg.norm(v), rtol=1e-14)
    Z = np.zeros((5, 3))
    assert qrcp(Z, 3, 1e-3)[3] == 0                 # zero sketch -> rank 0 (R4)
    rng = np.random.default_rng(4)
    H = rng.standard_normal((30, 5)) @ rng.standard_normal((5, 15))
    Q, R, piv, r = qrcp(H, 15, 1e-10)
    assert r == 5
    assert np.linalg.norm(H - Q @ (Q.T @ H)) <= 1e-12 * np.linalg.norm(H)
    assert qrcp(H, 3, 1e-10)[3] == 3                # cap binds first


def test_qrcp_column_shuffle_keeps_column_space():
    rng = np.random.default_rng(5)
    H = rng.standard_normal((25, 6)) @ rng.standard_normal((6, 12))
    Q1 = qrcp(H, 12, 1e-10)[0]
    Q2 = qrcp(H[:, rng.permutation(12)], 12, 1e-10)[0]
    np.testing.assert_allclose(Q1 @ Q1.T, Q2 @ Q2.T, atol=1e-12)


# ---------------------------------------------------------------- Halton (R3)
def test_halton_known_values():
    assert [oracle.halton(k, 2) for k in range(1, 6)] == [0.5, 0.25, 0.75, 0.125, 0.625]
    assert [oracle.halton(k, 3) for k in range(1, 5)] == [1 / 3, 2 / 3, 1 / 9, 4 / 9]
    assert oracle.halton(1, 5) == 0.2
