"""Kernel functions K(x,y) (oracle step O1) -- TEST INFRASTRUCTURE ONLY.

PAPER.md §6 P:1073-1077 lists Matern-3/2, Gaussian and IMQ with l as an
inverse scale; BASELINE.json fixes explicit formulas, which win (reading R13):
  0 Gaussian     exp(-r^2 / l^2)
  1 Matern-3/2   (1 + sqrt(3) r / l) exp(-sqrt(3) r / l)
  2 Exponential  exp(-r / l)                       (BASELINE C3 only)
  3 IMQ          1 / sqrt(r^2 + l^2)
The diagonal shift sigma*I is added only on exact diagonal
entries, i.e. when the row and column index the same point.
"""
import numpy as np

SQRT3 = np.sqrt(3.0)


def kernel_value(kid: int, ell: float, r2):
    """K as a function of the squared distance r2 (array or scalar)."""
    r2 = np.asarray(r2, dtype=np.float64)
    if kid == 0:
        return np.exp(-r2 / (ell * ell))
    if kid == 1:
        t = SQRT3 * np.sqrt(r2) / ell
        return (1.0 + t) * np.exp(-t)
    if kid == 2:
        return np.exp(-np.sqrt(r2) / ell)
    if kid == 3:
        return 1.0 / np.sqrt(r2 + ell * ell)
    raise ValueError(f"unknown kernel id {kid}")


def sqdist(X, Y):
    """Pairwise squared distances, summed coordinate by coordinate."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    r2 = np.zeros((X.shape[0], Y.shape[0]))
    for d in range(X.shape[1]):
        diff = X[:, d][:, None] - Y[:, d][None, :]
        r2 += diff * diff
    return r2


def kernel_matrix(kid, ell, X, Y, shift=0.0, rows=None, cols=None):
    """K(X, Y) (+ shift on entries whose row and column index coincide).

    rows/cols: integer labels of the points (e.g. tree positions); the shift is
    added where rows[a] == cols[b] ("sigma I + K_l(X,X)").
    """
    K = kernel_value(kid, ell, sqdist(X, Y))
    if shift != 0.0 and rows is not None and cols is not None:
        rows = np.asarray(rows)
        cols = np.asarray(cols)
        K = K + shift * (rows[:, None] == cols[None, :])
    return K
