"""Kernel functions K(x,y) (oracle step O1) -- TEST INFRASTRUCTURE ONLY.

PAPER.md §6 P:1073-1077 lists Matern-3/2, Gaussian and IMQ with l as an
inverse scale; BASELINE.json fixes explicit formulas, which win (reading R13):
  0 Gaussian     exp(-r^2 / l^2)
  1 Matern-3/2   (1 + sqrt(3) r / l) exp(-sqrt(3) r / l)
  2 Exponential  exp(-r / l)                       (BASELINE C3 only)
  3 IMQ          1 / sqrt(r^2 + l^2)
  4 RPY          Rotne-Prager-Yamakawa 3x3 tensor, l = particle radius a
                 (reading R28 below)
The diagonal shift sigma*I is added only on exact diagonal
entries, i.e. when the row and column index the same point (RPY: the same
degree of freedom).

RPY, r = x - y, rhat = r/|r|, a = particle radius:
  |r| = 0    :  (1/a) I_3
  |r| >= 2a  :  3/(4|r|) (I_3 + rhat rhat^T) + 3a^2/(2|r|^3) (I_3/3 - rhat rhat^T)
  |r| <  2a  :  (1/a) [ (1 - 9|r|/(32a)) I_3 + (3|r|/(32a)) rhat rhat^T ]
Reading R28: the printed near branch closes the 1/a bracket before the rhat
rhat^T term; with that placement the tensor is discontinuous at |r| = 2a unless
a = 1.  The 1/a multiplies both terms here (continuity at 2a, and the standard
RPY mobility divided by the self-mobility times a).
The matrix is 3N x 3N over DEGREES OF FREEDOM: dof 3p + c is component c of
point p.  A dof is stored as a row (x, y, z, c) (dof_points); kernel_matrix of
kid 4 takes such rows.
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


RPY = 4
DOFS = {RPY: 3}          # degrees of freedom per point (scalar kernels: 1)


def dofs_per_point(kid):
    return DOFS.get(kid, 1)


def dof_points(P, m=3):
    """(n, 3) points -> (m n, 4) dof rows (x, y, z, c), dof m p + c."""
    P = np.asarray(P, dtype=np.float64)
    out = np.zeros((m * P.shape[0], P.shape[1] + 1))
    for c in range(m):
        out[c::m, :P.shape[1]] = P
        out[c::m, P.shape[1]] = c
    return out


def rpy_tensor(a, r):
    """The 3x3 RPY tensor of one difference vector r (R28)."""
    r = np.asarray(r, dtype=np.float64)
    nr = np.sqrt(r @ r)
    I3 = np.eye(3)
    if nr == 0.0:
        return I3 / a
    rr = np.outer(r, r) / (nr * nr)
    if nr >= 2.0 * a:
        return 3.0 / (4.0 * nr) * (I3 + rr) + 3.0 * a * a / (2.0 * nr ** 3) * (I3 / 3.0 - rr)
    return (1.0 / a) * ((1.0 - 9.0 * nr / (32.0 * a)) * I3 + 3.0 * nr / (32.0 * a) * rr)


def rpy_matrix(a, X, Y):
    """K(X, Y) over dof rows (x, y, z, c): entry = rpy_tensor(a, x - y)[c_x, c_y]."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    D = X[:, None, :3] - Y[None, :, :3]                     # r = x - y
    r2 = np.zeros(D.shape[:2])
    for dd in range(3):
        r2 += D[..., dd] * D[..., dd]
    nr = np.sqrt(r2)
    cx = X[:, 3].astype(np.int64)
    cy = Y[:, 3].astype(np.int64)
    delta = (cx[:, None] == cy[None, :]).astype(np.float64)
    ra = np.take_along_axis(D, np.broadcast_to(cx[:, None, None], D.shape[:2] + (1,)), axis=2)[..., 0]
    rb = np.take_along_axis(D, np.broadcast_to(cy[None, :, None], D.shape[:2] + (1,)), axis=2)[..., 0]
    with np.errstate(divide="ignore", invalid="ignore"):
        rr = np.where(r2 > 0.0, ra * rb / r2, 0.0)
        far_v = 3.0 / (4.0 * nr) * (delta + rr) + 3.0 * a * a / (2.0 * nr ** 3) * (delta / 3.0 - rr)
    near_v = (1.0 / a) * ((1.0 - 9.0 * nr / (32.0 * a)) * delta + 3.0 * nr / (32.0 * a) * rr)
    K = np.where(nr >= 2.0 * a, far_v, near_v)
    return np.where(r2 == 0.0, delta / a, K)


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
    K = rpy_matrix(ell, X, Y) if kid == RPY else kernel_value(kid, ell, sqdist(X, Y))
    if shift != 0.0 and rows is not None and cols is not None:
        rows = np.asarray(rows)
        cols = np.asarray(cols)
        K = K + shift * (rows[:, None] == cols[None, :])
    return K
