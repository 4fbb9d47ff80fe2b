"""Dense primitives of the construction -- TEST INFRASTRUCTURE ONLY.

cholesky      A_ii = S_i S_i^T (Alg. 1, Alg. 4)
sym_sqrt_pair (I + B)^{+-1/2} by eigendecomposition (eqn:Si0)
qrcp          pivoted QR of Alg. 2 step 3, reading R4:
              Businger-Golub column pivoting, residual column norms
              recomputed at every step (no downdating), ties -> lowest column
              index, rank = min(cap, first t with |R_tt| <= tol |R_00|),
              Householder vectors chosen so that diag(R) >= 0 (hence Q is
              unique given the pivots).
"""
import numpy as np


class NotPD(ArithmeticError):
    """Not positive definite (reading R18)."""

    def __init__(self, msg, where=None, value=None):
        super().__init__(msg)
        self.where = where
        self.value = value


def cholesky(A, where=None):
    A = np.asarray(A, dtype=np.float64)
    if A.shape[0] == 0:
        return A.copy()
    try:
        return np.linalg.cholesky(A)
    except np.linalg.LinAlgError:
        lam = np.linalg.eigvalsh(0.5 * (A + A.T)).min()
        raise NotPD(f"matrix not positive definite at {where}: lambda_min={lam:.3e}",
                    where, lam)


def sym_sqrt_pair(B, where=None):
    """Return ((I+B)^{1/2}, (I+B)^{-1/2}) via eigh."""
    m = B.shape[0]
    if m == 0:
        return np.zeros((0, 0)), np.zeros((0, 0))
    lam, Q = np.linalg.eigh(np.eye(m) + 0.5 * (B + B.T))
    if lam.min() <= 0.0:
        raise NotPD(f"I+B indefinite at {where}: lambda_min={lam.min():.3e}",
                    where, lam.min())
    sq = np.sqrt(lam)
    return (Q * sq) @ Q.T, (Q / sq) @ Q.T


def house(x):
    """Householder vector v (v[0]=1) and beta with (I - beta v v^T) x = ||x|| e1.

    Golub & Van Loan, Matrix Computations, Alg. 5.1.1 (the sign choice that
    keeps the image positive, computed without cancellation).
    """
    x = np.asarray(x, dtype=np.float64)
    sigma = float(x[1:] @ x[1:])
    v = x.copy()
    v[0] = 1.0
    x0 = float(x[0])
    if sigma == 0.0:
        beta = 0.0 if x0 >= 0.0 else 2.0
        v[1:] = 0.0
        return v, beta
    mu = np.sqrt(x0 * x0 + sigma)
    v0 = x0 - mu if x0 <= 0.0 else -sigma / (x0 + mu)
    beta = 2.0 * v0 * v0 / (sigma + v0 * v0)
    v[1:] = x[1:] / v0
    return v, beta


_LIB = None


def _lib():
    """Load oracle/qrcp.c (plain C + OpenMP), compiling it on first use."""
    global _LIB
    if _LIB is None:
        import ctypes, os, subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        so = os.path.join(here, "_build", "liboracle_qrcp.so")
        src = os.path.join(here, "qrcp.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            os.makedirs(os.path.dirname(so), exist_ok=True)
            tmp = so + f".{os.getpid()}.tmp"
            subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off",
                                   "-shared", "-fPIC", src, "-o", tmp, "-lm"])
            os.replace(tmp, so)
        lib = ctypes.CDLL(so)
        P = ctypes.POINTER
        lib.oracle_qrcp.argtypes = [ctypes.c_int, ctypes.c_int, P(ctypes.c_double),
                                    ctypes.c_int, ctypes.c_double, P(ctypes.c_int),
                                    P(ctypes.c_double)]
        lib.oracle_qrcp.restype = ctypes.c_int
        lib.oracle_qrcp_follow.argtypes = [ctypes.c_int, ctypes.c_int, P(ctypes.c_double),
                                           ctypes.c_int, ctypes.c_double, P(ctypes.c_int),
                                           P(ctypes.c_double), P(ctypes.c_int), ctypes.c_int,
                                           P(ctypes.c_double), P(ctypes.c_double),
                                           P(ctypes.c_double), P(ctypes.c_int)]
        lib.oracle_qrcp_follow.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def qrcp(A, max_rank, rel_tol, want_q=True):
    """Pivoted QR  A P = Q R  truncated at the rank rule of R4 (oracle/qrcp.c).

    Returns (Q_r, R_r, piv, r): Q_r = Q[:, :r] (m x r, orthonormal, None if
    want_q is False), R_r = R[:r, :] (r x n, upper trapezoidal, columns in
    pivoted order), piv (n,) with A[:, piv] ~= Q R, and the rank r.
    """
    import ctypes
    A = np.array(A, dtype=np.float64, order="F", copy=True)
    m, n = A.shape
    piv = np.zeros(n, dtype=np.int32)
    beta = np.zeros(max(min(m, n), 1))
    P = ctypes.POINTER
    r = _lib().oracle_qrcp(m, n, A.ctypes.data_as(P(ctypes.c_double)), int(max_rank),
                           float(rel_tol), piv.ctypes.data_as(P(ctypes.c_int)),
                           beta.ctypes.data_as(P(ctypes.c_double)))
    R = np.triu(A[:r, :])
    Q = None
    if want_q:
        Q = np.zeros((m, r))
        Q[:r, :r] = np.eye(r)
        for t in range(r - 1, -1, -1):           # Q = H_0 H_1 ... H_{r-1} [I; 0]
            v = np.concatenate([[1.0], A[t + 1:, t]])
            Q[t:, :] -= beta[t] * np.outer(v, v @ Q[t:, :])
    return Q, R, piv.astype(np.int64), r


def qrcp_trace(A, max_rank, rel_tol, follow=None, runner_up=False):
    """The QRCP of `qrcp` with its per-step norms recorded (reading R19).

    follow=None: the oracle's own Businger-Golub run.  follow = a pivot sequence of
    ORIGINAL column indices (another implementation's pivots, length s): step t takes
    column follow[t] instead of the argmax and the run stops after s steps.
    Returns (R_r, piv, r, numax, nuf): numax[t] = largest residual column norm at step t
    (t < r, plus t = r when the run stopped before min(m, n, max_rank) in own mode, or
    when s < min(m, n, max_rank) in follow mode), nuf[t] = the norm of the column taken.
    r = -1 if a followed index is not a remaining column."""
    import ctypes
    A = np.array(A, dtype=np.float64, order="F", copy=True)
    m, n = A.shape
    kmax = max(0, min(m, n, int(max_rank)))
    piv = np.zeros(n, dtype=np.int32)
    beta = np.zeros(max(min(m, n), 1))
    numax = np.full(kmax + 1, np.nan)
    nuf = np.full(kmax + 1, np.nan)
    P = ctypes.POINTER
    if follow is not None:
        fo = np.ascontiguousarray(np.asarray(follow, dtype=np.int32))
        fptr, nf = fo.ctypes.data_as(P(ctypes.c_int)), int(fo.size)
    else:
        fptr, nf = None, 0
    nu2 = np.full(kmax + 1, np.nan)
    idx2 = np.full(kmax + 1, -1, dtype=np.int32)
    r = _lib().oracle_qrcp_follow(m, n, A.ctypes.data_as(P(ctypes.c_double)), int(max_rank),
                                  float(rel_tol), piv.ctypes.data_as(P(ctypes.c_int)),
                                  beta.ctypes.data_as(P(ctypes.c_double)), fptr, nf,
                                  numax.ctypes.data_as(P(ctypes.c_double)),
                                  nuf.ctypes.data_as(P(ctypes.c_double)),
                                  nu2.ctypes.data_as(P(ctypes.c_double)) if runner_up else None,
                                  idx2.ctypes.data_as(P(ctypes.c_int)) if runner_up else None)
    R = np.triu(A[:max(r, 0), :])
    if runner_up:
        return R, piv.astype(np.int64), r, numax, nuf, nu2, idx2.astype(np.int64)
    return R, piv.astype(np.int64), r, numax, nuf
