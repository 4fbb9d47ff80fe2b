"""GPU unit parity of the batched dense kernels (DMMA GEMM, potrf, trsm, QRCP)
against numpy / the oracle's QRCP."""
import numpy as np
import pytest

from gpu_util import cuda, host, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spd():
    import paper_2011_07632_b200 as spd
    spd.lib()
    return spd


@pytest.mark.parametrize("ta,tb,m,n,k", [(0, 0, 64, 64, 16), (0, 0, 130, 77, 45), (1, 0, 50, 200, 300),
                                         (0, 1, 7, 9, 3), (1, 1, 129, 65, 257), (0, 0, 1, 1, 1),
                                         # few output tiles, long K: split-K path (ragged last slice)
                                         (1, 0, 32, 96, 6144), (0, 0, 70, 40, 5000), (1, 0, 32, 1, 4100)])
def test_gemm(spd, ta, tb, m, n, k):
    import ctypes
    rng = np.random.default_rng(m * n + k)
    A = rng.standard_normal((k, m) if ta else (m, k))
    B = rng.standard_normal((n, k) if tb else (k, n))
    C = rng.standard_normal((m, n))
    dA, dB, dC = cuda(A), cuda(B), cuda(C)
    st = spd.lib().spd_test_gemm(ta, tb, m, n, k, 0.7, ctypes.c_void_p(dA.data_ptr()), A.shape[0],
                                 ctypes.c_void_p(dB.data_ptr()), B.shape[0], -0.3,
                                 ctypes.c_void_p(dC.data_ptr()), m, spd._stream())
    assert st == 0
    want = 0.7 * (A.T if ta else A) @ (B.T if tb else B) - 0.3 * C
    assert rel(host(dC), want) < 1e-14


@pytest.mark.parametrize("n", [1, 5, 64, 100, 256, 300])
def test_potrf_trsm(spd, n):
    import ctypes
    rng = np.random.default_rng(n)
    G = rng.standard_normal((n, n))
    A = G @ G.T + n * np.eye(n)
    dA = cuda(A)
    info = ctypes.c_int(-1)
    assert spd.lib().spd_test_potrf(ctypes.c_void_p(dA.data_ptr()), n, n, ctypes.byref(info), spd._stream()) == 0
    assert info.value == 0
    Lg = host(dA)
    Lw = np.linalg.cholesky(A)
    assert rel(Lg, Lw) < 1e-13
    X = rng.standard_normal((n, 37))
    for uplo, trans in [("L", 0), ("L", 1), ("U", 0), ("U", 1)]:
        T = Lw if uplo == "L" else Lw.T.copy()
        dT, dX = cuda(T), cuda(X)
        assert spd.lib().spd_test_trsm(uplo.encode(), trans, ctypes.c_void_p(dT.data_ptr()), n, n,
                                       ctypes.c_void_p(dX.data_ptr()), 37, n, spd._stream()) == 0
        want = np.linalg.solve(T.T if trans else T, X)
        assert rel(host(dX), want) < 1e-12, (uplo, trans)


@pytest.mark.parametrize("n,lda", [(1, 1), (31, 40), (32, 32), (33, 33), (100, 128), (129, 129), (256, 256),
                                   (300, 301), (600, 600)])
def test_potrf_panel_kernel_bitwise_equals_unblocked(spd, monkeypatch, n, lda):
    """The shared-memory panel Cholesky (32-column panels, left-looking register tiles) applies
    the same fused multiply-adds in the same order as the column-by-column kernel
    (the default; the panel kernel is SPD_POTRF_PANEL=1): L is bitwise equal, and so are the first failing pivot and its
    reported column when the matrix is not positive definite."""
    import ctypes
    rng = np.random.default_rng(7 * n + lda)
    G = rng.standard_normal((n, n))
    A = G @ G.T + 0.5 * n * np.eye(n)
    out = {}
    for case in ("pd", "notpd"):
        M = A.copy()
        if case == "notpd":
            j = (2 * n) // 3                          # first negative pivot exactly at column j
            M[j, j] = (M[j, :j] @ np.linalg.solve(M[:j, :j], M[:j, j]) if j else 0.0) - 1e-3
        buf = np.zeros((lda, n))                      # column-major, leading dimension lda
        buf[:n, :] = M
        for mode in ("panel", "global"):
            if mode == "global":
                monkeypatch.delenv("SPD_POTRF_PANEL", raising=False)
            else:
                monkeypatch.setenv("SPD_POTRF_PANEL", "1")
            dA = cuda(buf)
            info = ctypes.c_int(-1)
            spd.lib().spd_test_potrf(ctypes.c_void_p(dA.data_ptr()), n, lda, ctypes.byref(info), spd._stream())
            out[case, mode] = (info.value, host(dA))
    assert out["pd", "panel"][0] == 0 and out["pd", "global"][0] == 0
    assert np.array_equal(out["pd", "panel"][1], out["pd", "global"][1])
    L = out["pd", "panel"][1][:n, :]
    assert rel(L, np.linalg.cholesky(A)) < 1e-13
    assert out["notpd", "panel"][0] == out["notpd", "global"][0] == (2 * n) // 3 + 1


def test_potrf_reports_not_pd(spd):
    import ctypes
    A = np.array([[1.0, 2.0], [2.0, 1.0]])
    dA = cuda(A)
    info = ctypes.c_int(0)
    spd.lib().spd_test_potrf(ctypes.c_void_p(dA.data_ptr()), 2, 2, ctypes.byref(info), spd._stream())
    assert info.value == 2


@pytest.mark.parametrize("batch,m,n,cap,tol", [(3, 40, 25, 25, 0.0), (2, 300, 160, 150, 1e-3),
                                               (5, 128, 110, 100, 1e-3), (1, 6144, 300, 300, 1e-10),
                                               (4, 20, 60, 20, 0.0), (1, 2000, 900, 900, 1e-10)])
def test_qrcp_matches_oracle(spd, batch, m, n, cap, tol):
    import ctypes
    import torch
    import oracle
    rng = np.random.default_rng(m + n)
    mats = []
    for b in range(batch):
        # decaying spectrum so the rank rule is exercised
        U, _ = np.linalg.qr(rng.standard_normal((m, min(m, n))))
        V, _ = np.linalg.qr(rng.standard_normal((n, min(m, n))))
        s = np.logspace(0, -14, min(m, n))
        mats.append((U * s) @ V.T)
    A = np.stack(mats)                                   # batch x m x n
    dA = torch.tensor(np.ascontiguousarray(A.transpose(0, 2, 1)), device="cuda")  # col-major each
    piv = torch.zeros(batch * n, dtype=torch.int32, device="cuda")
    rank = torch.zeros(batch, dtype=torch.int32, device="cuda")
    Q = torch.zeros(batch * m * min(m, n, cap), dtype=torch.float64, device="cuda")
    st = spd.lib().spd_test_qrcp(batch, ctypes.c_void_p(dA.data_ptr()), m, n, m, m * n, cap, tol,
                                 ctypes.c_void_p(piv.data_ptr()), ctypes.c_void_p(rank.data_ptr()),
                                 ctypes.c_void_p(Q.data_ptr()), m * min(m, n, cap), spd._stream())
    assert st == 0, spd.lib().spd_last_error()
    Rg = host(dA).reshape(batch, n, m).transpose(0, 2, 1)
    pg = host(piv).reshape(batch, n)
    rg = host(rank)
    Qg = host(Q).reshape(batch, min(m, n, cap), m).transpose(0, 2, 1)
    from oracle.certify import certify_pivots
    for b in range(batch):
        Qo, Ro, po, ro = oracle.qrcp(A[b], cap, tol)
        # the whole pivot sequence and the rank: the oracle's, or certified ties (R19)
        cert = certify_pivots(A[b], pg[b], rg[b], tol, cap)
        assert cert["ok"], (b, cert["ties"][:5], cert["worst"], cert["rank_ok"], rg[b], ro)
        r = min(int(rg[b]), ro)
        # values: compare up to the first deviation (after a tie the factors differ)
        same = int(np.argmax(pg[b][:r] != po[:r])) if (pg[b][:r] != po[:r]).any() else r
        Rb = np.triu(Rg[b][:r])
        np.testing.assert_allclose(Rb[:, :same], Ro[:, :same], atol=1e-12 * abs(Ro[0, 0]))
        # Q columns are determined to ~eps/(R_tt/R_00): compare the well-conditioned ones
        good = min(same, int((np.abs(np.diag(Ro[:, :r])) > 1e-6 * abs(Ro[0, 0])).sum()))
        assert rel(Qg[b][:, :good], Qo[:, :good]) < 1e-9


@pytest.mark.parametrize("batch,m,n", [(3, 6144, 300), (2, 4096, 130), (4, 700, 64), (1, 6144, 1480), (5, 100, 33)])
def test_blocked_qr_r_factor(spd, batch, m, n):
    """Cluster-panel blocked Householder QR: R^T R = A^T A and R matches numpy's R
    up to row signs (diag(R) >= 0 here), including rank-deficient tails."""
    import ctypes
    import torch
    rng = np.random.default_rng(m + n)
    mats = []
    for b in range(batch):
        U, _ = np.linalg.qr(rng.standard_normal((m, n)))
        V, _ = np.linalg.qr(rng.standard_normal((n, n)))
        mats.append((U * np.logspace(0, -15, n)) @ V.T)
    A = np.stack(mats)
    dA = torch.tensor(np.ascontiguousarray(A.transpose(0, 2, 1)), device="cuda")
    st = spd.lib().spd_test_qr_unpivoted(batch, ctypes.c_void_p(dA.data_ptr()), m, n, m, m * n, spd._stream())
    assert st == 0, spd.lib().spd_last_error()
    torch.cuda.synchronize()
    Rg = host(dA).reshape(batch, n, m).transpose(0, 2, 1)
    for b in range(batch):
        R = np.triu(Rg[b][:n, :n])
        assert np.all(np.diag(R) >= 0)
        Rn = np.linalg.qr(A[b], mode="r")
        Rn = Rn * np.sign(np.diag(Rn))[:, None]
        np.testing.assert_allclose(R, Rn, atol=1e-13 * abs(Rn[0, 0]))
