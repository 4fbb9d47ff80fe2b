"""Full-size BASELINE.json configs C3, C4, C5 on the GPU (parity at the sizes the
bench's configs name, in the library's production launch configuration).

The oracle cannot build H2/HSS at N = 2.6e5 / 1.05e6 in seconds, so these check
what holds at any size against the oracle's plain kernel definition
(oracle.kernels, PAPER.md P:1073-1077 with BASELINE's formulas, reading R13):
  * H2 matvec: sampled rows of K x by direct O(N) sums, rel. error <= 10 tol
    (S:259 bound; SURVEY §8(c) pins), for every C5 width k in {1, 16, 64, 256};
  * SPD-HSS: the build succeeds (every I + B_ii Cholesky succeeds: SPD by
    construction), the solve is symmetric positive on probes, and
    PCG with the H2 operator reaches 1e-8 (R15); its recursively updated
    residual agrees with the true residual b - A x of the H2 operator.
"""
import numpy as np
import pytest

import synth
from oracle.kernels import kernel_matrix
from gpu_util import cuda, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spd():
    import paper_2011_07632_b200 as spd
    spd.lib()
    return spd


def sampled_rows(cfg, X, x, rows):
    """(K + sigma I)[rows, :] @ x by direct sums (oracle kernel definition)."""
    out = np.zeros((len(rows),) + x.shape[1:])
    for c0 in range(0, cfg.n, 1 << 17):
        cols = np.arange(c0, min(cfg.n, c0 + (1 << 17)))
        K = kernel_matrix(cfg.kernel, cfg.ell, X[rows], X[cols], cfg.shift, rows, cols)
        out += K @ x[cols]
    return out


def build(spd, cfg):
    import torch
    X = synth.points(cfg)
    h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    return X, h


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_config_build_and_pcg(spd, name):
    cfg = synth.CONFIGS[name]
    X, h = build(spd, cfg)
    rng = np.random.default_rng(7)
    rows = rng.choice(cfg.n, 24, replace=False)
    x = synth.multivec(cfg.n, 2)
    y = host(spd.h2_matvec(h, cuda(x)))
    ref = sampled_rows(cfg, X, x, rows)
    err = np.linalg.norm(y[rows] - ref) / np.linalg.norm(ref)
    print(f"{name}: H2 sampled-row error {err:.2e}; ranks max {h.ranks().max()}; h2 t {h.timings()[:2]}")
    assert err <= 10 * cfg.h2_tol
    H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=11)
    assert H.ranks().max() <= cfg.rank_cap
    v = synth.multivec(cfg.n, 3, seed=9)
    sv = host(spd.hss_solve(H, cuda(v)))
    G = v.T @ sv
    assert np.all(np.diag(G) > 0)
    assert np.abs(G - G.T).max() <= 1e-9 * np.abs(G).max()
    b = synth.rhs(cfg)
    # C4 (IMQ, sigma/K(0) = 1e-3, cap 150) needs ~4e3 iterations at N = 2^20 (the count
    # grows with N at fixed rank; probe: 509 / 1266 / 1835 at N = 2^15 / 2^17 / 2^18):
    # beyond the paper's 3000-iteration reporting cap, so the solver cap is raised (R25)
    maxit = 10000 if name == "C4" else cfg.maxit
    xs, rep = spd.pcg_solve(h, H, cuda(b), tol=cfg.pcg_tol, maxit=maxit)
    print(f"{name}: PCG iters {rep.iters} relres {rep.relres:.2e}; hss t {H.timings()[:4]}")
    assert rep.converged and rep.relres <= cfg.pcg_tol
    r_true = b - host(spd.h2_matvec(h, xs))
    assert np.linalg.norm(r_true) <= 1e-7 * np.linalg.norm(b)


@pytest.fixture(scope="module")
def c5(spd):
    return build(spd, synth.C5)


@pytest.mark.parametrize("k", [1, 16, 64, 256])
def test_full_c5_matvec_sweep(spd, c5, k):
    cfg = synth.C5
    X, h = c5
    x = synth.multivec(cfg.n, k)
    y = host(spd.h2_matvec(h, cuda(x)))
    rows = np.random.default_rng(k).choice(cfg.n, 12, replace=False)
    ref = sampled_rows(cfg, X, x, rows)
    err = np.linalg.norm(y[rows] - ref) / np.linalg.norm(ref)
    print(f"C5 k={k}: sampled-row error {err:.2e}; ranks max {h.ranks().max()}")
    assert err <= 10 * cfg.h2_tol
