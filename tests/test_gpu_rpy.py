"""The RPY workload of PAPER.md Table 3 at the paper's own size on
the GPU (reading R28): N = 4e4 points uniform in the ball of
radius (3N/(4 pi))^(1/3), particle radius a = 0.29 / 0.42, no shift, H2 tolerance
1e-8, SPD-HSS r = 100, PCG to 1e-4 with b ~ U[-0.5, 0.5].

* H2 accuracy: sampled rows of the 3N x 3N product against direct sums of the
  oracle's RPY tensor (R28) -- the dense matrix is never formed.
* The paper's iteration counts for this row of Table 3 (ball, N = 4e4):
      a = 0.29: SPDHSS r=100: 40, BJ: 95, unpreconditioned: 432
      a = 0.42: SPDHSS r=100: 64, BJ: 150, unpreconditioned: 632
  Our tree (binary KD, 128-point leaves) is not the paper's octree (< 400 points
  per box) and its H2 differs, so counts are compared within 25 %
  (preconditioned) / 35 % (unpreconditioned), and the ORDER is required:
  SPDHSS < BJ < none.  Measured on B200: 39 / 105 / 487 and 67 / 146 / 503.
"""
import numpy as np
import pytest

import synth
from gpu_util import cuda, host

pytestmark = pytest.mark.gpu

PAPER = {"R1": (40, 95, 432), "R2": (64, 150, 632)}


@pytest.fixture(scope="module")
def spd():
    import paper_2011_07632_b200 as spd
    spd.lib()
    return spd


@pytest.mark.parametrize("name", ["R1", "R2"])
def test_rpy_table3_ball_4e4(spd, name):
    import torch
    from oracle.kernels import dof_points, rpy_matrix
    cfg = synth.CONFIGS[name]
    X = synth.points(cfg)
    h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    assert h.n == 3 * cfg.n
    # sampled rows of K x by direct sums (oracle RPY tensor)
    x = synth.multivec(cfg.dofs, 2)
    y = host(spd.h2_matvec(h, cuda(x)))
    rows = np.random.default_rng(1).choice(cfg.dofs, 200, replace=False)
    D = dof_points(X)
    ref = rpy_matrix(cfg.ell, D[rows], D) @ x
    err = np.linalg.norm(y[rows] - ref) / np.linalg.norm(ref)
    assert err <= 10 * cfg.h2_tol, err
    H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=5)
    b = cuda(synth.rhs(cfg))
    _, rh = spd.pcg_solve(h, H, b, tol=cfg.pcg_tol, maxit=cfg.maxit)
    _, rb = spd.pcg_solve(h, H, b, tol=cfg.pcg_tol, maxit=cfg.maxit, precond="bj")
    _, rn = spd.pcg_solve(h, None, b, tol=cfg.pcg_tol, maxit=cfg.maxit)
    ph, pb, pn = PAPER[name]
    print(f"{name}: H2 sampled error {err:.2e}; PCG iterations SPDHSS {rh.iters} (paper {ph}), "
          f"BJ {rb.iters} (paper {pb}), none {rn.iters} (paper {pn}); HSS max rank {H.ranks().max()}")
    assert rh.converged and rb.converged and rn.converged
    assert rh.iters < rb.iters < rn.iters
    assert abs(rh.iters - ph) <= 0.25 * ph
    assert abs(rb.iters - pb) <= 0.25 * pb
    assert abs(rn.iters - pn) <= 0.35 * pn
