"""GPU edge cases the oracle pins (SURVEY.md §8(c) "Textbook special cases"):

* identity-like kernel (Gaussian, l -> 0: every off-diagonal entry underflows to 0):
  all H2 and HSS ranks 0, HSS = (1 + sigma) I exactly, the solve is b / (1 + sigma),
  PCG converges in one iteration -- the oracle gives the same;
* no truncation (HSS tolerance below rounding, cap above every node's rows): the
  SPD-HSS matrix IS the H2 matrix, so hss_solve inverts the H2 product and PCG
  converges in at most two iterations;
* not positive definite (reading R18): a numerically singular leaf block
  (Gaussian with l >> the box, sigma = 0) fails the leaf Cholesky with SPD_ENOTPD,
  naming level 1 and the same first failing leaf as the oracle.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda, host, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spd():
    import paper_2011_07632_b200 as spd
    spd.lib()
    return spd


def _pts(cfg):
    import torch
    return torch.tensor(synth.points(cfg), device="cuda")


def test_identity_like_kernel(spd):
    cfg = synth.C1.scaled(512, leaf=32, ell=1e-6, shift=0.5, rank_cap=16)
    h = spd.h2_build(_pts(cfg), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    assert np.all(h.ranks() == 0)
    H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=3)
    assert np.all(H.ranks() == 0)
    b = synth.rhs(cfg)
    np.testing.assert_allclose(host(spd.hss_solve(H, cuda(b))), b / 1.5, rtol=1e-15, atol=0)
    np.testing.assert_allclose(host(spd.h2_matvec(h, cuda(b))), 1.5 * b, rtol=1e-15, atol=0)
    x, rep = spd.pcg_solve(h, H, cuda(b), tol=1e-12, maxit=10)
    assert rep.converged and rep.iters == 1
    ho = oracle.h2_build(synth.points(cfg), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    Ho = oracle.spdhss_build(ho, cfg.rank_cap, cfg.hss_tol, synth.omega(cfg), form="chol")
    assert all(r == 0 for r in ho.rank.values()) and all(r == 0 for r in Ho.rank.values())


def test_no_truncation_hss_is_the_h2(spd):
    cfg = synth.C1.scaled(256, leaf=32, rank_cap=128, hss_tol=1e-15)
    h = spd.h2_build(_pts(cfg), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, 1e-14)
    H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=5)
    X = synth.multivec(cfg.n, 6, seed=2)
    AX = host(spd.h2_matvec(h, cuda(X)))
    assert rel(host(spd.hss_matvec(H, cuda(X))), AX) <= 1e-11
    assert rel(host(spd.hss_solve(H, cuda(AX))), X) <= 1e-9
    b = synth.rhs(cfg)
    x, rep = spd.pcg_solve(h, H, cuda(b), tol=1e-8, maxit=10)
    assert rep.converged and rep.iters <= 2


def test_not_positive_definite_leaf(spd):
    cfg = synth.C1.scaled(256, leaf=32, ell=50.0, shift=0.0, rank_cap=8)
    X = synth.points(cfg)
    h = spd.h2_build(_pts(cfg), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    with pytest.raises(spd.NotPositiveDefinite) as e:
        spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=1)
    msg = str(e.value)
    ho = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    with pytest.raises(oracle.NotPD) as eo:
        oracle.spdhss_build(ho, cfg.rank_cap, cfg.hss_tol, synth.omega(cfg), form="chol")
    level, node = eo.value.where
    assert level == 1
    assert f"level 1 node {node}" in msg, (msg, eo.value.where)
    assert e.value.code == spd.SPD_ENOTPD
