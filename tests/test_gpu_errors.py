"""Error paths and degenerate inputs of the C ABI on the GPU (include/spdhss.h's
"Errors" contract): invalid arguments give SPD_EINVAL with a message,
a PCG that hits maxit SPD_ENOCONV with the report filled (not fatal), and empty or
zero right-hand sides are no-ops.  (SPD_ENOTPD needs an indefinite operator, which
the kernels with shift >= 0 cannot produce; the negative shift that would is itself
rejected as SPD_EINVAL.)"""
import ctypes

import numpy as np
import pytest

import synth
from gpu_util import cuda, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spd():
    import paper_2011_07632_b200 as spd
    spd.lib()
    return spd


@pytest.fixture(scope="module")
def small(spd):
    import torch
    cfg = synth.C1.scaled(512, leaf=32, rank_cap=20)
    X = torch.tensor(synth.points(cfg), device="cuda")
    h = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=1)
    return cfg, h, H


def test_invalid_build_arguments(spd):
    import torch
    with pytest.raises(spd.SpdError) as e:
        spd.h2_build(torch.zeros((0, 3), dtype=torch.float64, device="cuda"), 1, 0.2, 0.0, 32, 1e-8)
    assert e.value.code == 1 and "n >= 1" in str(e.value)
    pts4 = torch.rand((64, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(spd.SpdError) as e:
        spd.h2_build(pts4, 1, 0.2, 0.0, 32, 1e-8)
    assert e.value.code == 1
    pts2 = torch.rand((64, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(spd.SpdError):                  # RPY needs 3D points
        spd.h2_build(pts2, spd.K_RPY, 0.3, 0.0, 32, 1e-8)
    pts3 = torch.rand((64, 3), dtype=torch.float64, device="cuda")
    for bad in ((9, 0.2, 0.0, 32, 1e-8), (1, -0.2, 0.0, 32, 1e-8), (1, 0.2, -1.0, 32, 1e-8),
                (1, 0.2, 0.0, 0, 1e-8), (1, 0.2, 0.0, 32, 1.5)):
        with pytest.raises(spd.SpdError) as e:
            spd.h2_build(pts3, *bad)
        assert e.value.code == 1
    pts3[3, 1] = float("nan")
    with pytest.raises(spd.SpdError):
        spd.h2_build(pts3, 1, 0.2, 0.0, 32, 1e-8)


def test_invalid_product_arguments(spd, small):
    cfg, h, H = small
    lib = spd.lib()
    x = cuda(np.ones((cfg.n, 2)))
    y = cuda(np.zeros((cfg.n, 2)))
    st = lib.h2_matvec(h.ptr, 0, ctypes.c_void_p(x.data_ptr()), cfg.n - 1, ctypes.c_void_p(y.data_ptr()), cfg.n, 2,
                       spd._stream())
    assert st == 1 and b"ld" in lib.spd_last_error()
    st = lib.h2_matvec(h.ptr, 7, ctypes.c_void_p(x.data_ptr()), cfg.n, ctypes.c_void_p(y.data_ptr()), cfg.n, 2,
                       spd._stream())
    assert st == 1
    st = lib.hss_solve(H.ptr, 0, None, cfg.n, None, cfg.n, 0, spd._stream())       # nrhs = 0: no-op
    assert st == 0


def test_pcg_maxit_is_not_fatal(spd, small):
    cfg, h, H = small
    b = cuda(synth.rhs(cfg))
    x, rep = spd.pcg_solve(h, H, b, tol=1e-14, maxit=3)
    assert rep.iters == 3 and not rep.converged and np.isfinite(rep.relres) and rep.relres > 1e-14
    assert np.isfinite(host(x)).all()


def test_zero_rhs(spd, small):
    cfg, h, H = small
    x, rep = spd.pcg_solve(h, H, cuda(np.zeros(cfg.n)))
    assert rep.converged and rep.iters == 0 and np.all(host(x) == 0.0)
