"""GPU parity of spdhss_build / hss_solve / pcg_solve against the CPU oracle
(same seeded points and injected Omega): HSS ranks, the exported HSS applied
by the oracle's HSS matvec (<= 1e-9), the solve (<= 1e-9), SPD, PCG iterations
within +-1."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda, host, rel
from oracle.certify import hss_tie_records
from parity_util import certify_hss

pytestmark = pytest.mark.gpu

CASES = {
    "C1s": synth.C1.scaled(1024, leaf=32, rank_cap=20),
    "C1": synth.C1,
    "C2s": synth.C2.scaled(2048, leaf=64, rank_cap=30),
    "C3s": synth.C3.scaled(2048, leaf=64, rank_cap=30),
    "C4s": synth.C4.scaled(4096, leaf=128, rank_cap=40),
    "ragged": synth.C1.scaled(1000, leaf=50, rank_cap=16),
    "L2": synth.C1.scaled(128, leaf=64, rank_cap=20),
    "L1": synth.C1.scaled(60, leaf=64, rank_cap=20),
    "R1s": synth.R1.scaled(800, leaf=64, h2_tol=1e-4, rank_cap=30),
    "R2s": synth.R2.scaled(1200, leaf=64, h2_tol=1e-6, rank_cap=40),
}


@pytest.fixture(scope="module")
def spd():
    import paper_2011_07632_b200 as spd
    spd.lib()
    return spd


_cache = {}


def built(spd, name):
    if name not in _cache:
        import torch
        cfg = CASES[name]
        X = synth.points(cfg)
        ho = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
        # the oracle's skeletons injected (R19 protocol step 4: later stages compared on
        # the oracle's state; the GPU's own skeletons are certified in test_gpu_h2.py)
        h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol,
                         inject_skeletons=ho.skel)
        om = synth.omega(cfg)
        Ho = oracle.spdhss_build(ho, cfg.rank_cap, cfg.hss_tol, om, form="chol", keep_sketch=True)
        H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, omega=cuda(om))
        _cache[name] = (cfg, X, h, ho, H, Ho, om)
    return _cache[name]


def drift_window(ho, apply_M, b, tol, maxit, it_o):
    """+-1, widened only by the oracle's own drift: the same PCG with the oracle's
    product summed in other orders -- reverse list order and five seeded shuffles
    (reading R24); the window is the largest deviation among those runs."""
    its = [oracle.pcg(lambda v: oracle.h2_matvec(ho, v, reverse=True), apply_M, b, tol, maxit)[1]]
    if it_o > 100:                      # long runs: sample more orders
        for sd in (1, 2, 3, 4, 5):
            its.append(oracle.pcg(lambda v, sd=sd: oracle.h2_matvec(ho, v, shuffle=sd), apply_M, b, tol, maxit)[1])
    return max([1] + [abs(i - it_o) for i in its]), its


def gpu_as_oracle_hss(H, ho):
    """Wrap the exported GPU HSS in the oracle's HSS container (for its matvec)."""
    t = ho.tree
    ranks = H.ranks()
    flat = H.export()
    G = oracle.HSS(ho, "gpu")
    off = 0
    for i in t.nodes_at(1):
        n = t.size(i)
        G.D[i] = flat[off:off + n * n].reshape(n, n, order="F"); off += n * n
        r = int(ranks[i])
        G.U[i] = flat[off:off + n * r].reshape(n, r, order="F"); off += n * r
        G.rank[i] = r
    for k in range(2, t.L):
        for i in t.nodes_at(k):
            c1, c2 = t.children(i)
            m, r = G.rank[c1] + G.rank[c2], int(ranks[i])
            G.R[i] = flat[off:off + m * r].reshape(m, r, order="F"); off += m * r
            G.rank[i] = r
    for p in range(t.nnodes):
        if t.level(p) < 2:
            continue
        c1, c2 = t.children(p)
        n = G.rank[c1] * G.rank[c2]
        G.B[(c1, c2)] = flat[off:off + n].reshape(G.rank[c1], G.rank[c2], order="F"); off += n
    assert off == flat.size or (off == 0 and flat.size == 1)
    return G


@pytest.mark.parametrize("name", [n for n in CASES if n != "L1"])
def test_hss_ranks_and_apply_match_oracle(spd, name):
    cfg, X, h, ho, H, Ho, om = built(spd, name)
    rank, piv, gap, idx2, margin = hss_tie_records(Ho, cfg.rank_cap, cfg.hss_tol, cfg.w)
    nodes = sorted(Ho.rank)
    same, ties, fails = certify_hss(H.pivots(cfg.w), H.ranks(), nodes, rank, piv, gap, idx2, margin)
    assert not fails, fails[:5]           # ranks and pivots exact modulo certified ties (R19)
    G = gpu_as_oracle_hss(H, ho)
    x = synth.multivec(cfg.dofs, 10, seed=11)
    yg = oracle.hss_matvec(G, x)
    yo = oracle.hss_matvec(Ho, x)
    assert rel(yg, yo) <= 1e-9


@pytest.mark.parametrize("name", list(CASES))
def test_hss_solve_matches_oracle(spd, name):
    cfg, X, h, ho, H, Ho, om = built(spd, name)
    b = synth.multivec(cfg.dofs, 3, seed=12)
    xg = host(spd.hss_solve(H, cuda(b)))
    xo = np.empty_like(b)
    xo[ho.tree.perm] = oracle.hss_solve(Ho, b[ho.tree.perm])
    assert rel(xg, xo) <= 1e-9
    if ho.tree.L > 1:        # residual of the GPU solve against the GPU HSS (oracle apply)
        G = gpu_as_oracle_hss(H, ho)
        res = oracle.hss_matvec(G, xg[ho.tree.perm]) - b[ho.tree.perm]
        assert np.linalg.norm(res) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("name", list(CASES))
def test_hss_matvec_matches_oracle_and_inverts(spd, name):
    """hss_matvec (the HSS matrix itself) against the oracle's product on the
    exported GPU factors, and hss_solve(hss_matvec(x)) = x."""
    cfg, X, h, ho, H, Ho, om = built(spd, name)
    x = synth.multivec(cfg.dofs, 3, seed=13)
    yg = host(spd.hss_matvec(H, cuda(x)))
    if ho.tree.L > 1:
        G = gpu_as_oracle_hss(H, ho)
        perm = ho.tree.perm
        yo = np.empty_like(x)
        yo[perm] = oracle.hss_matvec(G, x[perm])
        assert rel(yg, yo) <= 1e-12
    assert rel(host(spd.hss_solve(H, cuda(yg))), x) <= 1e-9


def test_gpu_hss_is_spd(spd):
    cfg, X, h, ho, H, Ho, om = built(spd, "C1")
    G = gpu_as_oracle_hss(H, ho)
    D = oracle.hss_densify(G)
    assert np.abs(D - D.T).max() <= 1e-12 * np.abs(D).max()
    assert np.linalg.eigvalsh(0.5 * (D + D.T)).min() > 0


@pytest.mark.parametrize("name", ["C1s", "C1", "C2s", "C4s", "R1s", "R2s"])
def test_pcg_iterations_match_oracle(spd, name):
    cfg, X, h, ho, H, Ho, om = built(spd, name)
    b = synth.rhs(cfg)
    xg, rep = spd.pcg_solve(h, H, cuda(b), tol=cfg.pcg_tol, maxit=cfg.maxit)
    perm = ho.tree.perm
    xo_t, it_o, conv_o, _ = oracle.pcg(lambda v: oracle.h2_matvec(ho, v), lambda v: oracle.hss_solve(Ho, v),
                                       b[perm], cfg.pcg_tol, cfg.maxit)
    assert rep.converged and conv_o
    window, it_rev = drift_window(ho, lambda v: oracle.hss_solve(Ho, v), b[perm], cfg.pcg_tol, cfg.maxit, it_o)
    assert abs(rep.iters - it_o) <= window, (rep.iters, it_o, it_rev)
    xo = np.empty_like(b)
    xo[perm] = xo_t
    assert rel(host(xg), xo) <= 1e-6
    # true residual through the GPU H2 operator, and the report's own
    r = b - host(spd.h2_matvec(h, xg))
    assert np.linalg.norm(r) <= 2 * cfg.pcg_tol * np.linalg.norm(b)
    assert abs(rep.relres_true - np.linalg.norm(r) / np.linalg.norm(b)) <= 1e-3 * cfg.pcg_tol


def test_philox_omega_path(spd):
    """Omega generated on the device (no parity hook): still SPD, solve exact."""
    import torch
    cfg = CASES["C1s"]
    cfg_, X, h, ho, H, Ho, om = built(spd, "C1s")
    H2 = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=7)
    G = gpu_as_oracle_hss(H2, ho)
    D = oracle.hss_densify(G)
    assert np.linalg.eigvalsh(0.5 * (D + D.T)).min() > 0
    b = synth.multivec(cfg.n, 2, seed=3)
    xg = host(spd.hss_solve(H2, cuda(b)))
    assert rel(D @ xg[ho.tree.perm], b[ho.tree.perm]) < 1e-10


def test_unpreconditioned_cg_and_trivial_rhs(spd):
    cfg, X, h, ho, H, Ho, om = built(spd, "C1s")
    b = synth.rhs(cfg)
    x, rep = spd.pcg_solve(h, None, cuda(b), tol=1e-8, maxit=5000)
    _, it_o, _, _ = oracle.pcg(lambda v: oracle.h2_matvec(ho, v), lambda v: v, b[ho.tree.perm], 1e-8, 5000)
    window, it_rev = drift_window(ho, lambda v: v, b[ho.tree.perm], 1e-8, 5000, it_o)
    assert rep.converged and abs(rep.iters - it_o) <= window, (rep.iters, it_o, it_rev)
    z, rep0 = spd.pcg_solve(h, H, cuda(np.zeros(cfg.n)), tol=1e-8, maxit=10)
    assert rep0.iters == 0 and rep0.converged and np.all(host(z) == 0)


@pytest.mark.parametrize("stored", ["0", "1", "partial"])
def test_pcg_stored_and_on_the_fly_k1_paths(spd, stored, monkeypatch):
    """All k=1 matvec paths (legacy per-level on-the-fly kernels; symmetric stored
    blocks, §8(f) f4; symmetric with half the blocks evaluated on the fly) give the
    oracle's PCG iterations and, afterwards, oracle-exact k=1 products."""
    import torch
    if stored == "partial":
        monkeypatch.setenv("SPD_SYM_BUDGET", str(4 << 20))    # ~half of the C2s blocks
    else:
        monkeypatch.setenv("SPD_STORED", stored)
    cfg = CASES["C2s"]
    X = synth.points(cfg)
    cfg_, X_, h_, ho, H_, Ho, om = built(spd, "C2s")
    h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol,
                     inject_skeletons=ho.skel)
    H = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, omega=cuda(om))
    b = synth.rhs(cfg)
    x, rep = spd.pcg_solve(h, H, cuda(b), tol=cfg.pcg_tol, maxit=cfg.maxit)
    _, it_o, _, _ = oracle.pcg(lambda v: oracle.h2_matvec(ho, v), lambda v: oracle.hss_solve(Ho, v),
                               b[ho.tree.perm], cfg.pcg_tol, cfg.maxit)
    assert rep.converged and abs(rep.iters - it_o) <= 1
    v = synth.multivec(cfg.n, 1, seed=21)[:, 0]
    y = host(spd.h2_matvec(h, cuda(v)))
    yo = np.empty_like(v)
    yo[ho.tree.perm] = oracle.h2_matvec(ho, v[ho.tree.perm])
    assert rel(y, yo) <= 1e-9


@pytest.mark.parametrize("name", ["C1s", "C2s", "C4s"])
def test_pcg_block_jacobi_matches_oracle(spd, name):
    """Block-Jacobi PCG (leaf Cholesky factors of the SPD-HSS build, the paper's BJ
    baseline) against the oracle's BJ PCG: iterations within R24's drift."""
    cfg, X, h, ho, H, Ho, om = built(spd, name)
    b = synth.rhs(cfg)
    x, rep = spd.pcg_solve(h, H, cuda(b), tol=cfg.pcg_tol, maxit=cfg.maxit, precond="bj")
    _, it_o, conv_o, _ = oracle.pcg(lambda v: oracle.h2_matvec(ho, v), lambda v: oracle.block_jacobi_solve(ho, v),
                                    b[ho.tree.perm], cfg.pcg_tol, cfg.maxit)
    assert rep.converged == conv_o
    window, it_rev = drift_window(ho, lambda v: oracle.block_jacobi_solve(ho, v), b[ho.tree.perm],
                                  cfg.pcg_tol, cfg.maxit, it_o)
    assert abs(rep.iters - it_o) <= window, (rep.iters, it_o, it_rev)
    # the GPU solution solves the oracle's H2 system to the PCG tolerance
    xg = host(x)[ho.tree.perm]
    res = oracle.h2_matvec(ho, xg) - b[ho.tree.perm]
    assert np.linalg.norm(res) <= 1e-7 * np.linalg.norm(b)


@pytest.mark.parametrize("name", ["C1s", "C2s"])
def test_adaptive_build_matches_oracle(spd, name):
    """Threshold-driven build (R27) with the same injected sketch: the GPU
    picks the oracle's cap, the same ranks, and the same HSS (applied by the oracle)."""
    import torch
    cfg = CASES[name]
    X = synth.points(cfg)
    ho = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol,
                     inject_skeletons=ho.skel)
    r_max = 64
    om = synth.omega(cfg, w=r_max + cfg.oversample)
    Ho, cap_o = oracle.spdhss_build_adaptive(ho, cfg.hss_tol, 4, r_max, om, p=cfg.oversample, form="chol")
    H, cap = spd.spdhss_build_adaptive(h, 4, r_max, cfg.hss_tol, cfg.oversample, omega=cuda(om))
    assert cap == cap_o
    rg = H.ranks()
    assert all(int(rg[i]) == r for i, r in Ho.rank.items())
    G = gpu_as_oracle_hss(H, ho)
    v = synth.multivec(cfg.n, 3, seed=8)[ho.tree.perm]
    assert rel(oracle.hss_matvec(G, v), oracle.hss_matvec(Ho, v)) <= 1e-9
