"""GPU <-> oracle parity at the BASELINE configs' own parameters (SURVEY.md §8(c)
parity protocol).

Cases (tests/golden/make_parity_goldens.py wrote the oracle's results; Omega is the
counter-based Philox sketch of reading R29, generated on the device by the
production path and by oracle/omega.py for the golden):
  C1      the C1 config itself (N = 2048, leaf 64, cap 50, w = 60)
  C2p     C2 recipe at N = 8192 (Matern, leaf 128, cap 100, w = 110)
  C3p     C3 recipe at N = 8192 (sphere, exponential, leaf 128, cap 100)
  C4p     C4 recipe at N = 16384 (IMQ, leaf 256, cap 150, w = 160)
  C5p     C5 recipe at N = 16384 (Gaussian l = 0.2, leaf 256): products k = 1 .. 256
  C2full  C2 itself (N = 32768): HSS and PCG iterations with the production Omega
Protocol: tree and lists bit-exact; every H2 skeleton set certified (R19: identical
or a tie within 16 sqrt(m) eps nu_0, replayed in the oracle); an H2 built with the
oracle's skeletons injected (spd_h2_opts.inject_skeletons) has exactly the oracle's
skeletons, and its HSS has exactly the oracle's ranks and pivots (modulo certified
ties); products, HSS apply and HSS solve within 1e-9 (relative Frobenius AND
elementwise max relative to the largest entry); PCG iterations within +-1, widened
only by the oracle's own drift under a change of summation order (R24).
"""
import importlib.util
import os

import numpy as np
import pytest

import synth
from gpu_util import cuda, host, rel
from parity_util import TreeInfo, certify_h2, certify_hss, maxrel, oracle_skel_dict

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
_spec = importlib.util.spec_from_file_location("make_parity_goldens",
                                               os.path.join(HERE, "golden", "make_parity_goldens.py"))
goldens = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(goldens)
CASES = list(goldens.CASES)
HSS_CASES = [c for c in CASES if goldens.CASES[c][2]]


@pytest.fixture(scope="module")
def spd():
    import paper_2011_07632_b200 as spd
    spd.lib()
    return spd


_cache = {}


def case(spd, name):
    if name not in _cache:
        import torch
        cfg, ks, do_hss = goldens.CASES[name]
        g = dict(np.load(os.path.join(HERE, "golden", "parity", f"{name}.npz")))
        X = synth.points(cfg)
        Xd = torch.tensor(X, device="cuda")
        h = spd.h2_build(Xd, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
        oskel = oracle_skel_dict(g["h2_rank"], g["h2_skel"])
        hi = spd.h2_build(Xd, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol, inject_skeletons=oskel)
        H = Hn = None
        if do_hss:
            seed = int(g["omega_seed"])
            H = spd.spdhss_build(hi, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=seed)
            Hn = spd.spdhss_build(h, cfg.rank_cap, cfg.hss_tol, cfg.oversample, seed=seed)
        _cache[name] = dict(cfg=cfg, ks=ks, g=g, X=X, h=h, hi=hi, H=H, Hn=Hn, oskel=oskel)
    return _cache[name]


@pytest.mark.parametrize("name", CASES)
def test_tree_and_lists_bit_exact(spd, name):
    c = case(spd, name)
    h, g = c["h"], c["g"]
    assert h.levels == int(g["levels"])
    np.testing.assert_array_equal(h.perm, g["perm"])
    np.testing.assert_array_equal(np.asarray(h.near_pairs()), g["near"])
    t3 = np.array(sorted(tuple(int(v) for v in r) for r in h.type3()), dtype=np.int32).reshape(-1, 3)
    np.testing.assert_array_equal(t3, g["type3"])


@pytest.mark.parametrize("name", [n for n in CASES if n != "C2full"])
def test_h2_skeletons_certified(spd, name):
    """Every node: the oracle's skeleton sequence, or a certified tie (R19) -- no
    percentage threshold."""
    c = case(spd, name)
    cfg, h, g = c["cfg"], c["h"], c["g"]
    info = TreeInfo(c["X"], cfg.kernel, cfg.leaf)
    nodes, same, ties, fails = certify_h2(info, cfg.kernel, cfg.ell, cfg.h2_tol, h.ranks(), h.skeletons(),
                                          oracle_skel=c["oskel"])
    print(f"{name}: {nodes} active nodes, {same} identical to the oracle, {ties} certified ties")
    assert not fails, fails[:5]
    assert same + ties == nodes


@pytest.mark.parametrize("name", CASES)
def test_injected_skeletons_are_the_oracles(spd, name):
    c = case(spd, name)
    g, hi = c["g"], c["hi"]
    np.testing.assert_array_equal(hi.ranks(), g["h2_rank"])
    sk = hi.skeletons()
    for i, s in c["oskel"].items():
        np.testing.assert_array_equal(sk[i], s)


def _products(spd, c, which, k):
    cfg, g = c["cfg"], c["g"]
    x = synth.multivec(cfg.dofs, k)
    y = host(spd.h2_matvec(c[which], cuda(x)))
    cols = g[f"mv{k}_cols"]
    return y[:, cols], g[f"mv{k}"]


@pytest.mark.parametrize("name,k", [(n, k) for n in CASES for k in goldens.CASES[n][1]])
def test_h2_products(spd, name, k):
    """Y = (K + sigma I) X on the GPU's own H2 and on the injected one: <= 1e-9
    (Frobenius and elementwise); k = 16 runs the 32-column tile, k = 64 / 256 the
    128-column tile (k = 256: two column tiles)."""
    c = case(spd, name)
    for which in ("h", "hi"):
        y, yo = _products(spd, c, which, k)
        assert rel(y, yo) <= 1e-9, (which, rel(y, yo))
        assert maxrel(y, yo) <= 1e-9, (which, maxrel(y, yo))


@pytest.mark.parametrize("name", HSS_CASES)
def test_hss_ranks_and_pivots(spd, name):
    """HSS on the injected H2 with the production (device Philox) Omega: ranks and
    pivots exactly the oracle's, modulo certified ties."""
    c = case(spd, name)
    cfg, g, H = c["cfg"], c["g"], c["H"]
    nn = c["hi"].nnodes
    nodes = list(range(1, nn))
    same, ties, fails = certify_hss(H.pivots(cfg.w), H.ranks(), nodes, g["hss_rank"], g["hss_piv"],
                                    g["hss_gap"], g["hss_idx2"], g["hss_margin"])
    print(f"{name}: {same} nodes identical, {ties} certified ties")
    assert not fails, fails[:5]


@pytest.mark.parametrize("name", HSS_CASES)
def test_hss_apply_and_solve(spd, name):
    c = case(spd, name)
    cfg, g = c["cfg"], c["g"]
    P = synth.multivec(cfg.dofs, 4, seed=11)
    B = synth.multivec(cfg.dofs, 2, seed=12)
    for which in ("H", "Hn"):
        H = c[which]
        if which == "Hn" and not _own_h2_identical(c):
            # the GPU's own H2 has certified ties: compare its HSS with itself only
            y = host(spd.hss_matvec(H, cuda(P)))
            assert rel(host(spd.hss_solve(H, cuda(y))), P) <= 1e-9
            continue
        y = host(spd.hss_matvec(H, cuda(P)))
        assert rel(y, g["hss_apply"]) <= 1e-9 and maxrel(y, g["hss_apply"]) <= 1e-9, which
        x = host(spd.hss_solve(H, cuda(B)))
        assert rel(x, g["hss_solve"]) <= 1e-9 and maxrel(x, g["hss_solve"]) <= 1e-9, which


def _own_h2_identical(c):
    g = c["g"]
    if not np.array_equal(c["h"].ranks(), g["h2_rank"]):
        return False
    sk = c["h"].skeletons()
    return all(np.array_equal(sk[i], s) for i, s in c["oskel"].items())


@pytest.mark.parametrize("name", HSS_CASES)
def test_pcg_iterations(spd, name):
    """+-1 iteration (north star), widened only by the oracle's own drift over other
    summation orders of its product (golden pcg_iters vs the reversed and shuffled
    orders, R24)."""
    c = case(spd, name)
    cfg, g = c["cfg"], c["g"]
    b = synth.rhs(cfg)
    it_o, it_rev = int(g["pcg_iters"]), int(g["pcg_iters_reversed"])
    others = [it_rev] + [int(v) for v in g.get("pcg_iters_shuffled", [])]
    window = max([1] + [abs(it_o - v) for v in others])
    for which_h, which_H in (("hi", "H"), ("h", "Hn")):
        if which_h == "h" and not _own_h2_identical(c):
            continue
        x, rep = spd.pcg_solve(c[which_h], c[which_H], cuda(b), tol=cfg.pcg_tol, maxit=20000)
        print(f"{name} ({which_h}): GPU {rep.iters} iterations, oracle {it_o}, other summation orders {others}")
        assert rep.converged and bool(g["pcg_converged"])
        assert abs(rep.iters - it_o) <= window, (rep.iters, it_o, it_rev)
        assert rel(host(x), g["pcg_x"]) <= 1e-6
