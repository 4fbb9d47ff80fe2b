"""GPU parity of h2_build / h2_matvec against the CPU oracle (tree, lists and
proxies bit-exact; skeletons modulo certified ties; products <= 1e-9)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda, host, rel
from parity_util import TreeInfo, certify_h2

pytestmark = pytest.mark.gpu

CASES = {
    "C1s": synth.C1.scaled(1024, leaf=32),
    "C2s": synth.C2.scaled(2048, leaf=64),
    "C3s": synth.C3.scaled(2048, leaf=64),
    "C4s": synth.C4.scaled(4096, leaf=128),
    "ragged": synth.C1.scaled(1000, leaf=50),
    # RPY tensor kernel over 3 dofs per point (§8(f) f1, R28); loose tols so IDs truncate
    "R1s": synth.R1.scaled(800, leaf=64, h2_tol=1e-4),
    "R2s": synth.R2.scaled(1200, leaf=64, h2_tol=1e-6),
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
        h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
        ho = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
        _cache[name] = (cfg, X, h, ho)
    return _cache[name]


@pytest.mark.parametrize("name", list(CASES))
def test_tree_and_lists_bit_exact(spd, name):
    cfg, X, h, ho = built(spd, name)
    t = ho.tree
    assert h.levels == t.L
    np.testing.assert_array_equal(h.perm, t.perm)
    nodes = h.nodes()
    np.testing.assert_array_equal(nodes[:, 0], t.begin)
    np.testing.assert_array_equal(nodes[:, 1], t.end)
    bx = h.boxes()
    np.testing.assert_array_equal(bx[:, 0], t.lo)
    np.testing.assert_array_equal(bx[:, 1], t.hi)
    near = [tuple(p) for p in h.near_pairs()]
    assert near == ho.lists.near
    t3 = sorted((int(k), int(i), int(j)) for k, i, j in h.type3())
    assert t3 == sorted((k, i, j) for k in ho.lists.type3 for (i, j) in ho.lists.type3[k])
    t1 = sorted((int(k), int(i), int(j)) for k, i, j in h.type1())
    assert t1 == sorted((k, i, j) for k in ho.lists.type1 for (i, j) in ho.lists.type1[k])


@pytest.mark.parametrize("name", ["C1s", "C3s"])
def test_proxies_bit_exact(spd, name):
    cfg, X, h, ho = built(spd, name)
    import paper_2011_07632_b200 as m
    for node in [1, 3, ho.tree.nnodes // 2, ho.tree.nnodes - 1]:
        Pg = m._proxies(h, node, ho.n_proxy)
        Po = oracle.proxy_points(ho.tree, node, ho.n_proxy)
        np.testing.assert_array_equal(Pg, Po)


@pytest.mark.parametrize("name", list(CASES))
def test_skeletons(spd, name):
    """Every node's skeleton sequence is the oracle's or a certified tie (R19): replayed
    in the oracle's QRCP, each deviating pivot within 16 sqrt(m) eps nu_0 of the largest
    residual norm and the rank within that band of the threshold.  No percentage window."""
    cfg, X, h, ho = built(spd, name)
    info = TreeInfo(X, cfg.kernel, cfg.leaf)
    nodes, same, ties, fails = certify_h2(info, cfg.kernel, cfg.ell, cfg.h2_tol, h.ranks(), h.skeletons(),
                                          oracle_skel=ho.skel, n_proxy=ho.n_proxy)
    print(f"{name}: {nodes} active nodes, {same} identical, {ties} certified ties")
    assert not fails, fails[:5]
    assert same + ties == nodes


def test_injected_skeletons(spd):
    """The parity hook spd_h2_opts.inject_skeletons (R19): the GPU ID takes the oracle's
    pivots, so its skeletons are the oracle's and its products match to <= 1e-9."""
    import torch
    cfg, X, h, ho = built(spd, "C2s")
    inj = {i: s for i, s in ho.skel.items()}
    hi = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol,
                      inject_skeletons=inj)
    sk = hi.skeletons()
    for i, s in ho.skel.items():
        np.testing.assert_array_equal(sk.get(i, np.zeros(0, np.int64)), s)
    x = synth.multivec(cfg.n, 3)
    yo = np.empty_like(x)
    yo[ho.tree.perm] = oracle.h2_matvec(ho, x[ho.tree.perm])
    assert rel(host(spd.h2_matvec(hi, cuda(x))), yo) <= 1e-9
    # a skeleton that is not a candidate of its node is rejected
    bad = dict(inj)
    leaf = ho.tree.nodes_at(1)[0]
    bad[leaf] = np.array([ho.tree.N - 1])
    with pytest.raises(spd.SpdError):
        spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol,
                     inject_skeletons=bad)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("k", [1, 7, 64])
def test_h2_matvec_vs_oracle(spd, name, k):
    cfg, X, h, ho = built(spd, name)
    x = synth.multivec(cfg.dofs, k)
    y = host(spd.h2_matvec(h, cuda(x)))
    yo = np.empty_like(x)
    yo[ho.tree.perm] = oracle.h2_matvec(ho, x[ho.tree.perm])
    assert rel(y, yo) <= 1e-9
    # tree layout gives the permuted result
    yt = host(spd.h2_matvec(h, cuda(x[ho.tree.perm]), layout=1))
    assert rel(yt, yo[ho.tree.perm]) <= 1e-9


@pytest.mark.parametrize("mode", ["evaluated", "mv_eval", "stored"])
@pytest.mark.parametrize("k", [7, 64])
def test_h2_matvec_block_source_paths(spd, mode, k, monkeypatch):
    """Every source of the kernel blocks of a multi-vector product gives the oracle's
    product: evaluated on the fly (SPD_STORE_FRAC=0: no store is built), evaluated although
    a store exists (SPD_MV_EVAL=1), read from the symmetric store (kmode 1/2).  The
    environment is read on every call (advisor, round 1)."""
    import torch
    cfg = CASES["C2s"]
    X = synth.points(cfg)
    h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    _, _, _, ho = built(spd, "C2s")
    if mode == "evaluated":
        monkeypatch.setenv("SPD_STORE_FRAC", "0")
    else:
        spd.pcg_solve(h, None, cuda(synth.rhs(cfg)), tol=1e-300, maxit=1)     # builds the store
        assert h.sym_store()[0] > 0
        if mode == "mv_eval":
            monkeypatch.setenv("SPD_MV_EVAL", "1")
    x = synth.multivec(cfg.n, k)
    y = host(spd.h2_matvec(h, cuda(x)))
    if mode == "evaluated":
        assert h.sym_store()[0] == 0
    yo = np.empty_like(x)
    yo[ho.tree.perm] = oracle.h2_matvec(ho, x[ho.tree.perm])
    assert rel(y, yo) <= 1e-9
    h.release_store()
    assert h.sym_store()[0] == 0
    assert rel(host(spd.h2_matvec(h, cuda(x))), yo) <= 1e-9


def test_h2_matvec_replayed_plan(spd, monkeypatch):
    """h2_matvec keeps the kblock plan of its last multi-column product in the handle and
    replays it while the width, buffers, sharding and block store are unchanged: the replayed
    product is bitwise the planned one, also after products of other widths and after the
    store is built / released, and equals the oracle's."""
    import torch
    cfg = CASES["C2s"]
    X = synth.points(cfg)
    h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    _, _, _, ho = built(spd, "C2s")
    monkeypatch.setenv("SPD_STORE_FRAC", "0")
    xa, xb = synth.multivec(cfg.n, 64), synth.multivec(cfg.n, 16)
    ya = host(spd.h2_matvec(h, cuda(xa)))
    assert np.array_equal(host(spd.h2_matvec(h, cuda(xa))), ya)          # replayed plan
    yb = host(spd.h2_matvec(h, cuda(xb)))                                 # another width: new plan
    assert np.array_equal(host(spd.h2_matvec(h, cuda(xa))), ya)
    assert np.array_equal(host(spd.h2_matvec(h, cuda(xa))), ya)
    assert np.array_equal(host(spd.h2_matvec(h, cuda(xb))), yb)
    x2 = 2.0 * xa - 1.0                                                    # same buffers, other data
    monkeypatch.setenv("SPD_MV_NOCACHE", "1")
    y2 = host(spd.h2_matvec(h, cuda(x2)))
    monkeypatch.delenv("SPD_MV_NOCACHE")
    assert np.array_equal(host(spd.h2_matvec(h, cuda(x2))), y2)
    monkeypatch.delenv("SPD_STORE_FRAC")
    spd.pcg_solve(h, None, cuda(synth.rhs(cfg)), tol=1e-300, maxit=1)     # builds the store
    ys = host(spd.h2_matvec(h, cuda(xa)))                                 # store: new plan
    assert np.array_equal(host(spd.h2_matvec(h, cuda(xa))), ys)
    h.release_store()                                  # (the next product may rebuild it on demand)
    monkeypatch.setenv("SPD_STORE_FRAC", "0")
    assert np.array_equal(host(spd.h2_matvec(h, cuda(xa))), ya)          # evaluated again: a new plan
    yo = np.empty_like(xa)
    yo[ho.tree.perm] = oracle.h2_matvec(ho, xa[ho.tree.perm])
    assert rel(ya, yo) <= 1e-9 and rel(ys, yo) <= 1e-9


def test_h2_matvec_vs_dense_kernel(spd):
    cfg, X, h, ho = built(spd, "C1s")
    from oracle.kernels import kernel_matrix
    idx = np.arange(cfg.n)
    A = kernel_matrix(cfg.kernel, cfg.ell, X, X, cfg.shift, idx, idx)
    x = synth.multivec(cfg.n, 5)
    y = host(spd.h2_matvec(h, cuda(x)))
    assert rel(y, A @ x) <= 10 * cfg.h2_tol


def test_h2_full_c2_sampled_rows(spd):
    """C2 at full size: sampled rows of K x by direct O(N) sums."""
    import torch
    from oracle.kernels import kernel_matrix
    cfg = synth.C2
    X = synth.points(cfg)
    h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    x = synth.multivec(cfg.n, 2)
    y = host(spd.h2_matvec(h, cuda(x)))
    rows = np.random.default_rng(0).choice(cfg.n, 300, replace=False)
    K = kernel_matrix(cfg.kernel, cfg.ell, X[rows], X, cfg.shift, rows, np.arange(cfg.n))
    ref = K @ x
    err = np.linalg.norm(y[rows] - ref) / np.linalg.norm(ref)
    print("C2 sampled-row H2 error", err, "ranks", np.bincount(h.ranks())[:0], h.timings()[:2])
    assert err <= 10 * cfg.h2_tol


@pytest.mark.parametrize("cfg", [synth.C4, synth.C3, synth.C1.scaled(3001, leaf=40)], ids=["C4", "C3", "ragged2D"])
def test_device_tree_lists_equal_host_builder_full_size(spd, cfg):
    """K12: the device tree and dual-tree lists (tree_dev.cu) at full size (N = 2^20 for
    C4/C5) equal the host builder (tree.cpp), itself bit-exact with the oracle above."""
    import torch
    X = synth.points(cfg)
    h = spd.h2_build(torch.tensor(X, device="cuda"), cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, 1e-3)
    perm, boxes, counts = spd.tree_host(X, cfg.leaf)
    np.testing.assert_array_equal(h.perm, perm)
    np.testing.assert_array_equal(h.boxes(), boxes)
    np.testing.assert_array_equal(h.list_counts(), counts)
