"""Subtree-sharded H2 build on one GPU through the library's
virtual communicator: every virtual rank computes its own subtrees' nodes in turn
(the code path of one NCCL rank, minus the transport), so the sharded build must
give the unsharded H2: the same tree, every skeleton set of both builds certified
against the oracle (identical or a certified tie, reading R19), and the same products."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda, host, rel
from parity_util import TreeInfo, certify_h2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spd():
    import paper_2011_07632_b200 as spd
    spd.lib()
    return spd


@pytest.mark.parametrize("name,P", [("C1s", 2), ("C2s", 2), ("C2s", 4), ("C3s", 8)])
def test_virtual_sharded_build_matches(spd, name, P):
    import torch
    cfg = {"C1s": synth.C1.scaled(1024, leaf=32), "C2s": synth.C2.scaled(2048, leaf=64),
           "C3s": synth.C3.scaled(4096, leaf=64)}[name]
    X = torch.tensor(synth.points(cfg), device="cuda")
    h1 = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    comm = spd.Comm(P, 0)
    hp = spd.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol, comm=comm)
    assert np.array_equal(h1.perm, hp.perm)
    Xh = synth.points(cfg)
    ho = oracle.h2_build(Xh, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol)
    info = TreeInfo(Xh, cfg.kernel, cfg.leaf)
    for h in (h1, hp):
        nodes, same, ties, fails = certify_h2(info, cfg.kernel, cfg.ell, cfg.h2_tol, h.ranks(), h.skeletons(),
                                              oracle_skel=ho.skel)
        assert not fails and same + ties == nodes, fails[:5]
    x = synth.multivec(cfg.n, 3)
    assert rel(host(spd.h2_matvec(hp, cuda(x))), host(spd.h2_matvec(h1, cuda(x)))) <= 1e-11
