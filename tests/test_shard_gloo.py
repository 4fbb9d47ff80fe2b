"""World-size-2 gloo test (CPU) of the subtree-sharded H2 build protocol of
libspdhss (comm.cpp / h2.cu):

* the ownership plan comes from the library itself (spd_test_shard_owner: rank p
  owns the contiguous node range of subtree p at every level with >= P nodes,
  levels with fewer nodes are computed by every rank);
* each rank computes, with the oracle's per-node proxy-ID step (R3/R4),
  only the nodes it owns, packs the level arrays in node order (ranks, then the
  interpolation matrices and skeletons at their cumulative offsets), all-reduces
  the ranks and broadcasts its contiguous ranges -- the same exchange the library
  issues with NCCL;
* afterwards both ranks must hold exactly the unsharded oracle build.
"""
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _node_id(h, i, n_proxy):
    """The oracle's per-node ID step (oracle.h2.h2_build loop body)."""
    from oracle.h2 import proxy_points
    from oracle.kernels import kernel_matrix
    from oracle.linalg import qrcp
    from scipy.linalg import solve_triangular
    cand = h.candidates(i)
    Y = proxy_points(h.tree, i, n_proxy)
    M = kernel_matrix(h.kid, h.ell, h.Xt[cand], Y)
    _, R, piv, s = qrcp(M.T, min(M.shape), h.tol, want_q=False)
    T = solve_triangular(R[:s, :s], R[:s, s:]) if s > 0 else np.zeros((0, len(cand) - s))
    E = np.zeros((len(cand), s))
    E[piv[:s], np.arange(s)] = 1.0
    E[piv[s:], :] = T.T
    return cand[piv[:s]], E, s


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2011_07632_b200 as spd
    import oracle
    from oracle.h2 import H2, active_nodes
    from oracle.tree import build_tree, interaction_lists
    import synth
    cfg = synth.C1.scaled(512, leaf=32)
    n_proxy = 512
    X = synth.points(cfg)
    tree = build_tree(X, cfg.leaf)
    lists = interaction_lists(tree)
    Xt = X[tree.perm]
    h = H2(tree, lists, Xt, cfg.kernel, cfg.ell, cfg.shift, cfg.h2_tol, n_proxy, active_nodes(tree, lists))
    ok = True
    for k in range(1, tree.L):
        nodes = list(tree.nodes_at(k))
        count = len(nodes)
        owner = [spd.shard_owner(world, count, a) for a in range(count)]
        sharded = owner[0] >= 0
        # every rank: compute its own nodes (all nodes on redundant levels)
        ranks = np.zeros(count, np.int64)
        local = {}
        for a, i in enumerate(nodes):
            if sharded and owner[a] != rank:
                continue
            if not h.active[i]:
                local[a] = (np.zeros(0, np.int64), np.zeros((0, 0)), 0)
                continue
            local[a] = _node_id(h, i, n_proxy)
            ranks[a] = local[a][2]
        if sharded:
            t = torch.tensor(ranks)
            dist.all_reduce(t)                        # owners' entries, the others 0
            ranks = t.numpy()
        # level arrays in node order at cumulative offsets (as the library packs them)
        ncand = [len(h.candidates(i)) if h.active[i] else 0 for i in nodes]
        e_off = np.concatenate([[0], np.cumsum([ncand[a] * ranks[a] for a in range(count)])]).astype(np.int64)
        s_off = np.concatenate([[0], np.cumsum(ranks)]).astype(np.int64)
        Eflat = torch.zeros(int(e_off[-1]), dtype=torch.float64)
        Sflat = torch.zeros(int(s_off[-1]), dtype=torch.int64)
        for a, (sk, E, s) in local.items():
            if s:
                Eflat[e_off[a]:e_off[a + 1]] = torch.tensor(E.T.reshape(-1))      # column-major
                Sflat[s_off[a]:s_off[a + 1]] = torch.tensor(sk)
        if sharded:
            per = count // world
            for qr in range(world):                   # owner qr broadcasts its contiguous range
                a0, a1 = qr * per, (qr + 1) * per
                for flat, off in ((Eflat, e_off), (Sflat, s_off)):
                    seg = flat[off[a0]:off[a1]].clone()
                    dist.broadcast(seg, src=qr)
                    flat[off[a0]:off[a1]] = seg
            # ownership is a partition of the level into contiguous equal ranges
            ok &= sorted(set(owner)) == list(range(world)) and all(owner[a] == a // per for a in range(count))
        for a, i in enumerate(nodes):
            s = int(ranks[a])
            h.rank[i] = s
            h.skel[i] = Sflat[s_off[a]:s_off[a + 1]].numpy().copy() if s else np.zeros(0, np.int64)
            if s:
                h.E[i] = Eflat[e_off[a]:e_off[a + 1]].numpy().reshape(s, ncand[a]).T.copy()
    ref = oracle.h2_build(X, cfg.kernel, cfg.ell, cfg.shift, cfg.leaf, cfg.h2_tol, n_proxy=n_proxy)
    for i, sk in ref.skel.items():
        ok &= np.array_equal(sk, h.skel.get(i, np.zeros(0, np.int64)))
        if len(sk):
            ok &= np.array_equal(ref.E[i], h.E[i])
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, bool(ok)))


def test_sharded_h2_protocol_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    assert res == [(0, True), (1, True)]


@pytest.mark.parametrize("P,count", [(1, 8), (2, 8), (4, 8), (8, 8), (8, 4), (4, 1024)])
def test_shard_owner_plan(P, count):
    sys.path.insert(0, ROOT)
    import paper_2011_07632_b200 as spd
    own = [spd.shard_owner(P, count, a) for a in range(count)]
    if P == 1 or count < P:
        assert own == [-1] * count                    # redundant level
    else:
        per = count // P
        assert own == [a // per for a in range(count)]   # subtree p = contiguous range p
