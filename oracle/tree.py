"""Partition tree, admissibility and interaction lists (oracle step O2).
TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §2 P:176-198 (nested index sets I_i, levels leaf=1 .. root=L,
perfect tree P:187), §5.1 P:657-663 (far-field sets F_i, "well separated"),
§5.2.2 P:891-913 (block types 1/2/3), with the DESIGN.md readings:

R1  binary KD tree of depth ceil(log2(N/leaf)); split dimension = argmax of
    the node's tight-bbox extent (ties -> lowest dimension); the node's points
    are sorted by (coordinate, original index); the left child takes the first
    ceil(n/2).  Nodes are numbered in heap order (root 0, children 2i+1, 2i+2).
R2  same-level nodes i != j are far iff for some d
        gap_d > 0 and gap_d >= max(ehat_i[d], ehat_j[d]),
    gap_d = max(lo_j[d]-hi_i[d], lo_i[d]-hi_j[d]), e = 0.5 (hi-lo),
    ehat[d] = max(e[d], 0.25 max_d' e[d']).
"""
from dataclasses import dataclass, field
import math
import numpy as np


@dataclass
class Tree:
    N: int
    d: int
    L: int                 # number of levels (root level L, leaf level 1)
    perm: np.ndarray       # tree position -> original point index
    begin: np.ndarray      # per node, range [begin, end) of tree positions
    end: np.ndarray
    lo: np.ndarray         # per node tight bbox
    hi: np.ndarray

    @property
    def nnodes(self):
        return len(self.begin)

    def level(self, i):
        depth = int(math.floor(math.log2(i + 1)))
        return self.L - depth

    def nodes_at(self, k):
        """lvl(k): heap ids of the nodes at level k."""
        depth = self.L - k
        return list(range(2 ** depth - 1, 2 ** (depth + 1) - 1))

    def children(self, i):
        if self.level(i) == 1:
            return []
        return [2 * i + 1, 2 * i + 2]

    def parent(self, i):
        return (i - 1) // 2 if i > 0 else -1

    def is_leaf(self, i):
        return self.level(i) == 1

    def size(self, i):
        return int(self.end[i] - self.begin[i])

    def lca_level(self, i, j):
        """Level of the lowest common ancestor of two same-level nodes."""
        lvl = self.level(i)
        while i != j:
            i, j = (i - 1) // 2, (j - 1) // 2
            lvl += 1
        return lvl


def tree_depth(N, leaf):
    if N <= leaf:
        return 0
    return int(math.ceil(math.log2(N / leaf)))


def build_tree(X, leaf):
    """KD median bisection (R1)."""
    X = np.asarray(X, dtype=np.float64)
    N, d = X.shape
    depth = tree_depth(N, leaf)
    L = depth + 1
    nn = 2 ** (depth + 1) - 1
    perm = np.arange(N, dtype=np.int64)
    begin = np.zeros(nn, np.int64)
    end = np.zeros(nn, np.int64)
    lo = np.zeros((nn, d))
    hi = np.zeros((nn, d))
    begin[0], end[0] = 0, N
    for i in range(nn):
        b, e = begin[i], end[i]
        idx = perm[b:e]
        pts = X[idx]
        lo[i] = pts.min(axis=0)
        hi[i] = pts.max(axis=0)
        if int(math.floor(math.log2(i + 1))) < depth:
            ext = hi[i] - lo[i]
            sd = int(np.argmax(ext))           # first maximum -> lowest dim
            order = np.lexsort((idx, pts[:, sd]))  # by coordinate, then index
            perm[b:e] = idx[order]
            mid = b + (e - b + 1) // 2         # left child takes ceil(n/2)
            begin[2 * i + 1], end[2 * i + 1] = b, mid
            begin[2 * i + 2], end[2 * i + 2] = mid, e
    return Tree(N, d, L, perm, begin, end, lo, hi)


def expand_dofs(tree: Tree, m: int) -> Tree:
    """Tree over m degrees of freedom per point (RPY, m = 3; reading R28): the point
    tree's nodes, boxes and levels, each tree position p becoming dofs m p .. m p + m-1,
    so dof tree position m p + c holds component c of point perm[p]."""
    if m == 1:
        return tree
    perm = (m * tree.perm[:, None] + np.arange(m)[None, :]).reshape(-1)
    return Tree(m * tree.N, tree.d, tree.L, perm, m * tree.begin, m * tree.end, tree.lo, tree.hi)


def far(tree: Tree, i, j):
    """Admissibility test R2 (symmetric by construction)."""
    if i == j:
        return False
    ei = 0.5 * (tree.hi[i] - tree.lo[i])
    ej = 0.5 * (tree.hi[j] - tree.lo[j])
    ehi = np.maximum(ei, 0.25 * ei.max())
    ehj = np.maximum(ej, 0.25 * ej.max())
    for dd in range(tree.d):
        gap = max(tree.lo[j][dd] - tree.hi[i][dd], tree.lo[i][dd] - tree.hi[j][dd])
        if gap > 0.0 and gap >= max(ehi[dd], ehj[dd]):
            return True
    return False


@dataclass
class Lists:
    near: list = field(default_factory=list)   # ordered near leaf pairs (a, b), a == b included
    type1: dict = field(default_factory=dict)  # level -> ordered near pairs (i, j), i != j
    type3: dict = field(default_factory=dict)  # level -> ordered far pairs whose parents are near
    lca: dict = field(default_factory=dict)    # (i, j) -> LCA level


def interaction_lists(tree: Tree) -> Lists:
    """Dual-tree traversal from (root, root).

    A visited pair (i, j) is Type-3 if far (its parents were near, otherwise
    it would not be visited); otherwise it is Type-1 (i != j) and recursion
    continues to all children pairs, ending in dense near leaf blocks.
    Type-2 pairs are never visited.
    """
    out = Lists()
    for k in range(1, tree.L + 1):
        out.type1[k] = []
        out.type3[k] = []
    stack = [(0, 0)]
    while stack:
        i, j = stack.pop()
        k = tree.level(i)
        if i != j and far(tree, i, j):
            out.type3[k].append((i, j))
            out.lca[(i, j)] = tree.lca_level(i, j)
            continue
        if i != j:
            out.type1[k].append((i, j))
        out.lca[(i, j)] = tree.lca_level(i, j)
        if k == 1:
            out.near.append((i, j))
        else:
            for ci in tree.children(i):
                for cj in tree.children(j):
                    stack.append((ci, cj))
    out.near.sort()
    for k in out.type1:
        out.type1[k].sort()
        out.type3[k].sort()
    return out
