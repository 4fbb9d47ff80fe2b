// tree.hpp -- cluster tree and interaction lists (host metadata of libspdhss).
//
// R1: binary KD tree, depth = smallest D with leaf * 2^D >= N,
//    split dimension = argmax tight-bbox extent (lowest dim on ties), points
//    of a node sorted by (coordinate, original index), left child = ceil(n/2).
//    Heap numbering: root 0, children 2i+1, 2i+2; level = L - depth (leaf 1).
// R2: same-level i != j far iff some d has gap_d > 0 and
//    gap_d >= max(ehat_i[d], ehat_j[d]); ehat = max(e, 0.25 max e), e = (hi-lo)/2.
// Lists from the dual-tree traversal of (root, root) (PAPER.md P:676-677,
// P:891-913): Type-3 = far pairs with near parents; Type-1 = near pairs
// i != j; near leaf pairs (incl. i == j) are the dense blocks.
#pragma once
#include <cstdint>
#include <utility>
#include <vector>

namespace spd {

struct TreeH {
    int64_t N = 0;
    int d = 0, L = 1, depth = 0, nnodes = 1;
    std::vector<int64_t> perm, begin, end;
    std::vector<double> lo, hi;          // nnodes * d
    int level(int i) const;
    int first(int k) const { return (1 << (L - k)) - 1; }
    int count(int k) const { return 1 << (L - k); }
    bool leaf(int i) const { return level(i) == 1; }
    int64_t size(int i) const { return end[i] - begin[i]; }
    int lca_level(int i, int j) const;
};

using Pair = std::pair<int, int>;
struct ListsH {
    std::vector<Pair> near;                       // sorted ordered near leaf pairs
    std::vector<std::vector<Pair>> type1, type3;  // [level] sorted ordered pairs
};

// pts: host, N x d row-major, original order
void build_tree(const double* pts, int64_t N, int d, int leaf, TreeH& t);
bool is_far(const TreeH& t, int i, int j);
void build_lists(const TreeH& t, ListsH& l);
#ifdef __CUDACC__
// device builders (tree_dev.cu): pts = DEVICE N x d row-major; same
// result as build_tree / build_lists.  build_tree_device returns false (nothing built)
// when a last-level node exceeds the shared-memory sort (leaf > 2048): use the host one.
bool build_tree_device(const double* pts, int64_t N, int d, int leaf, TreeH& t, cudaStream_t s);
void build_lists_device(const TreeH& t, ListsH& l, cudaStream_t s);
#endif

}  // namespace spd
