// tree.cpp -- KD tree (R1) and dual-tree interaction lists (R2); see tree.hpp.
// Integer work and exact comparisons only (no FMA-sensitive arithmetic), so the
// result is reproducible bit for bit.
#include "tree.hpp"
#include <algorithm>
#include <cmath>
#include <numeric>
#include <thread>

namespace spd {

static int floor_log2(int64_t x) { int r = 0; while (x >>= 1) ++r; return r; }

int TreeH::level(int i) const { return L - floor_log2((int64_t)i + 1); }

int TreeH::lca_level(int i, int j) const {
    int lv = level(i);
    while (i != j) { i = (i - 1) / 2; j = (j - 1) / 2; ++lv; }
    return lv;
}

// run fn(i) for i in [b, e) on up to hardware_concurrency threads (independent items)
template <class F>
static void parallel_for(int b, int e, int64_t work, F&& fn) {
    const int nt = (int)std::min<int64_t>({(int64_t)std::max(1u, std::thread::hardware_concurrency()), (int64_t)(e - b),
                                           std::max<int64_t>(1, work / 4096)});
    if (nt <= 1) { for (int i = b; i < e; ++i) fn(i); return; }
    std::vector<std::thread> th;
    for (int q = 0; q < nt; ++q)
        th.emplace_back([&, q] { for (int i = b + q; i < e; i += nt) fn(i); });
    for (auto& x : th) x.join();
}

void build_tree(const double* pts, int64_t N, int d, int leaf, TreeH& t) {
    t.N = N;
    t.d = d;
    int depth = 0;
    while ((int64_t)leaf << depth < N) ++depth;
    t.depth = depth;
    t.L = depth + 1;
    t.nnodes = (1 << (depth + 1)) - 1;
    t.perm.resize(N);
    std::iota(t.perm.begin(), t.perm.end(), (int64_t)0);
    t.begin.assign(t.nnodes, 0);
    t.end.assign(t.nnodes, 0);
    t.lo.assign((size_t)t.nnodes * d, 0.0);
    t.hi.assign((size_t)t.nnodes * d, 0.0);
    t.begin[0] = 0;
    t.end[0] = N;
    // level by level (the nodes of a level are independent); a node's split only needs
    // the SET of its ceil(n/2) smallest points by (coordinate, index), so nth_element
    // suffices except at the last split level, whose full sort fixes the order of the
    // points inside each leaf -- the permutation is bit-identical to sorting everywhere
    for (int dl = 0; dl <= depth; ++dl) {
        const int first = (1 << dl) - 1, count = 1 << dl;
        parallel_for(first, first + count, N, [&](int i) {
            const int64_t b = t.begin[i], e = t.end[i];
            for (int a = 0; a < d; ++a) {
                double lo = INFINITY, hi = -INFINITY;
                for (int64_t p = b; p < e; ++p) {
                    double x = pts[t.perm[p] * d + a];
                    lo = std::min(lo, x);
                    hi = std::max(hi, x);
                }
                t.lo[(size_t)i * d + a] = lo;
                t.hi[(size_t)i * d + a] = hi;
            }
            if (dl < depth) {
                int sd = 0;
                double best = t.hi[(size_t)i * d] - t.lo[(size_t)i * d];
                for (int a = 1; a < d; ++a) {
                    double ext = t.hi[(size_t)i * d + a] - t.lo[(size_t)i * d + a];
                    if (ext > best) { best = ext; sd = a; }
                }
                auto less = [&](int64_t x, int64_t y) {
                    double cx = pts[x * d + sd], cy = pts[y * d + sd];
                    return cx < cy || (cx == cy && x < y);
                };
                const int64_t mid = b + (e - b + 1) / 2;
                if (dl == depth - 1) std::sort(t.perm.begin() + b, t.perm.begin() + e, less);
                else if (mid < e) std::nth_element(t.perm.begin() + b, t.perm.begin() + mid, t.perm.begin() + e, less);
                t.begin[2 * i + 1] = b; t.end[2 * i + 1] = mid;
                t.begin[2 * i + 2] = mid; t.end[2 * i + 2] = e;
            }
        });
    }
}

bool is_far(const TreeH& t, int i, int j) {
    if (i == j) return false;
    const int d = t.d;
    double emax_i = 0.0, emax_j = 0.0;
    double ei[3], ej[3];
    for (int a = 0; a < d; ++a) {
        ei[a] = 0.5 * (t.hi[(size_t)i * d + a] - t.lo[(size_t)i * d + a]);
        ej[a] = 0.5 * (t.hi[(size_t)j * d + a] - t.lo[(size_t)j * d + a]);
        emax_i = std::max(emax_i, ei[a]);
        emax_j = std::max(emax_j, ej[a]);
    }
    for (int a = 0; a < d; ++a) {
        double ehi = std::max(ei[a], 0.25 * emax_i);
        double ehj = std::max(ej[a], 0.25 * emax_j);
        double gap = std::max(t.lo[(size_t)j * d + a] - t.hi[(size_t)i * d + a],
                              t.lo[(size_t)i * d + a] - t.hi[(size_t)j * d + a]);
        if (gap > 0.0 && gap >= std::max(ehi, ehj)) return true;
    }
    return false;
}

void build_lists(const TreeH& t, ListsH& l) {
    l.near.clear();
    l.type1.assign(t.L + 1, {});
    l.type3.assign(t.L + 1, {});
    // breadth-first until there are enough independent pairs, then the subtree
    // traversals in parallel; every list is sorted at the end, so the visiting order
    // does not matter (bit-identical lists)
    struct Out { std::vector<Pair> near; std::vector<std::vector<Pair>> t1, t3; };
    auto visit = [&](std::vector<Pair> stack, Out& o, size_t stop_at) {
        std::vector<Pair> frontier;
        while (!stack.empty()) {
            auto [i, j] = stack.back();
            stack.pop_back();
            const int k = t.level(i);
            if (i != j && is_far(t, i, j)) { o.t3[k].push_back({i, j}); continue; }
            if (i != j) o.t1[k].push_back({i, j});
            if (k == 1) { o.near.push_back({i, j}); continue; }
            for (int ci = 2 * i + 1; ci <= 2 * i + 2; ++ci)
                for (int cj = 2 * j + 1; cj <= 2 * j + 2; ++cj) {
                    if (stop_at && k - 1 <= (int)stop_at) frontier.push_back({ci, cj});
                    else stack.push_back({ci, cj});
                }
        }
        return frontier;
    };
    Out top{{}, std::vector<std::vector<Pair>>(t.L + 1), std::vector<std::vector<Pair>>(t.L + 1)};
    // pairs below level split_k are handed to the threads
    const int split_k = std::max(1, t.L - 4);
    std::vector<Pair> frontier = t.L > 5 ? visit({{0, 0}}, top, (size_t)split_k) : std::vector<Pair>{};
    if (t.L <= 5) visit({{0, 0}}, top, 0);
    const int nt = (int)std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(), frontier.size()));
    std::vector<Out> outs(nt, Out{{}, std::vector<std::vector<Pair>>(t.L + 1), std::vector<std::vector<Pair>>(t.L + 1)});
    {
        std::vector<std::thread> th;
        for (int q = 0; q < nt; ++q)
            th.emplace_back([&, q] {
                std::vector<Pair> st;
                for (size_t f = q; f < frontier.size(); f += nt) st.push_back(frontier[f]);
                visit(std::move(st), outs[q], 0);
            });
        for (auto& x : th) x.join();
    }
    outs.push_back(std::move(top));
    for (auto& o : outs) {
        l.near.insert(l.near.end(), o.near.begin(), o.near.end());
        for (int k = 0; k <= t.L; ++k) {
            l.type1[k].insert(l.type1[k].end(), o.t1[k].begin(), o.t1[k].end());
            l.type3[k].insert(l.type3[k].end(), o.t3[k].begin(), o.t3[k].end());
        }
    }
    std::sort(l.near.begin(), l.near.end());
    for (int k = 0; k <= t.L; ++k) {
        std::sort(l.type1[k].begin(), l.type1[k].end());
        std::sort(l.type3[k].begin(), l.type3[k].end());
    }
}

}  // namespace spd
