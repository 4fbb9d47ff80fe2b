// hsolve.cu -- single-vector HSS solve (the PCG preconditioner, k = 1), fused per level.
//
// The recursive solve of reading R12 ("ULV-style"):
//   H^{-1} = S^{-T} [ (I - V V^T) + V (I + H_2)^{-1} V^T ] S^{-1},  recursively,
// ending in (I + B_root)^{-1} = F_root^{-T} F_root^{-1}.  With P = S^{-T} V (the
// build's Phi^T; F^{-T} Vbar' above the leaves) the per-node work splits into two
// products that do not depend on each other:
//   up:    u0 = S^{-1} w,  zh = V^T S^{-1} w = P^T w
//   down:  x  = S^{-T} (u0 - V zh + V xh) = S^{-T} u0 + P (xh - zh)
// so each level is ONE launch with ONE round of independent loads per CTA (one CTA
// per node, 16 warps; F^{-1} is read as a lower triangle), 2L launches per solve.
// Summation order is fixed (no atomics): partial sums per (32-row tile, 32-column
// chunk) are reduced in chunk order.
#include "hss.hpp"
#include "phases.cuh"
#include "comm.hpp"
#include <algorithm>

namespace spd {

__global__ void __launch_bounds__(PH_T) hss_item_kernel(const HsNode* __restrict__ nodes,
                                                       const HsItem* __restrict__ items) {
    extern __shared__ double sm[];
    hss_item(nodes, items[blockIdx.x], sm);
}

__global__ void __launch_bounds__(256, 2) hss_item_warp_kernel(const HsNode* __restrict__ nodes,
                                                            const HsItem* __restrict__ items, int n) {
    const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (w < n) hss_item_warp(nodes, items[w]);
}

static void launch_phase(cudaStream_t s, const HsPhase& ph) {
    if (ph.items.empty()) return;
    int mmax = 1, rmax = 1;
    double by = 0;
    for (auto& n : ph.nodes) {
        mmax = std::max(mmax, n.m);
        rmax = std::max(rmax, n.r);
        by += ph.mode == 3 ? 8.0 * ((double)n.m * n.m + 2.0 * n.m)
                           : 8.0 * (0.5 * n.m * (n.m + 1) + (double)n.m * n.r + 2.0 * n.m + 2.0 * n.r);
    }
    SPD_REQUIRE(ph.mode == 3 || mmax <= 32 * HS_MT, "hss_solve: node too large for the k=1 solve");
    const size_t smem = sizeof(double) * (size_t)hss_item_smem_doubles(mmax, rmax);
    if (smem > 48 * 1024)
        SPD_CUDA(cudaFuncSetAttribute(hss_item_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DevArray<HsNode> dn(s, ph.nodes);
    DevArray<HsItem> di(s, ph.items);
    ProfScope prof(s, "hss_solve_vec", 0, by);
    static int nsm = 0;
    if (!nsm) {
        int dv = 0;
        SPD_CUDA(cudaGetDevice(&dv));
        SPD_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dv));
    }
    if (!hss_phase_uses_warps(ph.mode, ph.items.size(), nsm) || getenv("SPD_HSS_CTA")) {
        hss_item_kernel<<<(unsigned)ph.items.size(), PH_T, smem, s>>>(dn.p, di.p);
    } else {
        const int n = (int)ph.items.size();
        hss_item_warp_kernel<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(dn.p, di.p, n);
    }
    SPD_LAUNCH();
}

// The levels of one single-vector solve in execution order: up 1..L-1 (MODE 0),
// root (MODE 2), down L-1..1 (MODE 1).  zl[l]: level-l coefficients (zh up, xh down),
// zs[l]: zh kept for the down sweep, ub[l]: u0 of the level-l nodes at their
// children's offsets (leaves: u0 in z).
std::vector<HsPhase> hss_solve_plan(const spd_hss_s* H, const double* b, double* x, double* z,
                                    const std::vector<double*>& zl, const std::vector<double*>& zs,
                                    const std::vector<double*>& ub) {
    const spd_h2_s* h = H->h2;
    const TreeH& t = h->tree;
    const int L = t.L;
    const HssLevel& l1 = H->lv[1];
    std::vector<HsPhase> out;
    auto up_items = [](HsPhase& ph) {
        for (int q = 0; q < (int)ph.nodes.size(); ++q) {
            for (int rt = 0; rt * 32 < ph.nodes[q].m; ++rt) ph.items.push_back({q, 0, rt});
            for (int ct = 0; ct * 32 < ph.nodes[q].r; ++ct) ph.items.push_back({q, 1, ct});
        }
    };
    auto down_items = [](HsPhase& ph) {
        for (int q = 0; q < (int)ph.nodes.size(); ++q)
            for (int rt = 0; rt * 32 < ph.nodes[q].m; ++rt) ph.items.push_back({q, 2, rt});
    };
    HsPhase ph;
    ph.mode = 0;
    ph.level = 1;
    for (int a = 0; a < l1.count; ++a) {
        const int64_t off = t.begin[l1.first + a];
        if (!l1.m[a]) continue;
        ph.nodes.push_back({l1.Finv.p + l1.F_off[a], l1.P.p + l1.V_off[a], l1.m[a], l1.rank[a], b + off, nullptr,
                            nullptr, z + off, zl[1] + l1.off[a], zs[1] + l1.off[a], nullptr});
        ph.idx.push_back(a);
    }
    up_items(ph);
    out.push_back(ph);
    // dense top operator (spdhss.cu build_top_operator): up to level gt, one GEMV, down
    const int gt = H->gt_level;
    const int top_up = gt > 0 ? gt : L - 1;
    for (int l = 2; l <= top_up; ++l) {
        const HssLevel& lv = H->lv[l];
        const HssLevel& pv = H->lv[l - 1];
        ph = HsPhase();
        ph.level = l;
        for (int a = 0; a < lv.count; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            if (!lv.m[a]) continue;
            ph.nodes.push_back({lv.Finv.p + lv.F_off[a], lv.P.p + lv.V_off[a], lv.m[a], lv.rank[a],
                                zl[l - 1] + pv.off[c1], nullptr, nullptr, ub[l] + pv.off[c1], zl[l] + lv.off[a],
                                zs[l] + lv.off[a], nullptr});
            ph.idx.push_back(a);
        }
        up_items(ph);
        out.push_back(ph);
    }
    if (gt > 0) {
        ph = HsPhase();
        ph.mode = 3;
        const int R = (int)H->gt_R;
        ph.nodes.push_back({H->Gtop.p, nullptr, R, 0, zl[gt], nullptr, nullptr, nullptr, nullptr, nullptr,
                            H->gt_out.p});
        for (int rt = 0; rt * 32 < R; ++rt) ph.items.push_back({0, 3, rt});
        out.push_back(ph);
    } else {   // root: u = F w into ub[L], then x = F^T u back into zl[L-1]
        const HssLevel& rt = H->lv[L];
        if (rt.m[0]) {
            ph = HsPhase();
            ph.mode = 2;
            ph.nodes.push_back({rt.Finv.p, nullptr, rt.m[0], 0, zl[L - 1], nullptr, nullptr, ub[L], nullptr, nullptr,
                                nullptr});
            up_items(ph);
            out.push_back(ph);
            ph = HsPhase();
            ph.mode = 2;
            ph.nodes.push_back({rt.Finv.p, nullptr, rt.m[0], 0, ub[L], nullptr, nullptr, nullptr, nullptr, nullptr,
                                zl[L - 1]});
            down_items(ph);
            out.push_back(ph);
        }
    }
    // xh of level l: from the top operator at l = gt, else written into zl[l] by the level above
    auto xh_of = [&](int l) { return l == gt ? H->gt_out.p : zl[l]; };
    for (int l = (gt > 0 ? gt : L - 1); l >= 2; --l) {
        const HssLevel& lv = H->lv[l];
        const HssLevel& pv = H->lv[l - 1];
        ph = HsPhase();
        ph.mode = 1;
        ph.level = l;
        for (int a = 0; a < lv.count; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            if (!lv.m[a]) continue;
            ph.nodes.push_back({lv.Finv.p + lv.F_off[a], lv.P.p + lv.V_off[a], lv.m[a], lv.rank[a],
                                ub[l] + pv.off[c1], xh_of(l) + lv.off[a], zs[l] + lv.off[a], nullptr, nullptr, nullptr,
                                zl[l - 1] + pv.off[c1]});
            ph.idx.push_back(a);
        }
        down_items(ph);
        out.push_back(ph);
    }
    ph = HsPhase();
    ph.mode = 1;
    ph.level = 1;
    for (int a = 0; a < l1.count; ++a) {
        const int64_t off = t.begin[l1.first + a];
        if (!l1.m[a]) continue;
        ph.nodes.push_back({l1.Finv.p + l1.F_off[a], l1.P.p + l1.V_off[a], l1.m[a], l1.rank[a], z + off,
                            xh_of(1) + l1.off[a], zs[1] + l1.off[a], nullptr, nullptr, nullptr, x + off});
        ph.idx.push_back(a);
    }
    down_items(ph);
    out.push_back(ph);
    return out;
}

// Block-Jacobi preconditioner (the paper's BJ baseline): x_i =
// A_ii^{-1} b_i = S_i^{-T} S_i^{-1} b_i with the leaf Cholesky factors of the SPD-HSS
// build -- its diagonal blocks without the off-diagonal approximation.  Two phases:
// u0 = S^{-1} b (kind 0), x = S^{-T} u0 (kind 2 without coarse term).
std::vector<HsPhase> bj_solve_plan(const spd_hss_s* H, const double* b, double* x, double* z) {
    const spd_h2_s* h = H->h2;
    const TreeH& t = h->tree;
    const HssLevel& l1 = H->lv[1];
    std::vector<HsPhase> out(2);
    out[0].mode = 0;
    out[1].mode = 1;
    for (int a = 0; a < l1.count; ++a) {
        const int64_t off = t.begin[l1.first + a];
        const int m = l1.m[a];
        if (!m) continue;
        const double* F = l1.Finv.p + l1.F_off[a];
        out[0].nodes.push_back({F, nullptr, m, 0, b + off, nullptr, nullptr, z + off, nullptr, nullptr, nullptr});
        out[1].nodes.push_back({F, nullptr, m, 0, z + off, nullptr, nullptr, nullptr, nullptr, nullptr, x + off});
    }
    for (int q = 0; q < (int)out[0].nodes.size(); ++q)
        for (int rt = 0; rt * 32 < out[0].nodes[q].m; ++rt) {
            out[0].items.push_back({q, 0, rt});
            out[1].items.push_back({q, 2, rt});
        }
    return out;
}

void bj_solve_vec(spd_hss_s* H, const double* b, double* x, double* z, cudaStream_t s) {
    for (const auto& ph : bj_solve_plan(H, b, x, z)) launch_phase(s, ph);
}

// Subtree-sharded solve (real communicator of P ranks): at every level
// with >= P nodes a rank runs the up and down work of its own subtree's nodes only
// (shard_owner, the builds' plan); after the up sweep of the highest sharded level the
// owners' coarse coefficients zh of that level are exchanged (the split-level exchange:
// sum of its ranks, ~P r doubles), the levels above, the root / top operator run
// redundantly on every rank, the down sweep again only over owned nodes, and finally the
// owners' rows of x are exchanged so every rank holds the whole solution (N doubles).
static void hss_solve_sharded(spd_hss_s* H, std::vector<HsPhase> plan, double* x, const std::vector<double*>& zl,
                              cudaStream_t s) {
    const spd_comm_s* c = H->h2->comm;
    const TreeH& t = H->h2->tree;
    const int P = c->nranks;
    auto sharded = [&](int level) { return level >= 1 && H->lv[level].count >= P; };
    int le = 0;                                       // highest sharded level of the up sweep
    for (const auto& ph : plan)
        if (ph.mode == 0 && ph.level > 0 && sharded(ph.level)) le = std::max(le, ph.level);
    for (auto& ph : plan) {
        if ((ph.mode == 0 || ph.mode == 1) && ph.level > 0 && sharded(ph.level)) {
            const int cnt = H->lv[ph.level].count;
            HsPhase f;
            f.mode = ph.mode;
            f.level = ph.level;
            std::vector<int> remap(ph.nodes.size(), -1);
            for (size_t q = 0; q < ph.nodes.size(); ++q)
                if (shard_owner(c, cnt, ph.idx[q]) == c->rank) {
                    remap[q] = (int)f.nodes.size();
                    f.nodes.push_back(ph.nodes[q]);
                    f.idx.push_back(ph.idx[q]);
                }
            for (const auto& it : ph.items)
                if (remap[it.node] >= 0) f.items.push_back({remap[it.node], it.kind, it.tile});
            launch_phase(s, f);
        } else {
            launch_phase(s, ph);
        }
        if (ph.mode == 0 && ph.level == le && le > 0) {   // split-level exchange of zh
            const HssLevel& lv = H->lv[le];
            std::vector<int64_t> bq(P), eq(P);
            const int per = lv.count / P;
            for (int q = 0; q < P; ++q) { bq[q] = lv.off[q * per]; eq[q] = lv.off[std::min(lv.count, (q + 1) * per)]; }
            comm_bcast_ranges(c, zl[le], sizeof(double), bq, eq, s);
        }
    }
    // the owners' rows of x (their leaves are contiguous in tree order)
    const HssLevel& l1 = H->lv[1];
    const int per = l1.count / P;
    std::vector<int64_t> rb(P), re(P);
    for (int q = 0; q < P; ++q) {
        rb[q] = t.begin[l1.first + q * per];
        re[q] = t.end[l1.first + std::min(l1.count, (q + 1) * per) - 1];
    }
    comm_bcast_ranges(c, x, sizeof(double), rb, re, s);
}

void hss_solve_vec(spd_hss_s* H, const double* b, double* x, double* z, const std::vector<double*>& zl,
                   const std::vector<double*>& zs, const std::vector<double*>& ub, cudaStream_t s) {
    const spd_comm_s* c = H->h2->comm;
    if (comm_real(c) && H->lv[1].count >= c->nranks && !getenv("SPD_SOLVE_REPLICATED")) {
        hss_solve_sharded(H, hss_solve_plan(H, b, x, z, zl, zs, ub), x, zl, s);
        return;
    }
    for (const auto& ph : hss_solve_plan(H, b, x, z, zl, zs, ub)) launch_phase(s, ph);
}

}  // namespace spd
