// spdhss.cu -- Alg. 4 of PAPER.md (alg:spdhss_h2) on the device.
//
// Step map (P:line -> here):
//  P:1009  Y^(k) = (A - blockdiag_k A) Omega, k = 1..L-1 ........ lca_bucketed_products()
//          (one LCA-bucketed H2 product: Z^(c) = sum of blocks with LCA level c,
//           Y^(k) = sum_{c>k} Z^(c); equal to the L-1 masked products in exact arithmetic)
//  P:1014  A_ii = S_i S_i^T ........................................ potrf_batched
//  P:1016  Lambda = S_i^{-1} Y_i^(1) ................................. trsm_batched
//  P:1018  V_i by pivoted QR (Alg. 2 step 3, R4) ..................... qrcp_batched + formq
//  P:1020  Phi_i U_i^{H2} = V^T S^{-1} U^{H2}  (stored transposed)
//  P:1022  Type-1 B_ij = V_i^T S_i^{-1} A_ij S_j^{-T} V_j  (A_ij on the fly, kblock; R10)
//  P:1024  Type-3 B_ij = (Phi U)_i K(J_i, J_j) (Phi U)_j^T  (on the fly, kblock)
//  P:1031  (I + B_ii)^{+-1/2}: Cholesky F F^T = I + B_ii instead (reading R9:
//          R_i, B_ij, Phi identical; Vbar rotates by Q^T)
//  P:1033  Alg. 3 sketch F^{-1} [T_c1; T_c2], with T_i^(k') = P_i^T [T_c] kept for
//          every pending level k' (P_i = F_i^{-T} Vbar'_i, so Phi_i = P_i^T blockdiag(Phi_c))
//  P:1039  Vbar_i by pivoted QR
//  P:1041  (Phi U)_i^T = E_i^T blockdiag((Phi U)_c^T) P_i
//  P:1049  Type-1 B_ij = P_i^T bold(B_ij) P_j
//  P:1051  Type-3 B_ij as above
//  P:1053  R_i = F_i Vbar'_i   (= (I+B)^{1/2} Vbar_i)
//  root    F_root = chol(I + B_root) for the solve (reading R11)
#include "hss.hpp"
#include "comm.hpp"
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <cstdlib>

namespace spd {

static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ================================================================= Omega: Philox4x32-10 + Box-Muller
__device__ __forceinline__ void philox_round(uint32_t c[4], const uint32_t k[2]) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0, h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
    const uint32_t n0 = h1 ^ c[1] ^ k[0], n2 = h0 ^ c[3] ^ k[1];
    c[0] = n0; c[1] = l1; c[2] = n2; c[3] = l0;
}
__global__ void philox_normal_kernel(double* out, int64_t n, int w, uint64_t seed) {
    const int64_t total = n * w;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c[4] = {(uint32_t)e, (uint32_t)(e >> 32), 0x5350u, 0x48u};
        uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
        for (int r = 0; r < 10; ++r) {
            philox_round(c, k);
            k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u;
        }
        const double u1 = ((((uint64_t)c[0] << 21) ^ c[1]) & ((1ull << 53) - 1)) * 0x1p-53 + 0x1p-54;
        const double u2 = ((((uint64_t)c[2] << 21) ^ c[3]) & ((1ull << 53) - 1)) * 0x1p-53;
        out[e] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
}

void philox_normal(cudaStream_t s, double* out, int64_t n, int w, uint64_t seed) {
    if (n == 0 || w == 0) return;
    philox_normal_kernel<<<148 * 8, 256, 0, s>>>(out, n, w, seed);
    SPD_LAUNCH();
}

// ================================================================= dense kernel blocks A_ii
struct DenseKDesc { const double* x; int64_t ds; int n; int64_t id0; double* A; int ld; };
__global__ void dense_kernel_blocks(const DenseKDesc* descs, KernelParams kp, double shift, int d) {
    const DenseKDesc dk = descs[blockIdx.y];
    const int64_t total = (int64_t)dk.n * dk.n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(e % dk.n), j = (int)(e / dk.n);
        double v = kernel_entry(kp, dk.x + i, dk.ds, dk.x + j, dk.ds, d);
        if (i == j) v += shift;
        dk.A[i + (size_t)j * dk.ld] = v;
    }
}
static void dense_blocks(cudaStream_t s, const std::vector<DenseKDesc>& d, const KernelParams& kp, double shift, int dim) {
    if (d.empty()) return;
    DevArray<DenseKDesc> dd(s, d);
    ProfScope prof(s, "dense_blocks", 0, 0);
    for (size_t off = 0; off < d.size(); off += 65535) {
        unsigned ny = (unsigned)std::min<size_t>(65535, d.size() - off);
        dense_kernel_blocks<<<dim3(16, ny), 256, 0, s>>>(dd.p + off, kp, shift, dim);
        SPD_LAUNCH();
    }
}

__global__ void axpy_kernel(double* y, const double* x, int64_t n, double a) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        y[e] += a * x[e];
}
static void axpy(cudaStream_t s, double* y, const double* x, int64_t n, double a) {
    if (n <= 0) return;
    axpy_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(y, x, n, a);
    SPD_LAUNCH();
}

static void check_info(cudaStream_t s, const DBuf<int>& info, const DBuf<double>& bad, int level, int first,
                       const char* what) {
    std::vector<int> inf = info.download(s);
    for (size_t a = 0; a < inf.size(); ++a)
        if (inf[a] != 0) {
            std::vector<double> bv = bad.download(s);
            char msg[256];
            snprintf(msg, sizeof msg, "%s not positive definite at level %d node %d (pivot %d, value %.3e)",
                     what, level, first + (int)a, inf[a] - 1, bv[a]);
            throw Error(SPD_ENOTPD, msg);
        }
}

// ================================================================= subtree sharding
// With a real communicator (NCCL or host-staged; comm.cpp) of P ranks, at every level
// with >= P nodes rank p computes only the per-node work of its subtree (shard_owner,
// the H2 build's plan): Y^(k) rows of its leaves, factorisations, QRCP and bases of its
// nodes, the B_ij of pairs whose first node it owns.  Level arrays start zeroed and are
// all-reduced (summed) once their owners have written them, so every rank ends with the
// full HSS (the solve and PCG run replicated).  Levels with fewer nodes run redundantly.
struct HssShard {
    const spd_comm_s* c = nullptr;
    bool real = false;
    bool on(int count) const { return real && count >= c->nranks; }
    std::vector<char> own(int count) const {
        std::vector<char> o(count, 1);
        if (on(count))
            for (int a = 0; a < count; ++a) o[a] = shard_owner(c, count, a) == c->rank;
        return o;
    }
    void zero(DBuf<double>& b, int count, cudaStream_t s) const { if (on(count)) b.zero(s); }
    void sum(DBuf<double>& b, int64_t n, int count, cudaStream_t s) const {
        if (on(count) && n > 0) comm_allreduce_sum(c, b.p, (size_t)n, s);
    }
    void sum(DBuf<int>& b, int64_t n, int count, cudaStream_t s) const {
        if (on(count) && n > 0) comm_allreduce_sum(c, b.p, (size_t)n, s);
    }
};

// ================================================================= Y^(k) by LCA buckets
// sharded: near and coupling targets restricted to the owned nodes, so exactly the Y
// rows of the owned leaves are complete (the only rows this rank reads)
static void lca_bucketed_products(spd_hss_s* H, const double* om, DBuf<double>& Y, const HssShard& sh,
                                  cudaStream_t s) {
    spd_h2_s* h = H->h2;
    const TreeH& t = h->tree;
    const int L = t.L, w = H->w;
    const int64_t N = h->N;
    const bool stored = h2_store_for_products(h, s, false);     // kernel blocks from the symmetric store
    Y.alloc((size_t)(L - 1) * N * w);
    Y.zero(s);
    auto slice = [&](int c) { return Y.p + (size_t)(c - 2) * N * w; };   // bucket c = 2..L
    // --- near field: K_ab Omega_b into bucket lca(a, b), a != b
    {
        const int l1 = t.first(1), nl = t.count(1);
        std::vector<KbBlock> blocks;
        for (int a = 0; a < nl; ++a) blocks.push_back({h->X.p + t.begin[l1 + a], N, (int)t.size(l1 + a), t.begin[l1 + a]});
        std::vector<KbTarget> targets;
        std::vector<KbEntry> entries;
        size_t e = 0;
        const auto& near = h->lists.near;
        const std::vector<char> own = sh.own(nl);
        while (e < near.size()) {
            const int i = near[e].first;
            if (!own[i - l1]) { ++e; continue; }
            std::vector<std::pair<int, int>> js;       // (lca, j)
            while (e < near.size() && near[e].first == i) {
                if (near[e].second != i) js.push_back({t.lca_level(i, near[e].second), near[e].second});
                ++e;
            }
            std::stable_sort(js.begin(), js.end(), [](auto& x, auto& y) { return x.first < y.first; });
            KbTarget tg{i - l1, (int)entries.size(), 0};
            for (auto& [c, j] : js) {
                entries.push_back({j - l1, om + t.begin[j], (int)N, slice(c) + t.begin[i], (int)N, w});
                if (stored) h2_use_store(h, 0, i - l1, j - l1, (int)t.size(i), (int)t.size(j), entries.back());
            }
            tg.e_end = (int)entries.size();
            targets.push_back(tg);
        }
        kblock_apply(s, h->kp, 0.0, h->d, blocks, targets, entries);
    }
    // --- far field: up pass once, coupling into per-bucket coefficients, one down pass per bucket
    std::vector<DBuf<double>> xh(L);
    std::vector<double*> xhp(L, nullptr);
    for (int l = 1; l < L; ++l) { xh[l].alloc(std::max<int64_t>(1, h->lv[l].Sw * w)); xhp[l] = xh[l].p; }
    h2_up(h, om, N, w, xhp, L - 1, s);
    // bucket c holds coefficients for levels 1..c-1
    std::vector<std::vector<DBuf<double>>> yb(L + 1);
    std::vector<std::vector<double*>> ybp(L + 1);
    std::vector<char> used(L + 1, 0);
    for (int l = 1; l < L; ++l)
        for (auto& pr : h->lists.type3[l]) used[t.lca_level(pr.first, pr.second)] = 1;
    for (int c = 2; c <= L; ++c) {
        if (!used[c]) continue;
        yb[c].resize(c);
        ybp[c].assign(L, nullptr);
        for (int l = 1; l < c; ++l) {
            yb[c][l].alloc(std::max<int64_t>(1, h->lv[l].Sw * w));
            yb[c][l].zero(s);
            ybp[c][l] = yb[c][l].p;
        }
    }
    for (int l = 1; l < L; ++l) {
        const H2Level& lv = h->lv[l];
        const auto& T3 = h->lists.type3[l];
        if (T3.empty()) continue;
        std::vector<KbBlock> blocks;
        for (int a = 0; a < lv.count; ++a) blocks.push_back({lv.skelX.p + lv.off[a], lv.S, lv.rank[a], -1});
        std::vector<KbTarget> targets;
        std::vector<KbEntry> entries;
        const std::vector<char> own = sh.own(lv.count);
        size_t e = 0;
        while (e < T3.size()) {
            const int i = T3[e].first, a = i - lv.first;
            if (!own[a]) { ++e; continue; }
            std::vector<std::pair<int, int>> js;
            while (e < T3.size() && T3[e].first == i) { js.push_back({t.lca_level(i, T3[e].second), T3[e].second}); ++e; }
            std::stable_sort(js.begin(), js.end(), [](auto& x, auto& y) { return x.first < y.first; });
            KbTarget tg{a, (int)entries.size(), 0};
            for (auto& [c, j] : js) {
                const int b = j - lv.first;
                if (lv.rank[a] && lv.rank[b]) {
                    entries.push_back({b, xhp[l] + lv.off[b], (int)lv.Sw, ybp[c][l] + lv.off[a], (int)lv.Sw, w});
                    if (stored) h2_use_store(h, l, a, b, lv.rank[a], lv.rank[b], entries.back());
                }
            }
            tg.e_end = (int)entries.size();
            targets.push_back(tg);
        }
        kblock_apply(s, h->kp, 0.0, h->d, blocks, targets, entries);
    }
    for (int c = 2; c <= L; ++c)
        if (used[c]) h2_down(h, ybp[c], c - 1, slice(c), N, w, s);
    // Y^(k) = sum_{c > k} Z^(c): suffix sums over the slices (slice index k-1 becomes Y^(k))
    for (int c = L - 1; c >= 2; --c) axpy(s, slice(c), slice(c + 1), N * w, 1.0);
    H->sketch_groups = L - 1;
}

// ================================================================= helpers for B assembly
static const double* find_B(const HssLevel& lv, int i, int j, bool& trans) {
    auto key = pair_key(std::min(i, j), std::max(i, j));
    auto it = lv.B_off.find(key);
    if (it == lv.B_off.end()) throw Error(SPD_ECUDA, "internal: missing B for pair");
    trans = i > j;
    return lv.B.p + it->second;
}

// G_ij = K(P_i, P_j) X_j for a list of (i, j) pairs, then B_ij = Left_i^T G_ij
struct PairProd { int i, j; };
static void kernel_sandwich(spd_hss_s* H, cudaStream_t s, const std::vector<PairProd>& pairs,
                            const std::vector<KbBlock>& blocks, int first,
                            const std::vector<const double*>& X, const std::vector<int>& ldX,
                            const std::vector<const double*>& Left, const std::vector<int>& ldLeft,
                            const std::vector<int>& rank, HssLevel& dst, int slot) {
    if (pairs.empty()) return;
    spd_h2_s* h = H->h2;
    const bool stored = h2_store_for_products(h, s, false);     // slot: 0 leaf points, l level-l skeletons
    std::vector<int64_t> goff(pairs.size() + 1, 0);
    for (size_t q = 0; q < pairs.size(); ++q)
        goff[q + 1] = goff[q] + (int64_t)blocks[pairs[q].i - first].n * rank[pairs[q].j - first];
    DBuf<double> G(std::max<int64_t>(1, goff.back()));
    G.zero(s);
    std::vector<KbTarget> targets;
    std::vector<KbEntry> entries;
    size_t q = 0;
    while (q < pairs.size()) {
        const int i = pairs[q].i;
        KbTarget tg{i - first, (int)entries.size(), 0};
        while (q < pairs.size() && pairs[q].i == i) {
            const int j = pairs[q].j;
            const int ni = blocks[i - first].n;
            if (rank[j - first] > 0 && ni > 0 && blocks[j - first].n > 0) {
                entries.push_back({j - first, X[j - first], ldX[j - first], G.p + goff[q], ni, rank[j - first]});
                if (stored)
                    h2_use_store(h, slot, i - first, j - first, ni, blocks[j - first].n, entries.back());
            }
            ++q;
        }
        tg.e_end = (int)entries.size();
        targets.push_back(tg);
    }
    kblock_apply(s, h->kp, 0.0, h->d, blocks, targets, entries);
    std::vector<GemmDesc> gd;
    for (size_t p = 0; p < pairs.size(); ++p) {
        const int i = pairs[p].i, j = pairs[p].j;
        const int ri = rank[i - first], rj = rank[j - first];
        double* Bp = dst.B.p + dst.B_off.at(pair_key(i, j));
        GemmDesc g{Left[i - first], G.p + goff[p], Bp, ri, rj, blocks[i - first].n, ldLeft[i - first],
                   blocks[i - first].n, std::max(1, ri)};
        gd.push_back(g);
    }
    gemm_batched(s, gd, true, false, 1.0, 0.0);
}

static void alloc_B(HssLevel& lv, const std::vector<Pair>& t1, const std::vector<Pair>& t3, int first) {
    int64_t off = 0;
    lv.B_off.clear();
    for (const auto* L : {&t1, &t3})
        for (auto& pr : *L)
            if (pr.first < pr.second) {
                lv.B_off[pair_key(pr.first, pr.second)] = off;
                off += (int64_t)lv.rank[pr.first - first] * lv.rank[pr.second - first];
            }
    lv.B.alloc(std::max<int64_t>(1, off));
}

// QRCP of the per-node sketches; ranks to host; explicit V (m x r)
static void sketch_qr(spd_hss_s* H, cudaStream_t s, HssLevel& lv, const std::vector<double*>& A,
                      const std::vector<int>& ldA, const HssShard& sh) {
    const int n = lv.count, w = H->w;
    const std::vector<char> own = sh.own(n);
    DBuf<int> piv((size_t)n * w), rank(n);
    DBuf<double> beta((size_t)n * w), norms((size_t)n * w);
    if (sh.on(n)) { piv.zero(s); rank.zero(s); }
    for (int a = 0; a < n; ++a) H->shard_work[0] += own[a];
    H->shard_work[1] += n;
    std::vector<QrcpDesc> qd;
    for (int a = 0; a < n; ++a)
        if (own[a]) qd.push_back({A[a], lv.m[a], w, ldA[a], std::min(H->cap, std::min(lv.m[a], w)), piv.p + (size_t)a * w,
                      beta.p + (size_t)a * w, rank.p + a, norms.p + (size_t)a * w});
    qrcp_batched(s, qd, H->tol);
    sh.sum(rank, n, n, s);
    sh.sum(piv, (int64_t)n * w, n, s);
    lv.rank = rank.download(s);
    lv.piv = piv.download(s);
    lv.off.assign(n + 1, 0);
    lv.V_off.assign(n + 1, 0);
    for (int a = 0; a < n; ++a) {
        lv.off[a + 1] = lv.off[a] + lv.rank[a];
        lv.V_off[a + 1] = lv.V_off[a] + (int64_t)lv.m[a] * lv.rank[a];
    }
    lv.R = lv.off[n];
    lv.V.alloc(std::max<int64_t>(1, lv.V_off[n]));
    sh.zero(lv.V, n, s);
    std::vector<FormQDesc> fq;
    for (int a = 0; a < n; ++a)
        if (own[a]) fq.push_back({A[a], beta.p + (size_t)a * w, rank.p + a, lv.V.p + lv.V_off[a], lv.m[a], w, ldA[a],
                      std::max(1, lv.m[a])});
    formq_batched(s, fq);
    // P = F^{-T} V  (leaf: Phi^T = S^{-T} V)
    lv.P.alloc(std::max<int64_t>(1, lv.V_off[n]));
    SPD_CUDA(cudaMemcpyAsync(lv.P.p, lv.V.p, sizeof(double) * lv.V_off[n], cudaMemcpyDeviceToDevice, s));
    std::vector<TrsmDesc> td;
    for (int a = 0; a < n; ++a)
        if (own[a])
            td.push_back({lv.F.p + lv.F_off[a], lv.P.p + lv.V_off[a], lv.m[a], lv.rank[a], std::max(1, lv.m[a]),
                          std::max(1, lv.m[a])});
    trsm_batched(s, td, 'L', true);
    sh.sum(lv.V, lv.V_off[n], n, s);                  // bases of every node, for the B_ij of cross pairs
    sh.sum(lv.P, lv.V_off[n], n, s);
}

// ================================================================= solve factors
__global__ void set_identity_kernel(const MatDesc* descs) {
    const MatDesc d = descs[blockIdx.y];
    const int64_t total = (int64_t)d.m * d.n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(e % d.m), j = (int)(e / d.m);
        d.A[i + (size_t)j * d.ld] = (i == j) ? 1.0 : 0.0;
    }
}
static void invert_factors(cudaStream_t s, HssLevel& lv, const HssShard& sh) {
    const int n = lv.count;
    if (n == 0 || lv.F_off.empty()) return;
    lv.Finv.alloc(std::max<int64_t>(1, lv.F_off[n]));
    sh.zero(lv.Finv, n, s);
    const std::vector<char> own = sh.own(n);
    std::vector<MatDesc> md;
    std::vector<TrsmDesc> td;
    for (int a = 0; a < n; ++a) {
        const int m = lv.m[a];
        if (!m || !own[a]) continue;
        md.push_back({lv.Finv.p + lv.F_off[a], m, m, m});
        td.push_back({lv.F.p + lv.F_off[a], lv.Finv.p + lv.F_off[a], m, m, m, m});
    }
    if (!md.empty()) {
        DevArray<MatDesc> dm(s, md);
        for (size_t off = 0; off < md.size(); off += 65535) {
            set_identity_kernel<<<dim3(8, (unsigned)std::min<size_t>(65535, md.size() - off)), 256, 0, s>>>(dm.p + off);
            SPD_LAUNCH();
        }
        trsm_batched(s, td, 'L', false);              // F^{-1} = F \ I (lower triangular)
    }
    sh.sum(lv.Finv, lv.F_off[n], n, s);
}

// ================================================================= dense top of the solve
// The part of the recursive solve (R12) above level t -- up levels t+1..L-1, the root
// factor, down levels L-1..t+1 -- is a linear map of the level-t coefficients zh_t
// onto xh_t.  For the smallest t whose coefficient space R_t is at most 3072 it is
// formed once, densely, by running that part of the recursion on the identity
// (multi-column GEMMs), so the single-vector solve applies it as one GEMV.
static void solve_middle(spd_hss_s* H, int t, int k, const std::vector<double*>& zz, const std::vector<double*>& uu,
                         cudaStream_t s) {
    const int L = H->h2->tree.L;
    for (int l = t + 1; l < L; ++l) {
        const HssLevel& lv = H->lv[l];
        const HssLevel& pv = H->lv[l - 1];
        std::vector<GemmDesc> g0, g1, g2;
        for (int a = 0; a < lv.count; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            const int m = lv.m[a];
            if (!m) continue;
            double* u = uu[l] + pv.off[c1];
            g0.push_back({lv.Finv.p + lv.F_off[a], zz[l - 1] + pv.off[c1], u, m, k, m, m, (int)pv.R, (int)pv.R});
            if (lv.rank[a]) {
                g1.push_back({lv.V.p + lv.V_off[a], u, zz[l] + lv.off[a], lv.rank[a], k, m, m, (int)pv.R, (int)lv.R});
                g2.push_back({lv.V.p + lv.V_off[a], zz[l] + lv.off[a], u, m, k, lv.rank[a], m, (int)lv.R, (int)pv.R});
            }
        }
        gemm_batched(s, g0, false, false, 1.0, 0.0);
        gemm_batched(s, g1, true, false, 1.0, 0.0);
        gemm_batched(s, g2, false, false, -1.0, 1.0);
    }
    {
        const HssLevel& rt = H->lv[L];
        const HssLevel& pv = H->lv[L - 1];
        const int m = rt.m[0];
        if (m) {
            gemm_batched(s, {{rt.Finv.p, zz[L - 1], uu[L], m, k, m, m, (int)pv.R, (int)pv.R}}, false, false, 1.0, 0.0);
            gemm_batched(s, {{rt.Finv.p, uu[L], zz[L - 1], m, k, m, m, (int)pv.R, (int)pv.R}}, true, false, 1.0, 0.0);
        }
    }
    for (int l = L - 1; l > t; --l) {
        const HssLevel& lv = H->lv[l];
        const HssLevel& pv = H->lv[l - 1];
        std::vector<GemmDesc> g, g3;
        for (int a = 0; a < lv.count; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            const int m = lv.m[a];
            if (!m) continue;
            double* u = uu[l] + pv.off[c1];
            if (lv.rank[a])
                g.push_back({lv.V.p + lv.V_off[a], zz[l] + lv.off[a], u, m, k, lv.rank[a], m, (int)lv.R, (int)pv.R});
            g3.push_back({lv.Finv.p + lv.F_off[a], u, zz[l - 1] + pv.off[c1], m, k, m, m, (int)pv.R, (int)pv.R});
        }
        gemm_batched(s, g, false, false, 1.0, 1.0);
        gemm_batched(s, g3, true, false, 1.0, 0.0);
    }
}

__global__ void identity_kernel(double* A, int64_t n) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x)
        A[e] = (e % n == e / n) ? 1.0 : 0.0;
}

static void build_top_operator(spd_hss_s* H, cudaStream_t s) {
    const int L = H->h2->tree.L;
    H->gt_level = 0;
    if (L < 2 || getenv("SPD_NO_GTOP")) return;
    // largest dense top operator: one GEMV over R_t x R_t replaces 2 (L - t) latency-bound
    // solve phases; SPD_GTOP_MAX overrides (measured: 3072 vs 4096 at C2 in DESIGN.md)
    const int64_t gt_max = getenv("SPD_GTOP_MAX") ? atoll(getenv("SPD_GTOP_MAX")) : 3072;
    int t = 0;
    for (int l = 1; l < L; ++l)
        if (H->lv[l].R <= gt_max) { t = l; break; }
    if (t == 0 || H->lv[t].R == 0) return;
    const int64_t R = H->lv[t].R;
    const int k = (int)R;
    std::vector<DBuf<double>> zb(L), ubuf(L + 1);
    std::vector<double*> zz(L, nullptr), uu(L + 1, nullptr);
    H->Gtop.alloc((size_t)R * R);
    zz[t] = H->Gtop.p;
    for (int l = t + 1; l < L; ++l) { zb[l].alloc(std::max<int64_t>(1, H->lv[l].R * k)); zz[l] = zb[l].p; }
    for (int l = t + 1; l <= L; ++l) { ubuf[l].alloc(std::max<int64_t>(1, H->lv[l - 1].R * k)); uu[l] = ubuf[l].p; }
    identity_kernel<<<148 * 4, 256, 0, s>>>(H->Gtop.p, R);
    SPD_LAUNCH();
    solve_middle(H, t, k, zz, uu, s);
    H->gt_out.alloc(R);
    H->gt_level = t;
    H->gt_R = R;
}

// ================================================================= the build
void hss_build_impl(spd_hss_s* H, const double* omega_in, uint64_t seed, cudaStream_t s) {
    spd_h2_s* h = H->h2;
    const TreeH& t = h->tree;
    const int L = t.L, w = H->w, d = h->d;
    const int64_t N = h->N;
    const double t0 = now_s();
    const HssShard sh{h->comm, comm_real(h->comm)};
    H->shard_work[0] = H->shard_work[1] = 0;
    H->lv.clear();
    H->lv.resize(L + 1);
    if (L == 1) {                                   // single node: the HSS is the dense block
        HssLevel& r = H->lv[1];
        r.k = 1; r.first = 0; r.count = 1;
        r.m = {(int)N}; r.rank = {0}; r.off = {0, 0}; r.F_off = {0, N * N};
        r.F.alloc((size_t)N * N);
        dense_blocks(s, {{h->X.p, N, (int)N, 0, r.F.p, (int)N}}, h->kp, h->kern.shift, d);
        DBuf<int> info(1); DBuf<double> bad(1); info.zero(s);
        potrf_batched(s, {{r.F.p, (int)N, (int)N, (int)N}}, info.p, bad.p);
        check_info(s, info, bad, 1, 0, "leaf block A_ii");
        invert_factors(s, r, HssShard{});
        return;
    }
    // ---------------- Omega (parity hook or Philox)
    DBuf<double> Om;
    const double* om = omega_in;
    if (!om) {
        Om.alloc((size_t)N * w);
        philox_normal_kernel<<<148 * 8, 256, 0, s>>>(Om.p, N, w, seed);
        SPD_LAUNCH();
        om = Om.p;
    }
    // ---------------- P:1009  all Y^(k)
    DBuf<double> Y;
    stage_mark(s, nullptr);
    lca_bucketed_products(H, om, Y, sh, s);
    auto Yk = [&](int k) { return Y.p + (size_t)(k - 1) * N * w; };
    SPD_CUDA(cudaStreamSynchronize(s));
    const double t1 = now_s();
    H->timings[0] = t1 - t0;
    stage_mark(s, "hss Y products");

    // ---------------- leaf level
    HssLevel& l1 = H->lv[1];
    l1.k = 1; l1.first = t.first(1); l1.count = t.count(1);
    const int nl = l1.count;
    l1.m.resize(nl);
    l1.F_off.assign(nl + 1, 0);
    for (int a = 0; a < nl; ++a) {
        l1.m[a] = (int)t.size(l1.first + a);
        l1.F_off[a + 1] = l1.F_off[a] + (int64_t)l1.m[a] * l1.m[a];
    }
    l1.F.alloc(l1.F_off[nl]);
    sh.zero(l1.F, nl, s);
    const std::vector<char> own1 = sh.own(nl);
    {
        std::vector<DenseKDesc> dk;
        std::vector<MatDesc> md;
        for (int a = 0; a < nl; ++a) {
            if (!own1[a]) continue;
            const int i = l1.first + a;
            dk.push_back({h->X.p + t.begin[i], N, l1.m[a], t.begin[i], l1.F.p + l1.F_off[a], l1.m[a]});
            md.push_back({l1.F.p + l1.F_off[a], l1.m[a], l1.m[a], l1.m[a]});
        }
        dense_blocks(s, dk, h->kp, h->kern.shift, d);               // A_ii = K + sigma I
        DBuf<int> info(nl); DBuf<double> bad(nl); info.zero(s);
        potrf_batched(s, md, info.p, bad.p);                        // A_ii = S_i S_i^T
        check_info(s, info, bad, 1, l1.first, "leaf block A_ii");
        stage_mark(s, "hss leaf potrf");
    }
    {
        std::vector<TrsmDesc> td;                                   // Lambda = S^{-1} Y^(1)_i (in place)
        for (int a = 0; a < nl; ++a)
            if (own1[a])
                td.push_back({l1.F.p + l1.F_off[a], Yk(1) + t.begin[l1.first + a], l1.m[a], w, l1.m[a], (int)N});
        trsm_batched(s, td, 'L', false);
        std::vector<double*> A(nl);
        std::vector<int> ldA(nl, (int)N);
        for (int a = 0; a < nl; ++a) A[a] = Yk(1) + t.begin[l1.first + a];
        sketch_qr(H, s, l1, A, ldA, sh);                               // V_i, rank, Phi^T = S^{-T} V
        stage_mark(s, "hss leaf sketch qr");
    }
    // (Phi U)^T = E^T Phi^T for active leaves
    const H2Level& h1 = h->lv[1];
    auto alloc_PU = [&](HssLevel& lv, const H2Level& hl) {
        lv.PU_off.assign(lv.count + 1, 0);
        for (int a = 0; a < lv.count; ++a) lv.PU_off[a + 1] = lv.PU_off[a] + (int64_t)hl.rank[a] * lv.rank[a];
        lv.PU.alloc(std::max<int64_t>(1, lv.PU_off[lv.count]));
    };
    alloc_PU(l1, h1);
    sh.zero(l1.PU, nl, s);
    {
        std::vector<GemmDesc> gd;
        for (int a = 0; a < nl; ++a)
            if (own1[a] && h1.rank[a] && l1.rank[a])
                gd.push_back({h1.E.p + h1.E_off[a], l1.P.p + l1.V_off[a], l1.PU.p + l1.PU_off[a], h1.rank[a],
                              l1.rank[a], l1.m[a], h1.ncand[a], l1.m[a], h1.rank[a]});
        gemm_batched(s, gd, true, false, 1.0, 0.0);
    }
    sh.sum(l1.PU, l1.PU_off[nl], nl, s);
    // the last sharded level hands its pending sketches to the redundant level above
    auto handoff = [&](int k) { return sh.on(t.count(k)) && k + 1 <= L && !sh.on(t.count(k + 1)); };
    // pending sketches T^(k') = Phi_i Y_i^(k'), k' = 2..L-1  (Alg. 3 step 1)
    std::vector<DBuf<double>> Tprev(L), Tcur(L);
    for (int kp2 = 2; kp2 < L; ++kp2) {
        Tprev[kp2].alloc(std::max<int64_t>(1, l1.R * w));
        if (handoff(1)) Tprev[kp2].zero(s);
        std::vector<GemmDesc> gd;
        for (int a = 0; a < nl; ++a)
            if (own1[a] && l1.rank[a])
                gd.push_back({l1.P.p + l1.V_off[a], Yk(kp2) + t.begin[l1.first + a], Tprev[kp2].p + l1.off[a],
                              l1.rank[a], w, l1.m[a], l1.m[a], (int)N, (int)std::max<int64_t>(1, l1.R)});
        gemm_batched(s, gd, true, false, 1.0, 0.0);
        if (handoff(1)) sh.sum(Tprev[kp2], l1.R * w, nl, s);
    }
    // leaf B_ij: Type-1 (near, on the fly) and Type-3 (skeletons, on the fly)
    {
        alloc_B(l1, h->lists.type1[1], h->lists.type3[1], l1.first);
        sh.zero(l1.B, nl, s);
        stage_mark(s, "hss leaf PU/T/allocB");
        std::vector<KbBlock> blocks;
        std::vector<const double*> X, Left;
        std::vector<int> ldX, ldLeft;
        for (int a = 0; a < nl; ++a) {
            const int i = l1.first + a;
            blocks.push_back({h->X.p + t.begin[i], N, l1.m[a], t.begin[i]});
            X.push_back(l1.P.p + l1.V_off[a]); ldX.push_back(std::max(1, l1.m[a]));
            Left.push_back(l1.P.p + l1.V_off[a]); ldLeft.push_back(std::max(1, l1.m[a]));
        }
        std::vector<PairProd> pairs;                                // B_ij by the owner of i (i < j)
        for (auto& pr : h->lists.type1[1])
            if (pr.first < pr.second && own1[pr.first - l1.first]) pairs.push_back({pr.first, pr.second});
        kernel_sandwich(H, s, pairs, blocks, l1.first, X, ldX, Left, ldLeft, l1.rank, l1, 0);
        stage_mark(s, "hss leaf B type1");
        blocks.clear(); X.clear(); ldX.clear(); Left.clear(); ldLeft.clear();
        for (int a = 0; a < nl; ++a) {
            blocks.push_back({h1.skelX.p + h1.off[a], h1.S, h1.rank[a], -1});
            X.push_back(l1.PU.p + l1.PU_off[a]); ldX.push_back(std::max(1, h1.rank[a]));
            Left.push_back(l1.PU.p + l1.PU_off[a]); ldLeft.push_back(std::max(1, h1.rank[a]));
        }
        pairs.clear();
        for (auto& pr : h->lists.type3[1])
            if (pr.first < pr.second && own1[pr.first - l1.first]) pairs.push_back({pr.first, pr.second});
        kernel_sandwich(H, s, pairs, blocks, l1.first, X, ldX, Left, ldLeft, l1.rank, l1, 1);
        sh.sum(l1.B, l1.B.n, nl, s);
        sh.sum(l1.F, l1.F_off[nl], nl, s);
    }
    SPD_CUDA(cudaStreamSynchronize(s));
    const double t2 = now_s();
    H->timings[1] = t2 - t1;
    stage_mark(s, "hss leaf level");

    // ---------------- levels k = 2..L (k = L: root factor only)
    for (int k = 2; k <= L; ++k) {
        HssLevel& lv = H->lv[k];
        const HssLevel& pv = H->lv[k - 1];
        lv.k = k; lv.first = t.first(k); lv.count = t.count(k);
        const int n = lv.count;
        lv.m.resize(n);
        lv.F_off.assign(n + 1, 0);
        std::vector<int> r1(n);
        for (int a = 0; a < n; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            r1[a] = pv.rank[c1];
            lv.m[a] = pv.rank[c1] + pv.rank[c1 + 1];
            lv.F_off[a + 1] = lv.F_off[a] + (int64_t)lv.m[a] * lv.m[a];
        }
        lv.F.alloc(std::max<int64_t>(1, lv.F_off[n]));
        lv.F.zero(s);
        const std::vector<char> own = sh.own(n);
        {   // I + B_ii (lower part: B_c2c1 = B_c1c2^T), then Cholesky
            std::vector<CopyDesc> cd;
            std::vector<MatDesc> md;
            for (int a = 0; a < n; ++a) {
                if (!own[a]) continue;
                const int i = lv.first + a, c1 = 2 * i + 1, c2 = 2 * i + 2;
                const int m = lv.m[a];
                if (r1[a] > 0 && m - r1[a] > 0) {
                    bool tr;
                    const double* B = find_B(pv, c1, c2, tr);
                    cd.push_back({B, lv.F.p + lv.F_off[a] + r1[a], m - r1[a], r1[a], std::max(1, r1[a]), m, 1});
                }
                md.push_back({lv.F.p + lv.F_off[a], m, m, std::max(1, m)});
            }
            copy_batched(s, cd, 1.0, false);
            set_identity_plus(s, md);
            DBuf<int> info(n); DBuf<double> bad(n); info.zero(s);
            potrf_batched(s, md, info.p, bad.p);
            check_info(s, info, bad, k, lv.first, "I + B_ii");
            sh.sum(lv.F, lv.F_off[n], n, s);
            stage_mark(s, "hss lvl potrf");
        }
        if (k == L) break;
        // Alg. 3 sketch: Lambda_i = F^{-1} [T_c1; T_c2]^(k)
        std::vector<int64_t> lam_off(n + 1, 0);
        for (int a = 0; a < n; ++a) lam_off[a + 1] = lam_off[a] + (int64_t)lv.m[a] * w;
        DBuf<double> Lam(std::max<int64_t>(1, lam_off[n]));
        {
            std::vector<CopyDesc> cd;
            std::vector<TrsmDesc> td;
            for (int a = 0; a < n; ++a) {
                const int c1 = 2 * (lv.first + a) + 1 - pv.first;
                if (lv.m[a] == 0 || !own[a]) continue;
                cd.push_back({Tprev[k].p + pv.off[c1], Lam.p + lam_off[a], lv.m[a], w, (int)std::max<int64_t>(1, pv.R),
                              lv.m[a], 0});
                td.push_back({lv.F.p + lv.F_off[a], Lam.p + lam_off[a], lv.m[a], w, lv.m[a], lv.m[a]});
            }
            copy_batched(s, cd, 1.0, false);
            trsm_batched(s, td, 'L', false);
            std::vector<double*> A(n);
            std::vector<int> ldA(n);
            for (int a = 0; a < n; ++a) { A[a] = Lam.p + lam_off[a]; ldA[a] = std::max(1, lv.m[a]); }
            sketch_qr(H, s, lv, A, ldA, sh);                       // Vbar', P = F^{-T} Vbar'
            stage_mark(s, "hss lvl sketch qr");
        }
        // R_i = F_i Vbar'_i
        lv.Rt.alloc(std::max<int64_t>(1, lv.V_off[n]));
        sh.zero(lv.Rt, n, s);
        {
            std::vector<GemmDesc> gd;
            for (int a = 0; a < n; ++a)
                if (own[a] && lv.rank[a] && lv.m[a])
                    gd.push_back({lv.F.p + lv.F_off[a], lv.V.p + lv.V_off[a], lv.Rt.p + lv.V_off[a], lv.m[a], lv.rank[a],
                                  lv.m[a], lv.m[a], lv.m[a], lv.m[a]});
            gemm_batched(s, gd, false, false, 1.0, 0.0);
            sh.sum(lv.Rt, lv.V_off[n], n, s);
        }
        // (Phi U)_i^T = E_i^T blockdiag((Phi U)_c^T) P_i
        const H2Level& hk = h->lv[k];
        const H2Level& hp = h->lv[k - 1];
        alloc_PU(lv, hk);
        sh.zero(lv.PU, n, s);
        {
            std::vector<int64_t> woff(n + 1, 0);
            for (int a = 0; a < n; ++a) woff[a + 1] = woff[a] + (int64_t)hk.ncand[a] * lv.rank[a];
            DBuf<double> W(std::max<int64_t>(1, woff[n]));
            W.zero(s);
            std::vector<GemmDesc> g1, g2;
            for (int a = 0; a < n; ++a) {
                if (!own[a] || !hk.rank[a] || !lv.rank[a]) continue;
                const int c1 = 2 * (lv.first + a) + 1 - pv.first;
                const int sc1 = hp.rank[c1], sc2 = hp.rank[c1 + 1];
                const int nc = hk.ncand[a];
                if (sc1 && pv.rank[c1])
                    g1.push_back({pv.PU.p + pv.PU_off[c1], lv.P.p + lv.V_off[a], W.p + woff[a], sc1, lv.rank[a],
                                  pv.rank[c1], sc1, lv.m[a], nc});
                if (sc2 && pv.rank[c1 + 1])
                    g1.push_back({pv.PU.p + pv.PU_off[c1 + 1], lv.P.p + lv.V_off[a] + pv.rank[c1], W.p + woff[a] + sc1,
                                  sc2, lv.rank[a], pv.rank[c1 + 1], sc2, lv.m[a], nc});
                g2.push_back({hk.E.p + hk.E_off[a], W.p + woff[a], lv.PU.p + lv.PU_off[a], hk.rank[a], lv.rank[a], nc,
                              nc, nc, hk.rank[a]});
            }
            gemm_batched(s, g1, false, false, 1.0, 0.0);
            gemm_batched(s, g2, true, false, 1.0, 0.0);
        }
        sh.sum(lv.PU, lv.PU_off[n], n, s);
        // pending sketches for k' > k: T_i = P_i^T [T_c1; T_c2]
        for (int kp2 = k + 1; kp2 < L; ++kp2) {
            Tcur[kp2].alloc(std::max<int64_t>(1, lv.R * w));
            if (handoff(k)) Tcur[kp2].zero(s);
            std::vector<GemmDesc> gd;
            for (int a = 0; a < n; ++a) {
                if (!own[a] || !lv.rank[a]) continue;
                const int c1 = 2 * (lv.first + a) + 1 - pv.first;
                gd.push_back({lv.P.p + lv.V_off[a], Tprev[kp2].p + pv.off[c1], Tcur[kp2].p + lv.off[a], lv.rank[a], w,
                              lv.m[a], lv.m[a], (int)std::max<int64_t>(1, pv.R), (int)std::max<int64_t>(1, lv.R)});
            }
            gemm_batched(s, gd, true, false, 1.0, 0.0);
            if (handoff(k)) sh.sum(Tcur[kp2], lv.R * w, n, s);
        }
        // B_ij at level k
        alloc_B(lv, h->lists.type1[k], h->lists.type3[k], lv.first);
        sh.zero(lv.B, n, s);
        stage_mark(s, "hss lvl PU/T/allocB");
        {   // Type-1: B_ij = P_i^T bold(B_ij) P_j  (sharded: by the owner of i)
            std::vector<Pair> t1;
            for (auto& pr : h->lists.type1[k])
                if (pr.first < pr.second && own[pr.first - lv.first]) t1.push_back(pr);
            std::vector<int64_t> bo(t1.size() + 1, 0), go(t1.size() + 1, 0);
            for (size_t q = 0; q < t1.size(); ++q) {
                const int a = t1[q].first - lv.first, b = t1[q].second - lv.first;
                bo[q + 1] = bo[q] + (int64_t)lv.m[a] * lv.m[b];
                go[q + 1] = go[q] + (int64_t)lv.m[a] * lv.rank[b];
            }
            DBuf<double> BB(std::max<int64_t>(1, bo.back())), G(std::max<int64_t>(1, go.back()));
            BB.zero(s);
            std::vector<CopyDesc> cd;
            std::vector<GemmDesc> g1, g2;
            for (size_t q = 0; q < t1.size(); ++q) {
                const int i = t1[q].first, j = t1[q].second, a = i - lv.first, b = j - lv.first;
                const int mi = lv.m[a], mj = lv.m[b];
                int roff = 0;
                for (int ca = 2 * i + 1; ca <= 2 * i + 2; ++ca) {
                    const int ra = pv.rank[ca - pv.first];
                    int coff = 0;
                    for (int cb = 2 * j + 1; cb <= 2 * j + 2; ++cb) {
                        const int rb = pv.rank[cb - pv.first];
                        if (ra && rb) {
                            bool tr;
                            const double* Bp = find_B(pv, ca, cb, tr);
                            cd.push_back({Bp, BB.p + bo[q] + roff + (size_t)coff * mi, ra, rb, tr ? rb : ra, mi, tr ? 1 : 0});
                        }
                        coff += rb;
                    }
                    roff += ra;
                }
                if (lv.rank[a] && lv.rank[b] && mi && mj) {
                    g1.push_back({BB.p + bo[q], lv.P.p + lv.V_off[b], G.p + go[q], mi, lv.rank[b], mj, mi, mj, mi});
                    g2.push_back({lv.P.p + lv.V_off[a], G.p + go[q], lv.B.p + lv.B_off.at(pair_key(i, j)), lv.rank[a],
                                  lv.rank[b], mi, mi, mi, lv.rank[a]});
                }
            }
            copy_batched(s, cd, 1.0, false);
            gemm_batched(s, g1, false, false, 1.0, 0.0);
            gemm_batched(s, g2, true, false, 1.0, 0.0);
        }
        {   // Type-3: B_ij = (Phi U)_i K(J_i, J_j) (Phi U)_j^T
            std::vector<KbBlock> blocks;
            std::vector<const double*> X, Left;
            std::vector<int> ldX, ldLeft;
            for (int a = 0; a < n; ++a) {
                blocks.push_back({hk.skelX.p + hk.off[a], hk.S, hk.rank[a], -1});
                X.push_back(lv.PU.p + lv.PU_off[a]); ldX.push_back(std::max(1, hk.rank[a]));
                Left.push_back(lv.PU.p + lv.PU_off[a]); ldLeft.push_back(std::max(1, hk.rank[a]));
            }
            std::vector<PairProd> pairs;
            for (auto& pr : h->lists.type3[k])
                if (pr.first < pr.second && own[pr.first - lv.first]) pairs.push_back({pr.first, pr.second});
            kernel_sandwich(H, s, pairs, blocks, lv.first, X, ldX, Left, ldLeft, lv.rank, lv, k);
        }
        sh.sum(lv.B, lv.B.n, n, s);
        for (int kp2 = k + 1; kp2 < L; ++kp2) std::swap(Tprev[kp2], Tcur[kp2]);
        Tprev[k].release();
        SPD_CUDA(cudaStreamSynchronize(s));
        stage_mark(s, "hss level", k);
    }
    // solve factors: explicit S_i^{-1}, F_i^{-1} (triangular inverses by blocked TRSM on I),
    // so every step of hss_solve is an HBM-bound GEMV
    for (int k = 1; k <= L; ++k) invert_factors(s, H->lv[k], sh);
    build_top_operator(H, s);
    SPD_CUDA(cudaStreamSynchronize(s));
    stage_mark(s, "hss invert factors");
    H->timings[2] = now_s() - t2;
    H->timings[3] = now_s() - t0;
}

// ================================================================= forward product y = H x
// The HSS matrix of Alg. 4 in nested form (the representation hss_export
// writes): leaf D_i = S_i S_i^T (= A_ii), U_i = S_i V_i; nonleaf transfer R_i (Rt); sibling
// couplings B_{c1 c2}.  Up:  t_i = S_i^T x_i, xh_i = V_i^T t_i (leaf), xh_p = R_p^T [xh_c1; xh_c2];
// couple: yh_c1 += B xh_c2, yh_c2 += B^T xh_c1 (every parent, root included); down:
// [yh_c1; yh_c2] += R_p yh_p;  leaf: y_i = S_i (t_i + V_i yh_i).  Batched DMMA GEMMs per level.
void hss_apply_tree(spd_hss_s* H, const double* x, int64_t ldx, double* y, int64_t ldy, int k, cudaStream_t s) {
    const spd_h2_s* h = H->h2;
    const TreeH& t = h->tree;
    const int L = t.L;
    const int64_t N = h->N;
    if (L == 1) {                                    // y = S (S^T x)
        const HssLevel& r = H->lv[1];
        DBuf<double> tt((size_t)N * k);
        gemm_batched(s, {{r.F.p, x, tt.p, (int)N, k, (int)N, (int)N, (int)ldx, (int)N}}, true, false, 1.0, 0.0);
        gemm_batched(s, {{r.F.p, tt.p, y, (int)N, k, (int)N, (int)N, (int)N, (int)ldy}}, false, false, 1.0, 0.0);
        return;
    }
    const HssLevel& l1 = H->lv[1];
    DBuf<double> tt((size_t)N * k);
    std::vector<DBuf<double>> xh(L), yh(L);
    for (int l = 1; l < L; ++l) {
        xh[l].alloc((size_t)std::max<int64_t>(1, H->lv[l].R) * k);
        yh[l].alloc((size_t)std::max<int64_t>(1, H->lv[l].R) * k);
        yh[l].zero(s);
    }
    {   // leaves: t = S^T x, xh = V^T t
        std::vector<GemmDesc> g1, g2;
        for (int a = 0; a < l1.count; ++a) {
            const int m = l1.m[a], r = l1.rank[a];
            if (!m) continue;
            const int64_t b0 = t.begin[l1.first + a];
            g1.push_back({l1.F.p + l1.F_off[a], x + b0, tt.p + b0, m, k, m, m, (int)ldx, (int)N});
            if (r) g2.push_back({l1.V.p + l1.V_off[a], tt.p + b0, xh[1].p + l1.off[a], r, k, m, m, (int)N, (int)l1.R});
        }
        gemm_batched(s, g1, true, false, 1.0, 0.0);
        gemm_batched(s, g2, true, false, 1.0, 0.0);
    }
    for (int l = 2; l < L; ++l) {                   // xh_p = R_p^T [xh_c1; xh_c2]
        const HssLevel& lv = H->lv[l];
        const HssLevel& pv = H->lv[l - 1];
        std::vector<GemmDesc> g;
        for (int a = 0; a < lv.count; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            if (!lv.rank[a] || !lv.m[a]) continue;
            g.push_back({lv.Rt.p + lv.V_off[a], xh[l - 1].p + pv.off[c1], xh[l].p + lv.off[a], lv.rank[a], k, lv.m[a],
                         lv.m[a], (int)pv.R, (int)lv.R});
        }
        gemm_batched(s, g, true, false, 1.0, 0.0);
    }
    {   // sibling couplings, all levels (children of every parent, root included)
        std::vector<GemmDesc> gf, gt;
        for (int l = 2; l <= L; ++l) {
            const HssLevel& cv = H->lv[l - 1];
            for (int p = t.first(l); p < t.first(l) + t.count(l); ++p) {
                const int c1 = 2 * p + 1, c2 = 2 * p + 2;
                const int a1 = c1 - cv.first, a2 = c2 - cv.first;
                const int r1 = cv.rank[a1], r2 = cv.rank[a2];
                if (!r1 || !r2) continue;
                bool tr;
                const double* B = find_B(cv, c1, c2, tr);
                gf.push_back({B, xh[l - 1].p + cv.off[a2], yh[l - 1].p + cv.off[a1], r1, k, r2, r1, (int)cv.R, (int)cv.R});
                gt.push_back({B, xh[l - 1].p + cv.off[a1], yh[l - 1].p + cv.off[a2], r2, k, r1, r1, (int)cv.R, (int)cv.R});
            }
        }
        gemm_batched(s, gf, false, false, 1.0, 1.0);
        gemm_batched(s, gt, true, false, 1.0, 1.0);
    }
    for (int l = L - 1; l >= 2; --l) {              // [yh_c1; yh_c2] += R_p yh_p
        const HssLevel& lv = H->lv[l];
        const HssLevel& pv = H->lv[l - 1];
        std::vector<GemmDesc> g;
        for (int a = 0; a < lv.count; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            if (!lv.rank[a] || !lv.m[a]) continue;
            g.push_back({lv.Rt.p + lv.V_off[a], yh[l].p + lv.off[a], yh[l - 1].p + pv.off[c1], lv.m[a], k, lv.rank[a],
                         lv.m[a], (int)lv.R, (int)pv.R});
        }
        gemm_batched(s, g, false, false, 1.0, 1.0);
    }
    {   // leaves: t += V yh ; y = S t
        std::vector<GemmDesc> g1, g2;
        for (int a = 0; a < l1.count; ++a) {
            const int m = l1.m[a], r = l1.rank[a];
            if (!m) continue;
            const int64_t b0 = t.begin[l1.first + a];
            if (r) g1.push_back({l1.V.p + l1.V_off[a], yh[1].p + l1.off[a], tt.p + b0, m, k, r, m, (int)l1.R, (int)N});
            g2.push_back({l1.F.p + l1.F_off[a], tt.p + b0, y + b0, m, k, m, m, (int)N, (int)ldy});
        }
        gemm_batched(s, g1, false, false, 1.0, 1.0);
        gemm_batched(s, g2, false, false, 1.0, 0.0);
    }
}

// ================================================================= recursive solve (R12)
static void ensure_solve_ws(spd_hss_s* H, int k) {
    if (H->ws_k >= k && !H->z.empty()) return;
    const int L = H->h2->tree.L;
    H->bt.alloc((size_t)H->h2->N * k);
    H->xt.alloc((size_t)H->h2->N * k);
    H->z.clear();
    H->z.resize(L + 1);
    for (int l = 1; l < L; ++l) H->z[l].alloc(std::max<int64_t>(1, H->lv[l].R * k));
    H->ub.clear();
    H->ub.resize(L + 1);
    for (int l = 2; l <= L; ++l) H->ub[l].alloc(std::max<int64_t>(1, H->lv[l - 1].R * k));
    H->zs.clear();
    H->zs.resize(L + 1);
    for (int l = 1; l < L; ++l) H->zs[l].alloc(std::max<int64_t>(1, H->lv[l].R));
    H->ws_k = k;
}

void hss_solve_tree(spd_hss_s* H, const double* b, int64_t ldb, double* x, int64_t ldx, int k, cudaStream_t s) {
    spd_h2_s* h = H->h2;
    const TreeH& t = h->tree;
    const int L = t.L;
    const int64_t N = h->N;
    if (L == 1) {
        const HssLevel& r = H->lv[1];
        ensure_solve_ws(H, k);
        gemm_batched(s, {{r.Finv.p, b, H->bt.p, (int)N, k, (int)N, (int)N, (int)ldb, (int)N}}, false, false, 1.0, 0.0);
        gemm_batched(s, {{r.Finv.p, H->bt.p, x, (int)N, k, (int)N, (int)N, (int)N, (int)ldx}}, true, false, 1.0, 0.0);
        return;
    }
    ensure_solve_ws(H, k);
    double* z = H->bt.p;                               // N x k workspace (ld N)
    if (k == 1 && !getenv("SPD_SOLVE_GEMV")) {         // fused per-level single-vector path (hsolve.cu)
        std::vector<double*> zl(L + 1, nullptr), zsl(L + 1, nullptr), ubl(L + 1, nullptr);
        for (int l = 1; l < L; ++l) { zl[l] = H->z[l].p; zsl[l] = H->zs[l].p; }
        for (int l = 2; l <= L; ++l) ubl[l] = H->ub[l].p;
        hss_solve_vec(H, b, x, z, zl, zsl, ubl, s);
        return;
    }
    const HssLevel& l1 = H->lv[1];
    // up, leaf: z = S^{-1} b ; zh = V^T z ; z <- z - V zh
    {
        std::vector<GemmDesc> g0, g1, g2;
        for (int a = 0; a < l1.count; ++a) {
            const int64_t off = t.begin[l1.first + a];
            const int n = l1.m[a];
            g0.push_back({l1.Finv.p + l1.F_off[a], b + off, z + off, n, k, n, n, (int)ldb, (int)N});
            if (l1.rank[a]) {
                g1.push_back({l1.V.p + l1.V_off[a], z + off, H->z[1].p + l1.off[a], l1.rank[a], k, n, n, (int)N, (int)l1.R});
                g2.push_back({l1.V.p + l1.V_off[a], H->z[1].p + l1.off[a], z + off, n, k, l1.rank[a], n, (int)l1.R, (int)N});
            }
        }
        gemm_batched(s, g0, false, false, 1.0, 0.0);
        gemm_batched(s, g1, true, false, 1.0, 0.0);
        gemm_batched(s, g2, false, false, -1.0, 1.0);
    }
    // up, levels 2..L-1: u = F^{-1} zh_children ; zh = Vbar^T u ; u <- u - Vbar zh   (u stored in ub[l])
    for (int l = 2; l < L; ++l) {
        const HssLevel& lv = H->lv[l];
        const HssLevel& pv = H->lv[l - 1];
        std::vector<GemmDesc> g0, g1, g2;
        for (int a = 0; a < lv.count; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            const int m = lv.m[a];
            if (!m) continue;
            double* u = H->ub[l].p + pv.off[c1];
            g0.push_back({lv.Finv.p + lv.F_off[a], H->z[l - 1].p + pv.off[c1], u, m, k, m, m, (int)pv.R, (int)pv.R});
            if (lv.rank[a]) {
                g1.push_back({lv.V.p + lv.V_off[a], u, H->z[l].p + lv.off[a], lv.rank[a], k, m, m, (int)pv.R, (int)lv.R});
                g2.push_back({lv.V.p + lv.V_off[a], H->z[l].p + lv.off[a], u, m, k, lv.rank[a], m, (int)lv.R, (int)pv.R});
            }
        }
        gemm_batched(s, g0, false, false, 1.0, 0.0);
        gemm_batched(s, g1, true, false, 1.0, 0.0);
        gemm_batched(s, g2, false, false, -1.0, 1.0);
    }
    // root: xh = F^{-T} F^{-1} zh_top   (into ub[L], then back into z[L-1])
    {
        const HssLevel& rt = H->lv[L];
        const HssLevel& pv = H->lv[L - 1];
        const int m = rt.m[0];
        if (m) {
            gemm_batched(s, {{rt.Finv.p, H->z[L - 1].p, H->ub[L].p, m, k, m, m, (int)pv.R, (int)pv.R}}, false, false, 1.0, 0.0);
            gemm_batched(s, {{rt.Finv.p, H->ub[L].p, H->z[L - 1].p, m, k, m, m, (int)pv.R, (int)pv.R}}, true, false, 1.0, 0.0);
        }
    }
    // down: children xh = F^{-T} (u + Vbar xh)
    for (int l = L - 1; l >= 2; --l) {
        const HssLevel& lv = H->lv[l];
        const HssLevel& pv = H->lv[l - 1];
        std::vector<GemmDesc> g, g3;
        for (int a = 0; a < lv.count; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            const int m = lv.m[a];
            if (!m) continue;
            double* u = H->ub[l].p + pv.off[c1];
            if (lv.rank[a])
                g.push_back({lv.V.p + lv.V_off[a], H->z[l].p + lv.off[a], u, m, k, lv.rank[a], m, (int)lv.R, (int)pv.R});
            g3.push_back({lv.Finv.p + lv.F_off[a], u, H->z[l - 1].p + pv.off[c1], m, k, m, m, (int)pv.R, (int)pv.R});
        }
        gemm_batched(s, g, false, false, 1.0, 1.0);
        gemm_batched(s, g3, true, false, 1.0, 0.0);
    }
    // leaf: x = S^{-T} (z + V xh)
    {
        std::vector<GemmDesc> g, g3;
        for (int a = 0; a < l1.count; ++a) {
            const int64_t off = t.begin[l1.first + a];
            const int n = l1.m[a];
            if (l1.rank[a])
                g.push_back({l1.V.p + l1.V_off[a], H->z[1].p + l1.off[a], z + off, n, k, l1.rank[a], n, (int)l1.R, (int)N});
            g3.push_back({l1.Finv.p + l1.F_off[a], z + off, x + off, n, k, n, n, (int)N, (int)ldx});
        }
        gemm_batched(s, g, false, false, 1.0, 1.0);
        gemm_batched(s, g3, true, false, 1.0, 0.0);
    }
}

// ================================================================= queries / export
const spd_hss_s* hss_if_hss(const void* h) {
    return *(const uint32_t*)h == 0x48535348u ? (const spd_hss_s*)h : nullptr;
}
const double* hss_timings(const spd_hss_s* H) { return H->timings; }
const int64_t* hss_shard_work(const spd_hss_s* H) { return H->shard_work; }

static std::vector<double> dl(const double* p, int64_t n) {
    std::vector<double> v(n);
    if (n) SPD_CUDA(cudaMemcpy(v.data(), p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    return v;
}

static std::vector<double> hss_export(const spd_hss_s* H) {
    const spd_h2_s* h = H->h2;
    const TreeH& t = h->tree;
    const int L = t.L;
    std::vector<double> out;
    if (L == 1) return out;
    const HssLevel& l1 = H->lv[1];
    const int64_t N = h->N;
    for (int a = 0; a < l1.count; ++a) {
        const int n = l1.m[a];
        std::vector<double> S = dl(l1.F.p + l1.F_off[a], (int64_t)n * n);
        std::vector<double> V = dl(l1.V.p + l1.V_off[a], (int64_t)n * l1.rank[a]);
        // D = S S^T (= A_ii), U = S V
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                double v = 0.0;
                for (int q = 0; q <= std::min(i, j); ++q) v += S[i + (size_t)q * n] * S[j + (size_t)q * n];
                out.push_back(v);
            }
        for (int j = 0; j < l1.rank[a]; ++j)
            for (int i = 0; i < n; ++i) {
                double v = 0.0;
                for (int q = 0; q <= i; ++q) v += S[i + (size_t)q * n] * V[q + (size_t)j * n];
                out.push_back(v);
            }
    }
    (void)N;
    for (int k = 2; k < L; ++k) {
        const HssLevel& lv = H->lv[k];
        std::vector<double> R = dl(lv.Rt.p, lv.V_off[lv.count]);
        out.insert(out.end(), R.begin(), R.end());
    }
    for (int p = 0; p < t.nnodes; ++p) {
        const int k = t.level(p);
        if (k < 2) continue;
        const HssLevel& cv = H->lv[k - 1];
        const int c1 = 2 * p + 1, c2 = 2 * p + 2;
        const int64_t n = (int64_t)cv.rank[c1 - cv.first] * cv.rank[c2 - cv.first];
        if (!n) continue;
        bool tr;
        const double* B = find_B(cv, c1, c2, tr);
        std::vector<double> v = dl(B, n);
        out.insert(out.end(), v.begin(), v.end());
    }
    return out;
}

void hss_query(const spd_hss_s* H, int what, void* buf, size_t bytes) {
    const TreeH& t = H->h2->tree;
    auto need = [&](size_t want) {
        if (bytes < want) throw Error(SPD_EINVAL, "spd_query: buffer too small (" + std::to_string(want) + " bytes)");
        return want;
    };
    switch (what) {
    case SPD_Q_HSS_RANKS: {
        std::vector<int32_t> v(t.nnodes, 0);
        for (int k = 1; k < t.L; ++k)
            for (int a = 0; a < H->lv[k].count; ++a) v[H->lv[k].first + a] = H->lv[k].rank[a];
        std::memcpy(buf, v.data(), need(4 * v.size()));
        break;
    }
    case SPD_Q_HSS_EXPORT_SIZE: {
        int64_t n = (int64_t)hss_export(H).size();
        std::memcpy(buf, &n, need(8));
        break;
    }
    case SPD_Q_HSS_EXPORT: {
        std::vector<double> v = hss_export(H);
        std::memcpy(buf, v.data(), need(8 * v.size()));
        break;
    }
    case SPD_Q_HSS_PIVOTS: {
        std::vector<int32_t> v;
        for (int k = 1; k < t.L; ++k) v.insert(v.end(), H->lv[k].piv.begin(), H->lv[k].piv.end());
        std::memcpy(buf, v.data(), need(4 * v.size()));
        break;
    }
    default: throw Error(SPD_EINVAL, "spd_query: unknown HSS query");
    }
}

}  // namespace spd
