// h2sym.cu -- stored, symmetric kernel blocks for the single-vector H2 product
// (the PCG matvec, k = 1).
//
// At k = 1 evaluating K on the fly is FP64-ALU bound (exp/sqrt per entry for two
// useful flops), while a stored block is read once per product: HBM bound.  K is
// symmetric, so only the blocks (a, b) with a <= b are visited: the near-field leaf
// blocks K(X_a, X_b) + sigma I and, per level, the Type-3 couplings
// B^{H2}_ab = K(X_{J_a}, X_{J_b}) (eqn:uniformbasis_h2).  One block serves
// y_a += K_ab x_b and y_b += K_ab^T x_a, which halves the bytes (stored) or the
// kernel evaluations (on the fly) per product.  Blocks are stored while they fit
// the memory budget; the rest are evaluated on the fly by the same kernel.
//
// Layout: a block is cut into 32-row tiles ("pieces"); a piece is 32 x n_b
// doubles, column c holding K(rows of the tile, source point c) (rows past the
// node are zero), so a warp reads one column as one 256-byte line.
// Apply: one CTA per piece, warps take 32-column chunks; the forward product is a
// lane-per-row dot, the transposed product a butterfly transpose-reduction across
// the 32 lanes (lane c ends with column c's sum).  Partial results go to scratch,
// and a gather kernel sums each output node's partials in a fixed order (no
// atomics: the product is bitwise reproducible) and overwrites y / yh.
#include "h2.hpp"
#include "comm.hpp"
#include "phases.cuh"
#include <algorithm>

namespace spd {


template <int KID>
__global__ void __launch_bounds__(256) sym_build_kernel(KernelParams kp, double shift, int d,
                                                        const SymBuild* __restrict__ bp, double* __restrict__ vals) {
    const SymBuild b = bp[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double rx[4] = {0.0, 0.0, 0.0, 0.0};
    if (lane < b.nr)
        for (int a = 0; a < d; ++a) rx[a] = b.tx[(size_t)a * b.tds + lane];
    const bool sh = shift != 0.0 && b.tid0 >= 0;
    double* out = vals + b.vbase + lane;
    for (int c = warp; c < b.nb; c += 8) {
        double kv;
        if constexpr (KID == SPD_K_RPY) {
            kv = rpy_entry(kp, rx[0] - b.sx[c], rx[1] - b.sx[b.sds + c], rx[2] - b.sx[2 * (size_t)b.sds + c],
                           (int)rx[3], (int)b.sx[3 * (size_t)b.sds + c]);
        } else {
            double r2 = 0.0;
            for (int a = 0; a < d; ++a) {
                const double df = rx[a] - b.sx[(size_t)a * b.sds + c];
                r2 += df * df;
            }
            kv = kval_sym<KID>(kp, r2);
        }
        if (sh && b.tid0 + lane == b.sid0 + c) kv += shift;
        out[(size_t)c * 32] = lane < b.nr ? kv : 0.0;
    }
}

template <int KID, bool EVAL>
__global__ void __launch_bounds__(SY_NW * 32) sym_apply_kernel(const SymPiece* __restrict__ pieces, SymVecs xin,
                                                               const double* __restrict__ vals,
                                                               double* __restrict__ scratch, KernelParams kp,
                                                               double shift, int d) {
    extern __shared__ double tp[];
    sym_piece<KID, EVAL>(pieces[blockIdx.x], xin, vals, scratch, kp, shift, d, 0, tp);
}

// long lists: one CTA per (output node, 32-row tile); short lists: one warp each
__global__ void __launch_bounds__(PH_T) sym_gather_big_kernel(const SymGNode* __restrict__ nodes,
                                                              const SymContrib* __restrict__ con, SymVecsOut yout,
                                                              const double* __restrict__ scratch) {
    __shared__ double red[PH_W * 32];
    gather_item_cta(nodes[blockIdx.x], con, yout, scratch, red);
}
__global__ void __launch_bounds__(256) sym_gather_kernel(const SymGNode* __restrict__ nodes, int n,
                                                         const SymContrib* __restrict__ con, SymVecsOut yout,
                                                         const double* __restrict__ scratch) {
    const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (w < n) gather_item_warp(nodes[w], con, yout, scratch);
}

// ----------------------------------------------------------------- host side
namespace {
struct PlanBlock { int slot, a, b; };   // block (a <= b) of slot 0 (near, leaves) or level slot
}

// budget: doubles of stored blocks allowed (pieces past it are evaluated on the fly)
static void sym_plan(const spd_h2_s* h, int64_t budget, double frac, std::vector<SymBuild>* builds,
                     std::vector<SymPiece>* pieces, std::vector<SymGNode>* gnodes, std::vector<SymContrib>* gcon,
                     int64_t* nvals, int64_t* nscratch, double* flops, int64_t* nall, int* nbig_out = nullptr,
                     int* nbmax_out = nullptr, std::unordered_map<uint64_t, int64_t>* bases = nullptr) {
    int64_t npiece = 0;
    int nbmax = 1;
    const TreeH& t = h->tree;
    const int L = t.L, d = h->d;
    const int64_t N = h->N;
    (void)d;
    int64_t vb = 0, sc = 0, all = 0;
    double fl = 0.0;
    // per output node (slot, local index) and 32-row tile: list of contributions
    std::vector<std::vector<std::vector<std::vector<SymContrib>>>> con(L);
    const int l1 = t.first(1), nl = t.count(1);
    con[0].resize(nl);
    for (int a = 0; a < nl; ++a) con[0][a].resize(ceil_div(t.size(l1 + a), 32));
    for (int lk = 1; lk < L; ++lk) {
        con[lk].resize(h->lv[lk].count);
        for (int a = 0; a < h->lv[lk].count; ++a) con[lk][a].resize(ceil_div(h->lv[lk].rank[a], 32));
    }
    // subtree sharding (real communicator, §8(e)): keep the blocks that touch an owned
    // node and gather only owned outputs (boundary blocks are computed by both owners)
    const spd_comm_s* cm = h->comm;
    const bool shard = comm_real(cm) && nl >= cm->nranks;
    auto mine = [&](int slot, int a) {
        if (!shard) return true;
        const int o = shard_owner(cm, slot == 0 ? nl : h->lv[slot].count, a);
        return o < 0 || o == cm->rank;
    };
    auto add_block = [&](int slot, int a, int b) {
        // rows: node a, columns: node b (local indices within the slot)
        if (!mine(slot, a) && !mine(slot, b)) return;
        int na, nb;
        const double *tx, *sx;
        int64_t ds, tid0 = -1, sid0 = -1, xa0, xb0;
        if (slot == 0) {
            na = (int)t.size(l1 + a); nb = (int)t.size(l1 + b);
            tx = h->X.p + t.begin[l1 + a]; sx = h->X.p + t.begin[l1 + b]; ds = N;
            tid0 = t.begin[l1 + a]; sid0 = t.begin[l1 + b];
            xa0 = t.begin[l1 + a]; xb0 = t.begin[l1 + b];
        } else {
            const H2Level& lv = h->lv[slot];
            na = lv.rank[a]; nb = lv.rank[b];
            tx = lv.skelX.p + lv.off[a]; sx = lv.skelX.p + lv.off[b]; ds = lv.S;
            xa0 = lv.off[a]; xb0 = lv.off[b];
        }
        if (na == 0 || nb == 0) return;
        const bool diag = (a == b);
        fl += 2.0 * na * nb * (diag ? 1.0 : 2.0);
        const int64_t base0 = vb;
        bool all_stored = true;
        for (int r0 = 0; r0 < na; r0 += 32 * SY_NW) {
            const int nr = std::min(32 * SY_NW, na - r0);          // band of up to 4 row tiles
            const int nt = ceil_div(nr, 32);
            // stored if within the budget and, when only a fraction should be stored,
            // on the evenly spread pattern (stored and evaluated bands interleave, so
            // every SM streams and evaluates at the same time)
            const int64_t ip = npiece++;
            const bool pat = frac >= 1.0 || (int64_t)((ip + 1) * frac) > (int64_t)(ip * frac);
            const bool store = pat && vb + 32LL * nb * nt <= budget;
            all += 32LL * nb * nt;
            if (builds && store)
                for (int w = 0; w < nt; ++w)
                    builds->push_back({tx + r0 + 32 * w, sx, ds, ds, slot == 0 ? tid0 + r0 + 32 * w : -1,
                                       slot == 0 ? sid0 : -1, std::min(32, nr - 32 * w), nb, vb + 32LL * nb * w});
            SymPiece pc;
            pc.vbase = store ? vb : -1; pc.slot = slot; pc.nr = nr; pc.nb = nb;
            pc.tx = tx + r0; pc.sx = sx; pc.tds = ds; pc.sds = ds;
            pc.tid0 = slot == 0 ? tid0 + r0 : -1; pc.sid0 = slot == 0 ? sid0 : -1;
            pc.xa_off = xa0 + r0; pc.xb_off = xb0;
            pc.fwd = sc; sc += 32 * nt;
            pc.trn = diag ? -1 : sc;
            if (!diag) sc += nb;
            if (pieces) pieces->push_back(pc);
            if (store) vb += 32LL * nb * nt;
            else all_stored = false;
            nbmax = std::max(nbmax, nb);
            for (int w = 0; w < nt; ++w)
                con[slot][a][r0 / 32 + w].push_back({pc.fwd + 32 * w, 0, std::min(32, nr - 32 * w)});
            if (!diag)
                for (int tb = 0; tb * 32 < nb; ++tb) con[slot][b][tb].push_back({pc.trn + 32 * tb, 0, std::min(32, nb - 32 * tb)});
        }
        if (bases && all_stored) (*bases)[sym_key(slot, a, b)] = base0;
    };
    for (const auto& pr : h->lists.near)
        if (pr.first <= pr.second) add_block(0, pr.first - l1, pr.second - l1);
    for (int lk = 1; lk < L; ++lk) {
        const int f = h->lv[lk].first;
        for (const auto& pr : h->lists.type3[lk])
            if (pr.first < pr.second) add_block(lk, pr.first - f, pr.second - f);
    }
    if (gnodes) {
        // long lists (>= SYM_BIG partials) first: those are reduced by a whole CTA
        for (int pass = 0; pass < 2; ++pass) {
            for (int slot = 0; slot < L; ++slot) {
                const int cnt = slot == 0 ? nl : h->lv[slot].count;
                for (int a = 0; a < cnt; ++a) {
                    if (!mine(slot, a)) continue;
                    const int n = slot == 0 ? (int)t.size(l1 + a) : h->lv[slot].rank[a];
                    const int64_t off = slot == 0 ? t.begin[l1 + a] : h->lv[slot].off[a];
                    for (int tt = 0; tt * 32 < n; ++tt) {
                        const auto& L_ = con[slot][a][tt];
                        if ((pass == 0) != ((int)L_.size() >= SYM_BIG)) continue;
                        SymGNode g;
                        g.slot = slot; g.n = std::min(32, n - 32 * tt);
                        g.off = off + 32 * tt;
                        g.c0 = (int)gcon->size();
                        for (auto& q : L_) gcon->push_back(q);
                        g.c1 = (int)gcon->size();
                        gnodes->push_back(g);
                    }
                }
            }
            if (pass == 0 && nbig_out) *nbig_out = (int)gnodes->size();
        }
    }
    if (nbmax_out) *nbmax_out = nbmax;
    *nvals = vb;
    *nscratch = sc;
    *flops = fl;
    *nall = all;
}

size_t h2sym_bytes(const spd_h2_s* h) {
    int64_t nv = 0, ns = 0, na = 0;
    double fl = 0;
    sym_plan(h, 0, 1.0, nullptr, nullptr, nullptr, nullptr, &nv, &ns, &fl, &na);
    return 8 * (size_t)(na + ns);
}

void h2sym_build(spd_h2_s* h, double budget_bytes, cudaStream_t s) {
    H2SymStore& st = h->sym;
    if (st.built) return;
    std::vector<SymBuild> builds;
    std::vector<SymPiece> pieces;
    std::vector<SymGNode> gnodes;
    std::vector<SymContrib> gcon;
    int64_t nv = 0, ns = 0, na = 0;
    st.base.clear();
    sym_plan(h, (int64_t)(budget_bytes / 8), h->sym_frac, &builds, &pieces, &gnodes, &gcon, &nv, &ns, &st.flops, &na,
             &st.nbig, &st.nbmax, &st.base);
    st.vals.alloc(std::max<int64_t>(1, nv));
    st.scratch.alloc(std::max<int64_t>(1, ns));
    st.pieces.upload(pieces, s);
    st.gnodes.upload(gnodes, s);
    st.gnodes_h = gnodes;
    {
        const int L = h->tree.L;
        st.piece_off.assign(L + 1, 0);
        for (const auto& pc : pieces) st.piece_off[pc.slot + 1]++;
        for (int l = 0; l < L; ++l) st.piece_off[l + 1] += st.piece_off[l];
        for (size_t i = 1; i < pieces.size(); ++i)
            SPD_REQUIRE(pieces[i].slot >= pieces[i - 1].slot, "h2sym: pieces not ordered by slot");
    }
    st.gcon.upload(gcon, s);
    st.npieces = (int)pieces.size();
    st.ngnodes = (int)gnodes.size();
    st.bytes = 8.0 * nv;
    st.stored_frac = na ? (double)nv / (double)na : 1.0;
    if (!builds.empty()) {
        DevArray<SymBuild> db(s, builds);
        ProfScope prof(s, "sym_build", 0, 8.0 * nv);
        const KernelParams& kp = h->kp;
        const double sh = h->kern.shift;
        for (size_t off = 0; off < builds.size(); off += (1u << 30)) {
            const unsigned nb = (unsigned)std::min<size_t>(builds.size() - off, 1u << 30);
            switch (kp.id) {
            case SPD_K_GAUSSIAN: sym_build_kernel<SPD_K_GAUSSIAN><<<nb, 256, 0, s>>>(kp, sh, h->d, db.p + off, st.vals.p); break;
            case SPD_K_MATERN32: sym_build_kernel<SPD_K_MATERN32><<<nb, 256, 0, s>>>(kp, sh, h->d, db.p + off, st.vals.p); break;
            case SPD_K_EXPONENTIAL: sym_build_kernel<SPD_K_EXPONENTIAL><<<nb, 256, 0, s>>>(kp, sh, h->d, db.p + off, st.vals.p); break;
            case SPD_K_RPY: sym_build_kernel<SPD_K_RPY><<<nb, 256, 0, s>>>(kp, sh, h->d, db.p + off, st.vals.p); break;
            default: sym_build_kernel<SPD_K_IMQ><<<nb, 256, 0, s>>>(kp, sh, h->d, db.p + off, st.vals.p); break;
            }
            SPD_LAUNCH();
        }
    }
    st.built = true;
}

template <int KID>
static void launch_sym(cudaStream_t s, unsigned nb, size_t smem, const H2SymStore& st, const SymVecs& xin,
                       const KernelParams& kp, double sh, int d) {
    if (st.stored_frac >= 1.0) {
        if (smem > 48 * 1024)
            SPD_CUDA(cudaFuncSetAttribute(sym_apply_kernel<KID, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        sym_apply_kernel<KID, false><<<nb, SY_NW * 32, smem, s>>>(st.pieces.p, xin, st.vals.p, st.scratch.p, kp, sh, d);
    } else {
        if (smem > 48 * 1024)
            SPD_CUDA(cudaFuncSetAttribute(sym_apply_kernel<KID, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        sym_apply_kernel<KID, true><<<nb, SY_NW * 32, smem, s>>>(st.pieces.p, xin, st.vals.p, st.scratch.p, kp, sh, d);
    }
    SPD_LAUNCH();
}

// y (leaf slot) and yh[l] are OVERWRITTEN with the near / coupling products of
// x and xh[l]; the caller runs the up pass before and the down pass after.
void h2sym_apply(spd_h2_s* h, const double* x, double* y, const std::vector<double*>& xh,
                 const std::vector<double*>& yh, cudaStream_t s) {
    H2SymStore& st = h->sym;
    const int L = h->tree.L;
    SPD_REQUIRE(L <= SYM_MAX_SLOTS, "h2sym: too many levels");
    SymVecs xin{};
    SymVecsOut yout{};
    xin.p[0] = x;
    yout.p[0] = y;
    for (int l = 1; l < L; ++l) { xin.p[l] = xh[l]; yout.p[l] = yh[l]; }
    if (st.npieces) {
        ProfScope prof(s, st.stored_frac >= 1.0 ? "sym_gemv" : "sym_gemv_eval", st.flops, st.bytes);
        const unsigned nb = (unsigned)st.npieces;
        const KernelParams& kp = h->kp;
        const double sh = h->kern.shift;
        const size_t smem = sizeof(double) * SY_NW * st.nbmax;
        switch (kp.id) {
        case SPD_K_GAUSSIAN: launch_sym<SPD_K_GAUSSIAN>(s, nb, smem, st, xin, kp, sh, h->d); break;
        case SPD_K_MATERN32: launch_sym<SPD_K_MATERN32>(s, nb, smem, st, xin, kp, sh, h->d); break;
        case SPD_K_EXPONENTIAL: launch_sym<SPD_K_EXPONENTIAL>(s, nb, smem, st, xin, kp, sh, h->d); break;
        case SPD_K_RPY: launch_sym<SPD_K_RPY>(s, nb, smem, st, xin, kp, sh, h->d); break;
        default: launch_sym<SPD_K_IMQ>(s, nb, smem, st, xin, kp, sh, h->d); break;
        }
    }
    if (st.ngnodes) {
        ProfScope prof(s, "sym_gather", 0, 0);
        if (st.nbig) {
            sym_gather_big_kernel<<<(unsigned)st.nbig, PH_T, 0, s>>>(st.gnodes.p, st.gcon.p, yout, st.scratch.p);
            SPD_LAUNCH();
        }
        const int ns = st.ngnodes - st.nbig;
        if (ns > 0) {
            sym_gather_kernel<<<(unsigned)ceil_div(ns, 8), 256, 0, s>>>(st.gnodes.p + st.nbig, ns, st.gcon.p, yout,
                                                                       st.scratch.p);
            SPD_LAUNCH();
        }
    }
}

}  // namespace spd
