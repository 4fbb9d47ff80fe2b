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
#include <algorithm>

namespace spd {

constexpr int SY_NW = 4;               // warps per apply CTA

template <int KID>
__device__ __forceinline__ double kval_sym(const KernelParams& kp, double r2) {
    if (KID == SPD_K_GAUSSIAN) return exp(-r2 * kp.inv_l2);
    if (KID == SPD_K_MATERN32) { const double t = sqrt(r2) * kp.sqrt3_inv_l; return (1.0 + t) * exp(-t); }
    if (KID == SPD_K_EXPONENTIAL) return exp(-sqrt(r2) * kp.inv_l);
    return rsqrt(r2 + kp.l2);
}

template <int KID>
__global__ void __launch_bounds__(256) sym_build_kernel(KernelParams kp, double shift, int d,
                                                        const SymBuild* __restrict__ bp, double* __restrict__ vals) {
    const SymBuild b = bp[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double rx[3] = {0.0, 0.0, 0.0};
    if (lane < b.nr)
        for (int a = 0; a < d; ++a) rx[a] = b.tx[(size_t)a * b.tds + lane];
    const bool sh = shift != 0.0 && b.tid0 >= 0;
    double* out = vals + b.vbase + lane;
    for (int c = warp; c < b.nb; c += 8) {
        double r2 = 0.0;
        for (int a = 0; a < d; ++a) {
            const double df = rx[a] - b.sx[(size_t)a * b.sds + c];
            r2 += df * df;
        }
        double kv = kval_sym<KID>(kp, r2);
        if (sh && b.tid0 + lane == b.sid0 + c) kv += shift;
        out[(size_t)c * 32] = lane < b.nr ? kv : 0.0;
    }
}

template <int KID>
__global__ void __launch_bounds__(SY_NW * 32) sym_apply_kernel(const SymPiece* __restrict__ pieces, SymVecs xin,
                                                               const double* __restrict__ vals,
                                                               double* __restrict__ scratch, KernelParams kp,
                                                               double shift, int d) {
    __shared__ double red[SY_NW][32];
    const SymPiece pc = pieces[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* xs = xin.p[pc.slot];
    const bool trn = pc.trn >= 0;
    const double xa = (trn && lane < pc.nr) ? xs[pc.xa_off + lane] : 0.0;
    const bool stored = pc.vbase >= 0;
    const double* v = vals + (stored ? pc.vbase : 0) + lane;
    double rx0 = 0.0, rx1 = 0.0, rx2 = 0.0;     // on the fly: this lane's row point
    if (!stored && lane < pc.nr) {
        rx0 = pc.tx[lane];
        if (d > 1) rx1 = pc.tx[pc.tds + lane];
        if (d > 2) rx2 = pc.tx[2 * pc.tds + lane];
    }
    const bool sh = !stored && shift != 0.0 && pc.tid0 >= 0;
    double acc = 0.0;
    const int nch = (pc.nb + 31) >> 5;
    for (int ch = warp; ch < nch; ch += SY_NW) {
        const int c0 = ch * 32;
        const int cn = min(32, pc.nb - c0);
        const double xbv = lane < cn ? xs[pc.xb_off + c0 + lane] : 0.0;
        double kv[32];
        if (stored) {
            if (cn == 32) {
#pragma unroll
                for (int c = 0; c < 32; ++c) kv[c] = __ldg(v + (size_t)(c0 + c) * 32);
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c) kv[c] = c < cn ? __ldg(v + (size_t)(c0 + c) * 32) : 0.0;
            }
        } else {
            // source point c0 + lane, broadcast by shuffles; rows past nr give 0
            double s0 = 0.0, s1 = 0.0, s2 = 0.0;
            if (lane < cn) {
                s0 = pc.sx[c0 + lane];
                if (d > 1) s1 = pc.sx[pc.sds + c0 + lane];
                if (d > 2) s2 = pc.sx[2 * pc.sds + c0 + lane];
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const double d0 = rx0 - __shfl_sync(0xffffffffu, s0, c);
                const double d1 = rx1 - __shfl_sync(0xffffffffu, s1, c);
                const double d2 = rx2 - __shfl_sync(0xffffffffu, s2, c);
                double k = kval_sym<KID>(kp, d0 * d0 + d1 * d1 + d2 * d2);
                if (sh && pc.tid0 + lane == pc.sid0 + c0 + c) k += shift;
                kv[c] = (c < cn && lane < pc.nr) ? k : 0.0;
            }
        }
        double f0 = 0.0, f1 = 0.0;
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
            f0 += kv[c] * __shfl_sync(0xffffffffu, xbv, c);
            f1 += kv[c + 1] * __shfl_sync(0xffffffffu, xbv, c + 1);
        }
        acc += f0 + f1;
        if (trn) {
#pragma unroll
            for (int c = 0; c < 32; ++c) kv[c] *= xa;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int j = 0; j < o; ++j) {
                    const double send = up ? kv[j] : kv[j + o];
                    const double keep = up ? kv[j + o] : kv[j];
                    kv[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            if (lane < cn) scratch[pc.trn + c0 + lane] = kv[0];
        }
    }
    red[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && lane < pc.nr) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < SY_NW; ++w) s += red[w][lane];
        scratch[pc.fwd + lane] = s;
    }
}

// one CTA per (output node, 32-row tile): y[tile] = sum of the tile's partials in list order
// (warp w takes partials w, w+8, ...; the 8 warp sums are added in warp order)
__global__ void __launch_bounds__(256) sym_gather_kernel(const SymGNode* __restrict__ nodes,
                                                         const SymContrib* __restrict__ con, SymVecsOut yout,
                                                         const double* __restrict__ scratch) {
    __shared__ double red[8][32];
    const SymGNode g = nodes[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double a0 = 0.0, a1 = 0.0;
    int c = g.c0 + warp;
    for (; c + 8 < g.c1; c += 16) {
        const SymContrib q0 = con[c], q1 = con[c + 8];
        if (lane < q0.len) a0 += scratch[q0.soff + lane];
        if (lane < q1.len) a1 += scratch[q1.soff + lane];
    }
    if (c < g.c1) {
        const SymContrib q0 = con[c];
        if (lane < q0.len) a0 += scratch[q0.soff + lane];
    }
    red[warp][lane] = a0 + a1;
    __syncthreads();
    if (warp == 0 && lane < g.n) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) sum += red[w][lane];
        yout.p[g.slot][g.off + lane] = sum;
    }
}

// ----------------------------------------------------------------- host side
namespace {
struct PlanBlock { int slot, a, b; };   // block (a <= b) of slot 0 (near, leaves) or level slot
}

// budget: doubles of stored blocks allowed (pieces past it are evaluated on the fly)
static void sym_plan(const spd_h2_s* h, int64_t budget, std::vector<SymBuild>* builds, std::vector<SymPiece>* pieces,
                     std::vector<SymGNode>* gnodes, std::vector<SymContrib>* gcon, int64_t* nvals, int64_t* nscratch,
                     double* flops, int64_t* nall) {
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
    auto add_block = [&](int slot, int a, int b) {
        // rows: node a, columns: node b (local indices within the slot)
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
        for (int r0 = 0; r0 < na; r0 += 32) {
            const int nr = std::min(32, na - r0);
            const bool store = vb + 32LL * nb <= budget;
            all += 32LL * nb;
            if (builds && store)
                builds->push_back({tx + r0, sx, ds, ds, slot == 0 ? tid0 + r0 : -1, slot == 0 ? sid0 : -1, nr, nb, vb});
            SymPiece pc;
            pc.vbase = store ? vb : -1; pc.slot = slot; pc.nr = nr; pc.nb = nb;
            pc.tx = tx + r0; pc.sx = sx; pc.tds = ds; pc.sds = ds;
            pc.tid0 = slot == 0 ? tid0 + r0 : -1; pc.sid0 = slot == 0 ? sid0 : -1;
            pc.xa_off = xa0 + r0; pc.xb_off = xb0;
            pc.fwd = sc; sc += 32;
            pc.trn = diag ? -1 : sc;
            if (!diag) sc += nb;
            if (pieces) pieces->push_back(pc);
            if (store) vb += 32LL * nb;
            con[slot][a][r0 / 32].push_back({pc.fwd, 0, nr});
            if (!diag)
                for (int tb = 0; tb * 32 < nb; ++tb) con[slot][b][tb].push_back({pc.trn + 32 * tb, 0, std::min(32, nb - 32 * tb)});
        }
    };
    for (const auto& pr : h->lists.near)
        if (pr.first <= pr.second) add_block(0, pr.first - l1, pr.second - l1);
    for (int lk = 1; lk < L; ++lk) {
        const int f = h->lv[lk].first;
        for (const auto& pr : h->lists.type3[lk])
            if (pr.first < pr.second) add_block(lk, pr.first - f, pr.second - f);
    }
    if (gnodes) {
        for (int slot = 0; slot < L; ++slot) {
            const int cnt = slot == 0 ? nl : h->lv[slot].count;
            for (int a = 0; a < cnt; ++a) {
                const int n = slot == 0 ? (int)t.size(l1 + a) : h->lv[slot].rank[a];
                const int64_t off = slot == 0 ? t.begin[l1 + a] : h->lv[slot].off[a];
                for (int tt = 0; tt * 32 < n; ++tt) {
                    SymGNode g;
                    g.slot = slot; g.n = std::min(32, n - 32 * tt);
                    g.off = off + 32 * tt;
                    g.c0 = (int)gcon->size();
                    for (auto& q : con[slot][a][tt]) gcon->push_back(q);
                    g.c1 = (int)gcon->size();
                    gnodes->push_back(g);
                }
            }
        }
    }
    *nvals = vb;
    *nscratch = sc;
    *flops = fl;
    *nall = all;
}

size_t h2sym_bytes(const spd_h2_s* h) {
    int64_t nv = 0, ns = 0, na = 0;
    double fl = 0;
    sym_plan(h, 0, nullptr, nullptr, nullptr, nullptr, &nv, &ns, &fl, &na);
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
    sym_plan(h, (int64_t)(budget_bytes / 8), &builds, &pieces, &gnodes, &gcon, &nv, &ns, &st.flops, &na);
    st.vals.alloc(std::max<int64_t>(1, nv));
    st.scratch.alloc(std::max<int64_t>(1, ns));
    st.pieces.upload(pieces, s);
    st.gnodes.upload(gnodes, s);
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
            default: sym_build_kernel<SPD_K_IMQ><<<nb, 256, 0, s>>>(kp, sh, h->d, db.p + off, st.vals.p); break;
            }
            SPD_LAUNCH();
        }
    }
    st.built = true;
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
        switch (kp.id) {
        case SPD_K_GAUSSIAN: sym_apply_kernel<SPD_K_GAUSSIAN><<<nb, SY_NW * 32, 0, s>>>(st.pieces.p, xin, st.vals.p, st.scratch.p, kp, sh, h->d); break;
        case SPD_K_MATERN32: sym_apply_kernel<SPD_K_MATERN32><<<nb, SY_NW * 32, 0, s>>>(st.pieces.p, xin, st.vals.p, st.scratch.p, kp, sh, h->d); break;
        case SPD_K_EXPONENTIAL: sym_apply_kernel<SPD_K_EXPONENTIAL><<<nb, SY_NW * 32, 0, s>>>(st.pieces.p, xin, st.vals.p, st.scratch.p, kp, sh, h->d); break;
        default: sym_apply_kernel<SPD_K_IMQ><<<nb, SY_NW * 32, 0, s>>>(st.pieces.p, xin, st.vals.p, st.scratch.p, kp, sh, h->d); break;
        }
        SPD_LAUNCH();
    }
    if (st.ngnodes) {
        ProfScope prof(s, "sym_gather", 0, 0);
        sym_gather_kernel<<<(unsigned)st.ngnodes, 256, 0, s>>>(st.gnodes.p, st.gcon.p, yout, st.scratch.p);
        SPD_LAUNCH();
    }
}

}  // namespace spd
