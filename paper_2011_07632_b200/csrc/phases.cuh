// phases.cuh -- device bodies of the single-vector (k = 1) phases of one PCG
// iteration, shared by their stand-alone kernels (h2basis.cu, h2sym.cu,
// hsolve.cu) and by the persistent PCG kernel (pcgk.cu):
//   basis_up_item / basis_down_item   H2 basis passes in ID form      (CTA, PH_T threads)
//   sym_piece                          symmetric near + coupling band  (4-warp group)
//   gather_item_cta / _warp            partial sums -> y / yh          (CTA / one warp)
//   hss_item                           32 outputs of one HSS solve level   (CTA)
// Every body uses only its own CTA (or warp group), fixed summation orders (no
// atomics), and shared memory passed in by the caller.
#pragma once
#include "hss.hpp"

namespace spd {

constexpr int PH_T = 256, PH_W = PH_T / 32;     // CTA size of the CTA-wide bodies (8 warps)

// Vectors written by other CTAs earlier in the same (persistent) kernel are read
// through L2 (ld.global.cg): L1 is not coherent across SMs.  Read-only operands
// (factors, interpolation and stored kernel blocks) use __ldg.
__device__ __forceinline__ double ldv(const double* p) { return __ldcg(p); }

// ================================================================= H2 basis passes (ID form)
// E_i[piv[k], k] = 1 (k < s), E_i[piv[s + c], :] = T_i[:, c]^T, T_i: s x (n_c - s), ld s
struct BasisItem {
    const double* in;     // up: x_c (n_c) ; down: yh_i (s)
    double* out;          // up: xh_i (s)  ; down: y_c (n_c), accumulated
    const double* T;      // s x (n_c - s), ld s
    const int* piv;       // n_c
    int s, nc, tile;      // tile: 32-row tile of xh (up) / 32-column tile of T (down)
};

// up: xh[k] = x[piv[k]] + sum_c T[k, c] x[piv[s + c]] for k in the tile (lane = k);
// warp w takes columns c = w (mod 16), 8 loads in flight per lane; the warp sums are
// added in warp order.  sm: n_c - s doubles + PH_W * 32 doubles.
__device__ __forceinline__ void basis_up_item(const BasisItem& it, double* sm) {
    double* xg = sm;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = it.s, nr = it.nc - it.s;
    double* red = sm + nr;
    for (int c = threadIdx.x; c < nr; c += PH_T) xg[c] = ldv(it.in + it.piv[s + c]);
    __syncthreads();
    const int k = it.tile * 32 + lane;
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    if (k < s) {
        const double* p = it.T + k;
        int c = warp;
        for (; c + 15 * PH_W < nr; c += 16 * PH_W) {     // 16 loads in flight per lane
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = __ldg(p + (size_t)(c + u * PH_W) * s);
#pragma unroll
            for (int u = 0; u < 16; ++u) acc[u & 7] += v[u] * xg[c + u * PH_W];
        }
        for (; c + 7 * PH_W < nr; c += 8 * PH_W) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(p + (size_t)(c + u * PH_W) * s);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] += v[u] * xg[c + u * PH_W];
        }
        for (; c < nr; c += PH_W) acc[0] += __ldg(p + (size_t)c * s) * xg[c];
    }
    red[warp * 32 + lane] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    __syncthreads();
    if (warp == 0 && k < s) {
        double sum = ldv(it.in + it.piv[k]);
#pragma unroll
        for (int w = 0; w < PH_W; ++w) sum += red[w * 32 + lane];
        it.out[k] = sum;
    }
    __syncthreads();
}

// butterfly transpose-reduction: lane l holds v[0..31] (one value per column);
// on exit v[0] of lane c is the sum over the 32 lanes of column c
__device__ __forceinline__ void butterfly32(double (&v)[32]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < o; ++j) {
            const double send = up ? v[j] : v[j + o];
            const double keep = up ? v[j + o] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
}

// down: y[piv[s + c]] += sum_k T[k, c] yh[k] for the tile's 32 columns c and
// y[piv[k]] += yh[k] for k in [32 tile, 32 tile + 32).  Warp w takes the 32-row chunks
// q = w (mod 16): 32 coalesced loads (lane = row) scaled by yh, butterfly-reduced.
// sm: s doubles + PH_W * 32 doubles.
__device__ __forceinline__ void basis_down_item(const BasisItem& it, double* sm) {
    double* yh = sm;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = it.s, nr = it.nc - it.s;
    double* red = sm + s;
    for (int k = threadIdx.x; k < s; k += PH_T) yh[k] = ldv(it.in + k);
    __syncthreads();
    const int k0 = it.tile * 32;
    if (warp == 0 && k0 + lane < s) {
        double* o = it.out + it.piv[k0 + lane];
        *o = ldv(o) + yh[k0 + lane];
    }
    const int c0 = k0, cn = min(32, nr - c0);
    if (cn > 0) {
        double acc = 0.0;
        for (int q = warp; q * 32 < s; q += PH_W) {
            const int k = q * 32 + lane;
            const double y = k < s ? yh[k] : 0.0;
            const double* p = it.T + k + (size_t)c0 * s;
            double v[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = (k < s && c < cn) ? __ldg(p + (size_t)c * s) : 0.0;
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] *= y;
            butterfly32(v);
            acc += v[0];
        }
        red[warp * 32 + lane] = acc;
        __syncthreads();
        if (warp == 0 && lane < cn) {
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < PH_W; ++w) sum += red[w * 32 + lane];
            double* o = it.out + it.piv[s + c0 + lane];
            *o = ldv(o) + sum;
        }
    }
    __syncthreads();
}

// ================================================================= symmetric near + coupling blocks
constexpr int SY_NW = 4;               // warps per piece (one warp group)

template <int KID>
__device__ __forceinline__ double kval_sym(const KernelParams& kp, double r2) {
    if (KID == SPD_K_GAUSSIAN) return exp(-r2 * kp.inv_l2);
    if (KID == SPD_K_MATERN32) { const double t = sqrt(r2) * kp.sqrt3_inv_l; return (1.0 + t) * exp(-t); }
    if (KID == SPD_K_EXPONENTIAL) return exp(-sqrt(r2) * kp.inv_l);
    return rsqrt(r2 + kp.l2);
}

__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;\n" :: "r"(id), "r"(nthreads) : "memory");
}

// One band of a block (a <= b): up to SY_NW row tiles of 32 rows [pc.r0 + 32 w, ...),
// warp w of group `grp` owning tile w.  Per 32-column chunk a warp loads (stored) or
// evaluates the 32 x 32 tile, adds K x_b to its rows' forward sums and, off the
// diagonal, butterfly-reduces K^T x_a over its 32 rows into tp[w][cols].  At the end
// the forward sums go to scratch (one 32-vector per row tile) and the transposed sums
// of the band are added over the warps in warp order (one n_b-vector per band).
// tp: SY_NW * nb doubles of this group.
template <int KID, bool EVAL>
__device__ __forceinline__ void sym_piece(const SymPiece& pc, const SymVecs& xin, const double* __restrict__ vals,
                                          double* __restrict__ scratch, const KernelParams& kp, double shift, int d,
                                          int grp, double* tp) {
    const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & (SY_NW - 1);
    const int gt = threadIdx.x & (SY_NW * 32 - 1);
    const double* xs = xin.p[pc.slot];
    const bool trn = pc.trn >= 0;
    const int nb = pc.nb;
    const int r0 = warp * 32;                       // this warp's tile within the band
    const int nr = min(32, pc.nr - r0);             // valid rows of the tile (<= 0: idle warp)
    if (nr > 0) {
        const double xa = (trn && lane < nr) ? ldv(xs + pc.xa_off + r0 + lane) : 0.0;
        const bool stored = !EVAL || pc.vbase >= 0;      // !EVAL: every piece is stored
        const double* v = vals + (stored ? pc.vbase + (int64_t)warp * 32 * nb : 0) + lane;
        double rx0 = 0.0, rx1 = 0.0, rx2 = 0.0;     // on the fly: this lane's row point
        int rc = 0;                                 // RPY: component of the row dof
        if (!stored && lane < nr) {
            rx0 = pc.tx[r0 + lane];
            if (d > 1) rx1 = pc.tx[pc.tds + r0 + lane];
            if (d > 2) rx2 = pc.tx[2 * pc.tds + r0 + lane];
            if (KID == SPD_K_RPY) rc = (int)pc.tx[3 * pc.tds + r0 + lane];
        }
        const bool sh = !stored && shift != 0.0 && pc.tid0 >= 0;
        double acc = 0.0;
        const int nch = (nb + 31) >> 5;
        for (int ch = 0; ch < nch; ++ch) {
            const int c0 = ch * 32;
            const int cn = min(32, nb - c0);
            const double xbv = lane < cn ? ldv(xs + pc.xb_off + c0 + lane) : 0.0;
            double kv[32];
            if (stored) {
                if (cn == 32) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) kv[c] = __ldg(v + (size_t)(c0 + c) * 32);
                } else {
#pragma unroll
                    for (int c = 0; c < 32; ++c) kv[c] = c < cn ? __ldg(v + (size_t)(c0 + c) * 32) : 0.0;
                }
            } else if (EVAL) {
                double s0 = 0.0, s1 = 0.0, s2 = 0.0;  // source point c0 + lane, broadcast by shuffles
                int sc = 0;
                if (lane < cn) {
                    s0 = pc.sx[c0 + lane];
                    if (d > 1) s1 = pc.sx[pc.sds + c0 + lane];
                    if (d > 2) s2 = pc.sx[2 * pc.sds + c0 + lane];
                    if (KID == SPD_K_RPY) sc = (int)pc.sx[3 * pc.sds + c0 + lane];
                }
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const double d0 = rx0 - __shfl_sync(0xffffffffu, s0, c);
                    const double d1 = rx1 - __shfl_sync(0xffffffffu, s1, c);
                    const double d2 = rx2 - __shfl_sync(0xffffffffu, s2, c);
                    double k;
                    if constexpr (KID == SPD_K_RPY) k = rpy_entry(kp, d0, d1, d2, rc, __shfl_sync(0xffffffffu, sc, c));
                    else k = kval_sym<KID>(kp, d0 * d0 + d1 * d1 + d2 * d2);
                    if (sh && pc.tid0 + r0 + lane == pc.sid0 + c0 + c) k += shift;
                    kv[c] = (c < cn && lane < nr) ? k : 0.0;
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
                butterfly32(kv);
                if (lane < cn) tp[warp * nb + c0 + lane] = kv[0];
            }
        }
        if (lane < nr) scratch[pc.fwd + r0 + lane] = acc;
    }
    if (trn) {
        group_bar(1 + grp, SY_NW * 32);
        const int nw = min(SY_NW, (pc.nr + 31) >> 5);
        for (int c = gt; c < nb; c += SY_NW * 32) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += tp[w * nb + c];
            scratch[pc.trn + c] = t;
        }
        group_bar(1 + grp, SY_NW * 32);
    }
}

// one (output node, 32-row tile) by a whole CTA (long lists): warp w sums the w-th of
// PH_W contiguous slices of the list, the slice sums are added in warp order.  red: PH_W*32.
// sum of the partials con[cb, ce) over the 32 rows of a tile (lane = row) into a[4]
// (entry c goes to a[(c - cb) & 3]: the order of the sums is fixed).  The descriptors
// of 16 entries are fetched by 16 lanes at once and broadcast, then the 16 partial
// loads are all in flight before the first add (one round trip per 16 entries).
__device__ __forceinline__ void gather_range(const SymContrib* __restrict__ con, int cb, int ce,
                                             const double* __restrict__ scratch, double (&a)[4]) {
    const int lane = threadIdx.x & 31;
    for (int c0 = cb; c0 < ce; c0 += 16) {
        const int nc = min(16, ce - c0);
        int64_t mo = 0;
        int ml = 0;
        if (lane < nc) { const SymContrib q = con[c0 + lane]; mo = q.soff; ml = q.len; }
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int64_t o = __shfl_sync(0xffffffffu, mo, u);
            const int l = __shfl_sync(0xffffffffu, ml, u);
            v[u] = (u < nc && lane < l) ? ldv(scratch + o + lane) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) a[(c0 - cb + u) & 3] += v[u];
    }
}

// one (output node, 32-row tile) by a CTA: warp w sums a contiguous slice of the list,
// the slices are added in warp order
__device__ __forceinline__ void gather_item_cta(const SymGNode& g, const SymContrib* __restrict__ con,
                                                const SymVecsOut& yout, const double* __restrict__ scratch,
                                                double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int len = g.c1 - g.c0;
    const int cb = g.c0 + (int)((int64_t)len * warp / PH_W), ce = g.c0 + (int)((int64_t)len * (warp + 1) / PH_W);
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    gather_range(con, cb, ce, scratch, a);
    red[warp * 32 + lane] = (a[0] + a[1]) + (a[2] + a[3]);
    __syncthreads();
    if (warp == 0 && lane < g.n) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < PH_W; ++w) sum += red[w * 32 + lane];
        yout.p[g.slot][g.off + lane] = sum;
    }
    __syncthreads();
}

// one (output node, 32-row tile) by ONE warp: y[tile] = sum of its partials in list
// order (lane = row; four independent accumulators over c = 4q + u, added in u order)
__device__ __forceinline__ void gather_item_warp(const SymGNode& g, const SymContrib* __restrict__ con,
                                                 const SymVecsOut& yout, const double* __restrict__ scratch) {
    const int lane = threadIdx.x & 31;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    gather_range(con, g.c0, g.c1, scratch, a);
    if (lane < g.n) yout.p[g.slot][g.off + lane] = (a[0] + a[1]) + (a[2] + a[3]);
}

// ================================================================= HSS solve levels (reading R12)
constexpr int HS_CC = 32, HS_MT = 10;   // m <= 32 * HS_MT

struct HsNode {
    const double* F;   // m x m lower triangular (ld m): S_i^{-1} (leaf) / F_i^{-1}
    const double* P;   // m x r (ld m): S_i^{-T} V_i / F_i^{-T} Vbar'_i
    int m, r;
    const double* in;  // up/root: w (m) ; down: u0 (m)
    const double* xh;  // down: coarse solution (r)
    const double* zhi; // down: zh of the up sweep (r)
    double* u;         // up: u0 (m)
    double* zh;        // up: P^T w (r), input of the next level
    double* zh2;       // up: copy of zh kept for the down sweep
    double* out;       // down/root: result (m)
};

// Each HSS level is split into independent 32-output work items (every output of a
// level depends only on the level's input vectors), so even the top levels with one
// or two nodes spread over many SMs:
//   kind 0  u0[rt] = F[rt rows, :] w             (lower: columns <= row)
//   kind 1  zh[ct] = P[:, ct cols]^T w           (also written to zh2)
//   kind 2  out[rt] = (F^T u)[rt] + P[rt rows, :] (xh - zh)   (root: zh, xh absent)
//   kind 3  out[rt] = F[rt rows, :] w   (F full m x m: the dense top-of-tree operator)
struct HsItem { int node, kind, tile; };

// sm: m + r + PH_W * 32 doubles
__device__ __forceinline__ void hss_item(const HsNode* __restrict__ nodes, const HsItem& it, double* sm) {
    const HsNode nd = nodes[it.node];
    const int m = nd.m, r = nd.r;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* w = sm;                      // m: input vector (w or u0)
    double* dv = sm + m;                 // r: xh - zh (kind 2)
    double* red = dv + r;                // PH_W * 32
    for (int i = threadIdx.x; i < m; i += PH_T) w[i] = ldv(nd.in + i);
    if (it.kind == 2 && nd.xh)
        for (int j = threadIdx.x; j < r; j += PH_T) dv[j] = ldv(nd.xh + j) - ldv(nd.zhi + j);
    __syncthreads();
    if (it.kind == 0 || it.kind == 3) {
        const bool lower = it.kind == 0;
        const int i = it.tile * 32 + lane;
        const int ncc = lower ? min((m + 31) >> 5, it.tile + 1) : (m + 31) >> 5;   // lower: columns <= rows
        double acc = 0.0;
        for (int cc = warp; cc < ncc; cc += PH_W) {
            const int j0 = cc * 32;
            const int j1 = lower ? min(min(m, j0 + 32), i + 1) : min(m, j0 + 32);
            const double* p = nd.F + i + (size_t)j0 * m;
            double v[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = (i < m && j0 + c < j1) ? __ldg(p + (size_t)c * m) : 0.0;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int c = 0; c < 32; c += 2) {
                a0 += v[c] * (j0 + c < j1 ? w[j0 + c] : 0.0);
                a1 += v[c + 1] * (j0 + c + 1 < j1 ? w[j0 + c + 1] : 0.0);
            }
            acc += a0 + a1;
        }
        red[warp * 32 + lane] = acc;
        __syncthreads();
        if (warp == 0 && i < m) {
            double sum = 0.0;
#pragma unroll
            for (int q = 0; q < PH_W; ++q) sum += red[q * 32 + lane];
            if (lower) nd.u[i] = sum;
            else nd.out[i] = sum;
        }
    } else if (it.kind == 1) {
        for (int q = 0; q < 4; ++q) {
            const int j = it.tile * 32 + warp * 4 + q;
            if (j >= r) break;
            const double* p = nd.P + (size_t)j * m;
            double v[HS_MT];
#pragma unroll
            for (int t = 0; t < HS_MT; ++t) {
                const int i = t * 32 + lane;
                v[t] = i < m ? __ldg(p + i) : 0.0;
            }
#pragma unroll
            for (int t = 0; t < HS_MT; ++t) {            // multiplies after all loads (in-order issue)
                const int i = t * 32 + lane;
                v[t] *= i < m ? w[i] : 0.0;
            }
            double sum = 0.0;
#pragma unroll
            for (int t = 0; t < HS_MT; ++t) sum += v[t];
            sum = warp_sum(sum);
            if (lane == 0) { nd.zh[j] = sum; nd.zh2[j] = sum; }
        }
    } else {
        // (F^T u)[i] for the tile's 32 outputs: warp takes 4 columns, lanes over rows k >= i
        for (int q = 0; q < 4; ++q) {
            const int i = it.tile * 32 + warp * 4 + q;
            double sum = 0.0;
            if (i < m) {
                const double* p = nd.F + (size_t)i * m;
                double v[HS_MT];
#pragma unroll
                for (int t = 0; t < HS_MT; ++t) {
                    const int k = t * 32 + lane;
                    v[t] = (k >= i && k < m) ? __ldg(p + k) : 0.0;
                }
#pragma unroll
                for (int t = 0; t < HS_MT; ++t) {
                    const int k = t * 32 + lane;
                    v[t] *= (k >= i && k < m) ? w[k] : 0.0;
                }
#pragma unroll
                for (int t = 0; t < HS_MT; ++t) sum += v[t];
                sum = warp_sum(sum);
            }
            if (lane == 0) red[warp * 4 + q] = sum;             // red[0 .. 32): F^T u of the tile
        }
        // (P d)[i]: lane = row, warps split the r columns (contiguous slices, added in warp order)
        const int i = it.tile * 32 + lane;
        double acc = 0.0;
        if (nd.xh && i < m) {
            const int jb = (int)((int64_t)r * warp / PH_W), je = (int)((int64_t)r * (warp + 1) / PH_W);
            int j = jb;
            for (; j + 8 <= je; j += 8) {               // 8 loads in flight, then the FMAs
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldg(nd.P + i + (size_t)(j + u) * m);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc += v[u] * dv[j + u];
            }
            for (; j < je; ++j) acc += __ldg(nd.P + i + (size_t)j * m) * dv[j];
        }
        red[32 + warp * 32 + lane] = acc;
        __syncthreads();
        if (warp == 0 && i < m) {
            double sum = red[lane];
#pragma unroll
            for (int q = 0; q < PH_W; ++q) sum += red[32 + q * 32 + lane];
            nd.out[i] = sum;
        }
    }
    __syncthreads();
}
__host__ __device__ inline int hss_item_smem_doubles(int mmax, int rmax) { return mmax + rmax + (PH_W + 1) * 32; }

// The same items (kinds 0, 1, 2) computed by ONE WARP each, with no shared memory and
// no CTA barrier: the inputs come through L2 (ldv) in 32-element chunks broadcast by
// shuffles, every chunk issues 32 independent loads per lane, and the warps of a CTA
// work on different items -- a level's items all run at once instead of a few per CTA
// in sequence (the CTA form is latency-bound on the per-item barriers and input fills).
// Summation order is fixed per output (chunk order), so results are reproducible.
// Warp items win when a level has many items (each warp walks its item's chunks in
// sequence; measured on C2: leaf levels 2x faster), CTA items when it has few (the 8
// warps split one item's chunks): warp form for >= 3.4 items per CTA slot (2 per SM).
inline bool hss_phase_uses_warps(int mode, size_t nitems, int nsm) {
    return mode != 3 && (double)nitems >= 3.4 * 2 * nsm;
}
__device__ __forceinline__ void hss_item_warp(const HsNode* __restrict__ nodes, const HsItem& it) {
    const HsNode nd = nodes[it.node];
    const int m = nd.m, r = nd.r;
    const int lane = threadIdx.x & 31;
    if (it.kind == 0) {                               // u0[i] = sum_{j <= i} F[i, j] w[j]
        const int i = it.tile * 32 + lane;
        double a0 = 0.0, a1 = 0.0;
        for (int cc = 0; cc <= it.tile; ++cc) {
            const int j0 = cc * 32;
            const double wj = j0 + lane < m ? ldv(nd.in + j0 + lane) : 0.0;
            const double* p = nd.F + i + (size_t)j0 * m;
            double v[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = (i < m && j0 + c <= i) ? __ldg(p + (size_t)c * m) : 0.0;
#pragma unroll
            for (int c = 0; c < 32; c += 2) {
                a0 += v[c] * __shfl_sync(0xffffffffu, wj, c);
                a1 += v[c + 1] * __shfl_sync(0xffffffffu, wj, c + 1);
            }
        }
        if (i < m) nd.u[i] = a0 + a1;
    } else if (it.kind == 1) {                        // zh[c] = sum_k P[k, c] w[k], 32 columns
        const int c0 = it.tile * 32, cn = min(32, r - c0);
        double acc = 0.0;
        for (int k0 = 0; k0 < m; k0 += 32) {
            const int k = k0 + lane;
            const double wk = k < m ? ldv(nd.in + k) : 0.0;
            const double* p = nd.P + k + (size_t)c0 * m;
            double v[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = (k < m && c < cn) ? __ldg(p + (size_t)c * m) : 0.0;
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] *= wk;      // after ALL loads: in-order issue
            butterfly32(v);
            acc += v[0];
        }
        if (lane < cn) { nd.zh[c0 + lane] = acc; nd.zh2[c0 + lane] = acc; }
    } else {                                          // out[i] = (F^T u)[i] + (P (xh - zh))[i]
        const int c0 = it.tile * 32, cn = min(32, m - c0);
        double acc = 0.0;                             // lane c: sum_{k >= c0 + c} F[k, c0 + c] u[k]
        for (int k0 = c0; k0 < m; k0 += 32) {
            const int k = k0 + lane;
            const double uk = k < m ? ldv(nd.in + k) : 0.0;
            const double* p = nd.F + k + (size_t)c0 * m;
            double v[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = (k < m && c < cn && k >= c0 + c) ? __ldg(p + (size_t)c * m) : 0.0;
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] *= uk;
            butterfly32(v);
            acc += v[0];
        }
        const int i = c0 + lane;                      // lane = row i: + sum_j P[i, j] (xh - zh)[j]
        if (nd.xh) {
            double b0 = 0.0, b1 = 0.0;
            for (int j0 = 0; j0 < r; j0 += 32) {
                const double dj = j0 + lane < r ? ldv(nd.xh + j0 + lane) - ldv(nd.zhi + j0 + lane) : 0.0;
                const double* p = nd.P + i + (size_t)j0 * m;
                double v[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) v[c] = (i < m && j0 + c < r) ? __ldg(p + (size_t)c * m) : 0.0;
#pragma unroll
                for (int c = 0; c < 32; c += 2) {
                    b0 += v[c] * __shfl_sync(0xffffffffu, dj, c);
                    b1 += v[c + 1] * __shfl_sync(0xffffffffu, dj, c + 1);
                }
            }
            acc += b0 + b1;
        }
        if (i < m) nd.out[i] = acc;
    }
}

// ================================================================= host-side plans (work items)
std::vector<std::vector<BasisItem>> basis_up_plan(const spd_h2_s* h, const double* x, const std::vector<double*>& xh,
                                                  int top, int* ncmax_out, std::vector<double>* bytes,
                                                  const BasisFilter* f = nullptr);
std::vector<std::vector<BasisItem>> basis_down_plan(const spd_h2_s* h, const std::vector<double*>& yh, int top,
                                                    double* y, int* smax_out, std::vector<double>* bytes,
                                                    const BasisFilter* f = nullptr);
// level: the tree level of an up (mode 0) / down (mode 1) phase, 0 for the root / top
// operator; idx: each node's index within its level (the subtree-sharded solve keeps the
// owned ones)
struct HsPhase { int mode = 0; std::vector<HsNode> nodes; std::vector<HsItem> items; int level = 0; std::vector<int> idx; };
std::vector<HsPhase> bj_solve_plan(const spd_hss_s* H, const double* b, double* x, double* z);
std::vector<HsPhase> hss_solve_plan(const spd_hss_s* H, const double* b, double* x, double* z,
                                    const std::vector<double*>& zl, const std::vector<double*>& zs,
                                    const std::vector<double*>& ub);

}  // namespace spd
