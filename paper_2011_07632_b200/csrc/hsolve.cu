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
#include <algorithm>

namespace spd {

constexpr int HS_T = 512, HS_W = HS_T / 32, HS_CC = 32, HS_MT = 10;   // m <= 32 * HS_MT

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

// Partial products of y = A x (y[i] = sum_j A[i + j ld] x[j], j < n, j <= i if lower).
// Work items are (32-row tile, 32-column chunk); a warp issues the chunk's 32 loads
// at once (lane = row, coalesced 256-byte lines) and writes part[cc * m + i].
__device__ void cta_gemv_n_items(const double* __restrict__ A, int ld, int m, int n, bool lower, const double* x,
                                 double* part) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nrt = (m + 31) >> 5, ncc = (n + HS_CC - 1) / HS_CC;
    for (int item = warp; item < nrt * ncc; item += HS_W) {
        const int rt = item / ncc, cc = item - rt * ncc;
        const int i = rt * 32 + lane, j0 = cc * HS_CC;
        if (lower && j0 > rt * 32 + 31) continue;
        int j1 = min(n, j0 + HS_CC);
        if (lower) j1 = min(j1, i + 1);
        const int cn = j1 - j0;
        const double* p = A + i + (size_t)j0 * ld;
        double v[HS_CC];
        if (i < m && cn == HS_CC) {
#pragma unroll
            for (int c = 0; c < HS_CC; ++c) v[c] = __ldg(p + (size_t)c * ld);
        } else {
#pragma unroll
            for (int c = 0; c < HS_CC; ++c) v[c] = (i < m && c < cn) ? __ldg(p + (size_t)c * ld) : 0.0;
        }
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int c = 0; c < HS_CC; c += 2) {
            a0 += v[c] * (c < cn ? x[j0 + c] : 0.0);           // x past n is not initialised
            a1 += v[c + 1] * (c + 1 < cn ? x[j0 + c + 1] : 0.0);
        }
        if (i < m) part[cc * m + i] = a0 + a1;
    }
}
// (after a barrier) the row sums of the partials, in chunk order
__device__ __forceinline__ double cta_gemv_n_row(const double* part, int m, int n, bool lower, int i) {
    const int ncc = (n + HS_CC - 1) / HS_CC;
    const int ccmax = lower ? min(ncc, ((i | 31) / HS_CC) + 1) : ncc;
    double s = 0.0;
    for (int cc = 0; cc < ccmax; ++cc) s += part[cc * m + i];
    return s;
}

// y[j] = sum_i A[i + j ld] x[i] over i < m (i >= j if lower), j < n.  A warp takes
// two columns at a time and issues all their loads (<= 2 * HS_MT per lane) at once.
__device__ void cta_gemv_t(const double* __restrict__ A, int ld, int m, int n, bool lower, const double* x,
                           double* y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = 2 * warp; j < n; j += 2 * HS_W) {
        const bool two = j + 1 < n;
        const double* p0 = A + (size_t)j * ld;
        const double* p1 = p0 + ld;
        const int lo0 = lower ? j : 0, lo1 = lower ? j + 1 : 0;
        double v0[HS_MT], v1[HS_MT];
#pragma unroll
        for (int q = 0; q < HS_MT; ++q) {
            const int i = q * 32 + lane;
            v0[q] = (i < m && i >= lo0) ? __ldg(p0 + i) : 0.0;
            v1[q] = (two && i < m && i >= lo1) ? __ldg(p1 + i) : 0.0;
        }
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int q = 0; q < HS_MT; ++q) {
            const int i = q * 32 + lane;
            const double xv = i < m ? x[i] : 0.0;
            s0 += v0[q] * xv;
            s1 += v1[q] * xv;
        }
        s0 = warp_sum(s0);
        s1 = warp_sum(s1);
        if (lane == 0) {
            y[j] = s0;
            if (two) y[j + 1] = s1;
        }
    }
}

// mode 0: up    u0 = F w ; zh = P^T w                      (writes u0, zh, zh2)
// mode 1: down  out = F^T u0 + P (xh - zh)
// mode 2: root  out = F^T (F w)
template <int MODE>
__global__ void __launch_bounds__(HS_T, 1) hss_level_kernel(const HsNode* __restrict__ nodes, int mmax) {
    extern __shared__ double sm[];
    const HsNode nd = nodes[blockIdx.x];
    const int m = nd.m, r = nd.r;
    double* w = sm;                        // mmax
    double* u = w + mmax;                  // mmax
    double* zh = u + mmax;                 // mmax (r <= m)
    double* part = zh + mmax;              // ceil(mmax/32) * mmax
    for (int i = threadIdx.x; i < m; i += HS_T) w[i] = nd.in[i];
    if (MODE == 1)
        for (int i = threadIdx.x; i < r; i += HS_T) zh[i] = nd.xh[i] - nd.zhi[i];
    __syncthreads();
    if (MODE == 0) {
        cta_gemv_n_items(nd.F, m, m, m, true, w, part);
        if (r > 0) cta_gemv_t(nd.P, m, m, r, false, w, zh);
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += HS_T) nd.u[i] = cta_gemv_n_row(part, m, m, true, i);
        for (int i = threadIdx.x; i < r; i += HS_T) { nd.zh[i] = zh[i]; nd.zh2[i] = zh[i]; }
    } else if (MODE == 1) {
        if (r > 0) cta_gemv_n_items(nd.P, m, m, r, false, zh, part);
        cta_gemv_t(nd.F, m, m, m, true, w, u);
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += HS_T)
            nd.out[i] = u[i] + (r > 0 ? cta_gemv_n_row(part, m, r, false, i) : 0.0);
    } else {
        cta_gemv_n_items(nd.F, m, m, m, true, w, part);
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += HS_T) u[i] = cta_gemv_n_row(part, m, m, true, i);
        __syncthreads();
        cta_gemv_t(nd.F, m, m, m, true, u, nd.out);
    }
}

static size_t level_smem(int mmax) {
    return sizeof(double) * ((size_t)3 * mmax + (size_t)((mmax + HS_CC - 1) / HS_CC) * mmax);
}

template <int MODE>
static void launch_level(cudaStream_t s, const std::vector<HsNode>& nodes) {
    if (nodes.empty()) return;
    int mmax = 1;
    double by = 0;
    for (auto& n : nodes) {
        mmax = std::max(mmax, n.m);
        by += 8.0 * (0.5 * n.m * (n.m + 1) * (MODE == 2 ? 2 : 1) + (double)n.m * n.r + 2.0 * n.m + 2.0 * n.r);
    }
    const size_t smem = level_smem(mmax);
    SPD_REQUIRE(mmax <= 32 * HS_MT, "hss_solve: node too large for the fused k=1 solve");
    if (smem > 48 * 1024)
        SPD_CUDA(cudaFuncSetAttribute(hss_level_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DevArray<HsNode> dn(s, nodes);
    ProfScope prof(s, "hss_solve_vec", 0, by);
    hss_level_kernel<MODE><<<(unsigned)nodes.size(), HS_T, smem, s>>>(dn.p, mmax);
    SPD_LAUNCH();
}

// x = H^{-1} b for one vector (tree order, contiguous), L >= 2.  zl[l]: level-l
// coefficients (zh up, xh down), zs[l]: zh kept for the down sweep, ub[l]: u0 of the
// level-l nodes at their children's offsets (leaves: u0 in z).
void hss_solve_vec(spd_hss_s* H, const double* b, double* x, double* z, const std::vector<double*>& zl,
                   const std::vector<double*>& zs, const std::vector<double*>& ub, cudaStream_t s) {
    const spd_h2_s* h = H->h2;
    const TreeH& t = h->tree;
    const int L = t.L;
    const HssLevel& l1 = H->lv[1];
    std::vector<HsNode> nodes;
    for (int a = 0; a < l1.count; ++a) {
        const int64_t off = t.begin[l1.first + a];
        if (!l1.m[a]) continue;
        nodes.push_back({l1.Finv.p + l1.F_off[a], l1.P.p + l1.V_off[a], l1.m[a], l1.rank[a], b + off, nullptr, nullptr,
                         z + off, zl[1] + l1.off[a], zs[1] + l1.off[a], nullptr});
    }
    launch_level<0>(s, nodes);
    for (int l = 2; l < L; ++l) {
        const HssLevel& lv = H->lv[l];
        const HssLevel& pv = H->lv[l - 1];
        nodes.clear();
        for (int a = 0; a < lv.count; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            if (!lv.m[a]) continue;
            nodes.push_back({lv.Finv.p + lv.F_off[a], lv.P.p + lv.V_off[a], lv.m[a], lv.rank[a], zl[l - 1] + pv.off[c1],
                             nullptr, nullptr, ub[l] + pv.off[c1], zl[l] + lv.off[a], zs[l] + lv.off[a], nullptr});
        }
        launch_level<0>(s, nodes);
    }
    {
        const HssLevel& rt = H->lv[L];
        if (rt.m[0]) {
            nodes.assign(1, {rt.Finv.p, nullptr, rt.m[0], 0, zl[L - 1], nullptr, nullptr, nullptr, nullptr, nullptr,
                             zl[L - 1]});
            launch_level<2>(s, nodes);
        }
    }
    for (int l = L - 1; l >= 2; --l) {
        const HssLevel& lv = H->lv[l];
        const HssLevel& pv = H->lv[l - 1];
        nodes.clear();
        for (int a = 0; a < lv.count; ++a) {
            const int c1 = 2 * (lv.first + a) + 1 - pv.first;
            if (!lv.m[a]) continue;
            nodes.push_back({lv.Finv.p + lv.F_off[a], lv.P.p + lv.V_off[a], lv.m[a], lv.rank[a], ub[l] + pv.off[c1],
                             zl[l] + lv.off[a], zs[l] + lv.off[a], nullptr, nullptr, nullptr, zl[l - 1] + pv.off[c1]});
        }
        launch_level<1>(s, nodes);
    }
    nodes.clear();
    for (int a = 0; a < l1.count; ++a) {
        const int64_t off = t.begin[l1.first + a];
        if (!l1.m[a]) continue;
        nodes.push_back({l1.Finv.p + l1.F_off[a], l1.P.p + l1.V_off[a], l1.m[a], l1.rank[a], z + off,
                         zl[1] + l1.off[a], zs[1] + l1.off[a], nullptr, nullptr, nullptr, x + off});
    }
    launch_level<1>(s, nodes);
}

}  // namespace spd
