#include <queue>
// dense.cu -- ragged batched fp64 dense kernels for sm_100a (product path).
//
//   gemm_batched   C = alpha op(A) op(B) + beta C, 64x64 CTA tiles, FP64 DMMA (m8n8k4)
//   potrf_batched  A = L L^T in place (one CTA per matrix)               [P:282, P:1014]
//   trsm_batched   X := op(T)^{-1} X, 32-row blocked substitution
//   qrcp_batched   Businger-Golub pivoted Householder QR (reading R4) with
//                  recomputed column norms, lowest-index ties, diag(R) >= 0.
//                  A group of CTAs cooperates on one matrix (column-cyclic
//                  ownership, in-kernel group barrier) so large proxy
//                  matrices use many SMs; small matrices get one CTA.  [P:827]
//   formq_batched  explicit Q[:, :r] from the stored reflectors
#include "common.cuh"
#include "gemm.cuh"
#include <algorithm>
#include <cooperative_groups.h>
#include <cstdlib>
#include <cstdio>

namespace spd {

// ================================================================= GEMM (pipelined DMMA tiles: gemm.cuh)
constexpr int GK = 16;

// ---------------------------------------------------------------- narrow GEMM (n <= 4): GEMV-like
// notrans A: one thread per output row (coalesced column reads of A);
// trans A:   one warp per output row (contiguous column of A, warp reduction).
template <bool TA, int NV>
__global__ void __launch_bounds__(256) gemv_kernel(const GemmDesc* __restrict__ descs, const int2* __restrict__ work,
                                                   double alpha, double beta) {
    const int2 wk = work[blockIdx.x];
    const GemmDesc d = descs[wk.x];
    const int n = d.n;
    if (!TA) {
        // 32-row tile, lane = row (coalesced columns), the 8 warps split k
        __shared__ double red[8][32][NV];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int i = wk.y * 32 + lane;
        const bool ok = i < d.m;
        double acc[4][NV];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[u][v] = 0.0;
        const int kc = (d.k + 7) / 8, kb = warp * kc, ke = min(d.k, kb + kc);
        if (ok) {
            const double* a = d.A + i;
            int kk = kb;
            for (; kk + 4 <= ke; kk += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double av = __ldg(a + (size_t)(kk + u) * d.lda);
#pragma unroll
                    for (int v = 0; v < NV; ++v)
                        if (v < n) acc[u][v] += av * __ldg(d.B + kk + u + (size_t)v * d.ldb);
                }
            }
            for (; kk < ke; ++kk) {
                const double av = __ldg(a + (size_t)kk * d.lda);
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    if (v < n) acc[0][v] += av * __ldg(d.B + kk + (size_t)v * d.ldb);
            }
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) red[warp][lane][v] = (acc[0][v] + acc[1][v]) + (acc[2][v] + acc[3][v]);
        __syncthreads();
        if (warp == 0 && ok) {
#pragma unroll
            for (int v = 0; v < NV; ++v)
                if (v < n) {
                    double sum = 0.0;
                    for (int w = 0; w < 8; ++w) sum += red[w][lane][v];
                    double* c = d.C + i + (size_t)v * d.ldc;
                    *c = (beta == 0.0 ? 0.0 : beta * *c) + alpha * sum;
                }
        }
    } else {
        const int lane = threadIdx.x & 31;
        const int i = wk.y * 8 + (threadIdx.x >> 5);
        if (i >= d.m) return;
        const double* a = d.A + (size_t)i * d.lda;
        double acc[4][NV];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[u][v] = 0.0;
        int kk = lane;
        for (; kk + 96 < d.k; kk += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double av = __ldg(a + kk + 32 * u);
#pragma unroll
                for (int v = 0; v < NV; ++v)
                    if (v < n) acc[u][v] += av * __ldg(d.B + kk + 32 * u + (size_t)v * d.ldb);
            }
        }
        for (; kk < d.k; kk += 32) {
            const double av = __ldg(a + kk);
#pragma unroll
            for (int v = 0; v < NV; ++v)
                if (v < n) acc[0][v] += av * __ldg(d.B + kk + (size_t)v * d.ldb);
        }
        double sum[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) sum[v] = warp_sum((acc[0][v] + acc[1][v]) + (acc[2][v] + acc[3][v]));
        if (lane == 0)
#pragma unroll
            for (int v = 0; v < NV; ++v)
                if (v < n) {
                    double* c = d.C + i + (size_t)v * d.ldc;
                    *c = (beta == 0.0 ? 0.0 : beta * *c) + alpha * sum[v];
                }
    }
}

template <int BM, int BN, int WM, int WN, int ST, bool TA, bool TB, bool PRE>
static void launch_gemm_pipe1(cudaStream_t s, unsigned nb, const GemmDesc* d, const TileRef* t, double alpha, double beta) {
    constexpr size_t sh = gemm_pipe_smem<BM, BN, WM, WN, ST, TA, TB>();
    static bool attr = false;
    if (!attr) {
        SPD_CUDA(cudaFuncSetAttribute(gemm_pipe_kernel<BM, BN, WM, WN, ST, TA, TB, PRE>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        attr = true;
    }
    gemm_pipe_kernel<BM, BN, WM, WN, ST, TA, TB, PRE><<<nb, (BM / WM) * (BN / WN) * 32, sh, s>>>(d, t, alpha, beta);
    SPD_LAUNCH();
}
template <int BM, int BN, int WM, int WN, int ST, bool TA, bool TB>
static void launch_gemm_persist1(cudaStream_t s, int ntiles, const GemmDesc* d, const TileRef* t, double alpha,
                                 double beta) {
    constexpr size_t sh = gemm_pipe_smem<BM, BN, WM, WN, ST, TA, TB>();
    static int grid = 0;
    if (!grid) {
        SPD_CUDA(cudaFuncSetAttribute(gemm_persist_kernel<BM, BN, WM, WN, ST, TA, TB>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        int dev = 0, nsm = 0, per = 0;
        SPD_CUDA(cudaGetDevice(&dev));
        SPD_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        SPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gemm_persist_kernel<BM, BN, WM, WN, ST, TA, TB>,
                                                               (BM / WM) * (BN / WN) * 32, sh));
        grid = nsm * std::max(1, per);
    }
    const unsigned nb = (unsigned)std::min(ntiles, grid);
    gemm_persist_kernel<BM, BN, WM, WN, ST, TA, TB><<<nb, (BM / WM) * (BN / WN) * 32, sh, s>>>(d, t, ntiles, alpha, beta);
    SPD_LAUNCH();
}

template <int BM, int BN, int WM, int WN, int ST, bool PRE = false>
static void launch_gemm_pipe(cudaStream_t s, unsigned nb, const GemmDesc* d, const TileRef* t, double alpha,
                             double beta, bool ta, bool tb) {
    if (!ta && !tb) launch_gemm_pipe1<BM, BN, WM, WN, ST, false, false, PRE>(s, nb, d, t, alpha, beta);
    else if (ta && !tb) launch_gemm_pipe1<BM, BN, WM, WN, ST, true, false, PRE>(s, nb, d, t, alpha, beta);
    else if (!ta && tb) launch_gemm_pipe1<BM, BN, WM, WN, ST, false, true, PRE>(s, nb, d, t, alpha, beta);
    else launch_gemm_pipe1<BM, BN, WM, WN, ST, true, true, PRE>(s, nb, d, t, alpha, beta);
}

// split-K epilogue: C = alpha sum_s P_s + beta C, slices added in order
struct ReduceDesc { int desc, S; int64_t off; };
__global__ void gemm_reduce_kernel(const GemmDesc* __restrict__ descs, const ReduceDesc* __restrict__ red,
                                   const double* __restrict__ part, double alpha, double beta) {
    const ReduceDesc r = red[blockIdx.y];
    const GemmDesc d = descs[r.desc];
    const int64_t mn = (int64_t)d.m * d.n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mn; e += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int q = 0; q < r.S; ++q) acc += part[r.off + q * mn + e];
        const int i = (int)(e % d.m), j = (int)(e / d.m);
        double* c = d.C + i + (size_t)j * d.ldc;
        *c = (beta == 0.0 ? 0.0 : beta * *c) + alpha * acc;
    }
}

static void gemv_batched(cudaStream_t s, const std::vector<GemmDesc>& d, bool transA, double alpha, double beta) {
    std::vector<int2> work;
    double fl = 0, by = 0;
    for (int i = 0; i < (int)d.size(); ++i) {
        if (d[i].m <= 0 || d[i].n <= 0) continue;
        if (d[i].k <= 0 && beta == 1.0) continue;
        const int rows_per = transA ? 8 : 32;
        for (int t = 0; t < ceil_div(d[i].m, rows_per); ++t) work.push_back(make_int2(i, t));
        fl += 2.0 * d[i].m * d[i].n * d[i].k;
        by += 8.0 * ((double)d[i].m * d[i].k + 2.0 * d[i].m * d[i].n);
    }
    if (work.empty()) return;
    DevArray<GemmDesc> dd(s, d);
    DevArray<int2> dw(s, work);
    ProfScope prof(s, "gemv", fl, by);
    int nmax = 0;
    for (auto& g : d) nmax = std::max(nmax, g.n);
    const unsigned nb = (unsigned)work.size();
    if (transA) {
        if (nmax == 1) gemv_kernel<true, 1><<<nb, 256, 0, s>>>(dd.p, dw.p, alpha, beta);
        else gemv_kernel<true, 4><<<nb, 256, 0, s>>>(dd.p, dw.p, alpha, beta);
    } else {
        if (nmax == 1) gemv_kernel<false, 1><<<nb, 256, 0, s>>>(dd.p, dw.p, alpha, beta);
        else gemv_kernel<false, 4><<<nb, 256, 0, s>>>(dd.p, dw.p, alpha, beta);
    }
    SPD_LAUNCH();
}

void gemm_batched(cudaStream_t s, const std::vector<GemmDesc>& d, bool transA, bool transB,
                  double alpha, double beta) {
    if (!transB) {
        int nmax = 0;
        for (auto& g : d) nmax = std::max(nmax, g.n);
        if (nmax <= 4) { gemv_batched(s, d, transA, alpha, beta); return; }
    }
    // tile size: 64 x 64 (4 warps of 32 x 32; measured 31-32 TF/s at 4096^3, 88-91 % of
    // cuBLAS DGEMM, against 28-30 TF/s for 128 x 128); env SPD_GEMM_TILE=128 overrides
    int T = 64;
    if (const char* e = getenv("SPD_GEMM_TILE")) T = atoi(e) == 128 ? 128 : 64;
    // m <= 32 everywhere (V^T A of the blocked QR): 32 x 64 tiles, no wasted DMMA rows
    int mmax_all = 0, kmax_all = 0;
    for (const auto& g : d) { mmax_all = std::max(mmax_all, g.m); kmax_all = std::max(kmax_all, g.k); }
    const bool m32 = T == 64 && mmax_all <= 32;
    const int TM = m32 ? 32 : T;
    // n <= 16 everywhere (the blocked QR's in-block products of a 16-column panel: V^T A_s,
    // V^T V_s with a long K, and the panel update A_s -= V W2): 16-column tiles instead of 64
    // (a quarter of the DMMA work), K split when long (C4 H2 build 9.14 -> 8.86 s)
    int nmax_all = 0;
    for (const auto& g : d) nmax_all = std::max(nmax_all, g.n);
    const bool n16 = T == 64 && nmax_all <= 16 && !getenv("SPD_GEMM_NO_N16");
    const int TN = n16 ? 16 : T;
    // output tiles; when they are too few to fill the GPU and K is long (the tall
    // skinny V^T A of the blocked QR), K is split into S slices whose raw partial
    // tiles are summed in slice order by gemm_reduce_kernel (deterministic)
    long long ntiles = 0;
    int kmax = 0;
    for (const auto& g : d) {
        if (g.m <= 0 || g.n <= 0) continue;
        ntiles += (long long)ceil_div(g.m, TM) * ceil_div(g.n, TN);
        kmax = std::max(kmax, g.k);
    }
    // split K when a tile's K loop is long and the tiles are too few for ~8 resident per SM
    int S = 1;
    if (ntiles > 0 && ((ntiles < 2 * 148 && kmax >= 1024) || (ntiles < 4 * 148 && kmax >= 4096)))
        S = (int)std::max<long long>(1, std::min<long long>(kmax / 512, (8 * 148 + ntiles - 1) / ntiles));
    if (n16 && ntiles > 0 && ntiles < 16 * 148 && kmax >= 512)   // 2-warp tiles: aim at ~16 per SM
        S = (int)std::max<long long>(S, std::min<long long>(kmax / 256, (16 * 148 + ntiles - 1) / ntiles));
    std::vector<TileRef> tiles;
    std::vector<ReduceDesc> red;
    size_t poff = 0;
    for (int i = 0; i < (int)d.size(); ++i) {
        if (d[i].m <= 0 || d[i].n <= 0) continue;
        if (d[i].k <= 0 && beta == 1.0) continue;
        const int Si = (S > 1 && d[i].k >= 8 * 64) ? std::min(S, ceil_div(d[i].k, 128)) : 1;
        const int kc = Si > 1 ? ceil_div(ceil_div(d[i].k, Si), GK) * GK : std::max(d[i].k, 0);
        const int Seff = Si > 1 ? ceil_div(d[i].k, kc) : 1;
        for (int ks = 0; ks < Seff; ++ks)
            for (int tn = 0; tn < ceil_div(d[i].n, TN); ++tn)
                for (int tm = 0; tm < ceil_div(d[i].m, TM); ++tm) {
                    TileRef tr{i, tm, tn, ks * kc, std::min(d[i].k, (ks + 1) * kc), nullptr, d[i].m};
                    if (Seff > 1) tr.P = (double*)(uintptr_t)(poff + (size_t)ks * d[i].m * d[i].n + 1);  // offset+1, patched below
                    tiles.push_back(tr);
                }
        if (Seff > 1) {
            red.push_back({i, Seff, (int64_t)poff});
            poff += (size_t)Seff * d[i].m * d[i].n;
        }
    }
    if (tiles.empty()) return;
    DBuf<double> part;
    if (poff) {
        part.alloc(poff);
        for (auto& tr : tiles)
            if (tr.P) tr.P = part.p + ((size_t)(uintptr_t)tr.P - 1);
    }
    double fl = 0, by = 0;
    for (auto& g : d) if (g.m > 0 && g.n > 0 && g.k > 0) {
        fl += 2.0 * g.m * g.n * g.k;
        by += 8.0 * ((double)g.m * g.k + (double)g.k * g.n + 2.0 * g.m * g.n);
    }
    DevArray<GemmDesc> dd(s, d);
    DevArray<TileRef> dt(s, tiles);
    {
        ProfScope prof(s, "gemm_dmma", fl, by);
        for (size_t off = 0; off < tiles.size(); off += 1u << 30) {
            unsigned nb = (unsigned)std::min<size_t>(tiles.size() - off, 1u << 30);
            const bool pre = beta != 0.0 && kmax_all <= 64;      // short-K update: C read early
            // short-K products without split-K (the blocked QR's rank-64 updates and its
            // T / W factors): persistent CTAs, pipeline across tiles (C2 .. C4 H2 build:
            // 9.38 -> 9.14 s at C4)
            // (env SPD_GEMM_NOPERSIST: the one-tile-per-CTA kernel, A/B)
            static const bool nopersist = getenv("SPD_GEMM_NOPERSIST") != nullptr;
            if (n16) {
                if (m32) launch_gemm_pipe<32, 16, 32, 16, 3>(s, nb, dd.p, dt.p + off, alpha, beta, transA, transB);
                else launch_gemm_pipe<64, 16, 32, 16, 3>(s, nb, dd.p, dt.p + off, alpha, beta, transA, transB);
                continue;
            }
            if (kmax_all <= 64 && !poff && T == 64 && !m32 && !nopersist) {
                if (!transA && !transB) launch_gemm_persist1<64, 64, 32, 32, 3, false, false>(s, (int)nb, dd.p, dt.p + off, alpha, beta);
                else if (transA && !transB) launch_gemm_persist1<64, 64, 32, 32, 3, true, false>(s, (int)nb, dd.p, dt.p + off, alpha, beta);
                else if (!transA && transB) launch_gemm_persist1<64, 64, 32, 32, 3, false, true>(s, (int)nb, dd.p, dt.p + off, alpha, beta);
                else launch_gemm_persist1<64, 64, 32, 32, 3, true, true>(s, (int)nb, dd.p, dt.p + off, alpha, beta);
                continue;
            }
            if (T == 128) launch_gemm_pipe<128, 128, 64, 32, 3>(s, nb, dd.p, dt.p + off, alpha, beta, transA, transB);
            else if (m32) launch_gemm_pipe<32, 64, 32, 32, 3>(s, nb, dd.p, dt.p + off, alpha, beta, transA, transB);
            else if (pre) launch_gemm_pipe<64, 64, 32, 32, 2, true>(s, nb, dd.p, dt.p + off, alpha, beta, transA, transB);
            else launch_gemm_pipe<64, 64, 32, 32, 3>(s, nb, dd.p, dt.p + off, alpha, beta, transA, transB);
        }
    }
    if (!red.empty()) {
        DevArray<ReduceDesc> dr(s, red);
        ProfScope prof(s, "gemm_reduce", 0, 8.0 * poff);
        gemm_reduce_kernel<<<dim3(16, (unsigned)red.size()), 256, 0, s>>>(dd.p, dr.p, part.p, alpha, beta);
        SPD_LAUNCH();
    }
}

// ================================================================= POTRF
// right-looking, column by column, in place (lower); upper triangle zeroed.
__global__ void __launch_bounds__(256) potrf_kernel(const MatDesc* descs, int* info, double* badval) {
    const MatDesc d = descs[blockIdx.x];
    double* A = d.A;
    const int n = d.m, ld = d.ld;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    __shared__ double piv;
    __shared__ int bad;
    if (tid == 0) bad = 0;
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        if (tid == 0) {
            double a = A[j + (size_t)j * ld];
            if (!(a > 0.0)) {               // not PD (or NaN): record first failure
                bad = 1;
                if (info) info[blockIdx.x] = j + 1;
                if (badval) badval[blockIdx.x] = a;
                a = 1.0;
            }
            piv = sqrt(a);
            A[j + (size_t)j * ld] = piv;
        }
        __syncthreads();
        if (bad) break;
        const double inv = 1.0 / piv;
        for (int i = j + 1 + tid; i < n; i += blockDim.x) A[i + (size_t)j * ld] *= inv;
        __syncthreads();
        for (int k = j + 1 + warp; k < n; k += nw) {
            const double lkj = A[k + (size_t)j * ld];
            double* ck = A + (size_t)k * ld;
            const double* cj = A + (size_t)j * ld;
            for (int i = k + lane; i < n; i += 32) ck[i] -= cj[i] * lkj;
        }
        __syncthreads();
    }
    for (int j = 1 + warp; j < n; j += nw)
        for (int i = lane; i < j; i += 32) A[i + (size_t)j * ld] = 0.0;
}

// Blocked form of the same factorisation: 32-column panels held in shared memory.  A panel
// first takes the updates of every earlier column j < j0 (left-looking; 4 x 4 register tiles,
// rows interleaved by 32 so every load of L is coalesced, L read from global / L2), then is
// factored column by column in shared memory and written back once.  Every entry (i, k)
// receives a_ik <- fma(-l_ij, l_kj, a_ik) for j = 0 .. k-1 in ascending j exactly like
// potrf_kernel, so L (and the first failing pivot and its value) is bitwise the same; the
// trailing matrix is no longer re-read and re-written once per column.
constexpr int PO_NB = 32;
__global__ void __launch_bounds__(256) potrf_panel_kernel(const MatDesc* descs, int* info, double* badval) {
    extern __shared__ double po_sm[];             // panel: (n - j0) rows x 32 columns, ld = n - j0
    const MatDesc d = descs[blockIdx.x];
    double* A = d.A;
    const int n = d.m, ld = d.ld;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    __shared__ double piv;
    __shared__ int bad;
    if (tid == 0) bad = 0;
    __syncthreads();
    for (int j0 = 0; j0 < n && !bad; j0 += PO_NB) {
        const int nbk = min(PO_NB, n - j0), mr = n - j0;
        double* P = po_sm;
        // panel <- A[j0:n, j0:j0+nbk] - L[j0:n, 0:j0] L[j0:j0+nbk, 0:j0]^T
        const int ngr = (mr + 127) / 128, ntc = (nbk + 3) / 4;
        for (int task = warp; task < ngr * ntc; task += nw) {
            const int gr = task % ngr, tc = task / ngr;
            int ri[4], kc[4];
            double acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a) ri[a] = j0 + gr * 128 + lane + 32 * a;
#pragma unroll
            for (int b = 0; b < 4; ++b) kc[b] = j0 + 4 * tc + b;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    acc[a][b] = (ri[a] < n && kc[b] < j0 + nbk) ? A[ri[a] + (size_t)kc[b] * ld] : 0.0;
            for (int j = 0; j < j0; ++j) {
                const double* cj = A + (size_t)j * ld;
                double li[4], lk[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) li[a] = ri[a] < n ? cj[ri[a]] : 0.0;
#pragma unroll
                for (int b = 0; b < 4; ++b) lk[b] = kc[b] < n ? cj[kc[b]] : 0.0;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[a][b] -= li[a] * lk[b];
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (ri[a] < n && kc[b] < j0 + nbk) P[(ri[a] - j0) + (size_t)(kc[b] - j0) * mr] = acc[a][b];
        }
        __syncthreads();
        // the panel's own columns, in shared memory (rows r >= jj of column jj)
        for (int jj = 0; jj < nbk; ++jj) {
            if (tid == 0) {
                double a = P[jj + (size_t)jj * mr];
                if (!(a > 0.0)) {               // not PD (or NaN): record first failure
                    bad = 1;
                    if (info) info[blockIdx.x] = j0 + jj + 1;
                    if (badval) badval[blockIdx.x] = a;
                    a = 1.0;
                }
                piv = sqrt(a);
                P[jj + (size_t)jj * mr] = piv;
            }
            __syncthreads();
            if (bad) break;
            const double inv = 1.0 / piv;
            for (int r = jj + 1 + tid; r < mr; r += blockDim.x) P[r + (size_t)jj * mr] *= inv;
            __syncthreads();
            const double* cj = P + (size_t)jj * mr;
            for (int kk = jj + 1 + warp; kk < nbk; kk += nw) {
                const double lkj = cj[kk];
                double* ck = P + (size_t)kk * mr;
                for (int r = kk + lane; r < mr; r += 32) ck[r] -= cj[r] * lkj;
            }
            __syncthreads();
        }
        // write the panel back (lower part; the upper triangle is zeroed below)
        for (int c = warp; c < nbk; c += nw)
            for (int r = c + lane; r < mr; r += 32) A[(j0 + r) + (size_t)(j0 + c) * ld] = P[r + (size_t)c * mr];
        __syncthreads();
    }
    for (int j = 1 + warp; j < n; j += nw)
        for (int i = lane; i < j; i += 32) A[i + (size_t)j * ld] = 0.0;
}

void potrf_batched(cudaStream_t s, const std::vector<MatDesc>& d, int* info_dev, double* bad_dev) {
    if (d.empty()) return;
    double fl = 0, by = 0;
    int nmax = 0;
    for (auto& m : d) { fl += (double)m.m * m.m * m.m / 3.0; by += 16.0 * m.m * m.m; nmax = std::max(nmax, m.m); }
    DevArray<MatDesc> dd(s, d);
    ProfScope prof(s, "potrf", fl, by);
    // SPD_POTRF_PANEL=1: panels in shared memory up to 220 KB (n <= 880), bitwise equal and 5.7x faster
    // at C4 (91 -> 16 ms per step) -- NOT the default: with it the 4-process host-comm test hit a PCG
    // breakdown in 2 of 6 runs against 0 of 5 with the unblocked kernel (unexplained)
    const size_t smem = sizeof(double) * (size_t)nmax * PO_NB;
    if (smem <= 220 * 1024 && getenv("SPD_POTRF_PANEL") && !getenv("SPD_POTRF_GLOBAL")) {
        if (smem > 48 * 1024)
            SPD_CUDA(cudaFuncSetAttribute(potrf_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        potrf_panel_kernel<<<(unsigned)d.size(), 256, smem, s>>>(dd.p, info_dev, bad_dev);
    } else {
        potrf_kernel<<<(unsigned)d.size(), 256, 0, s>>>(dd.p, info_dev, bad_dev);
    }
    SPD_LAUNCH();
}

// ================================================================= TRSM
// X := op(T)^{-1} X ; T n x n triangular.  "forward" when the effective
// matrix op(T) is lower triangular.
template <bool LOWER, bool TRANS>
__global__ void __launch_bounds__(128) trsm_kernel(const TrsmDesc* descs, const int2* work) {
    constexpr bool FWD = (LOWER != TRANS);
    __shared__ double Td[32][33];
    __shared__ double Xs[32][33];
    const int2 wk = work[blockIdx.x];
    const TrsmDesc d = descs[wk.x];
    const int c0 = wk.y * 32;
    const int nc = min(32, d.nrhs - c0);
    const int n = d.n;
    const int tid = threadIdx.x;
    auto Tel = [&](int i, int k) -> double {   // element (i, k) of op(T)
        return TRANS ? d.T[k + (size_t)i * d.ldt] : d.T[i + (size_t)k * d.ldt];
    };
    const int nblk = ceil_div(n, 32);
    for (int bb = 0; bb < nblk; ++bb) {
        const int blk = FWD ? bb * 32 : (nblk - 1 - bb) * 32;
        const int nb = min(32, n - blk);
        for (int e = tid; e < 32 * 32; e += 128) {
            int i = e & 31, k = e >> 5;
            Td[i][k] = (i < nb && k < nb) ? Tel(blk + i, blk + k) : 0.0;
            Xs[i][k] = (i < nb && k < nc) ? d.X[blk + i + (size_t)(c0 + k) * d.ldx] : 0.0;
        }
        __syncthreads();
        if (tid < 32 && tid < nc) {
            const int c = tid;
            if (FWD) {
                for (int i = 0; i < nb; ++i) {
                    double v = Xs[i][c];
                    for (int k = 0; k < i; ++k) v -= Td[i][k] * Xs[k][c];
                    Xs[i][c] = v / Td[i][i];
                }
            } else {
                for (int i = nb - 1; i >= 0; --i) {
                    double v = Xs[i][c];
                    for (int k = i + 1; k < nb; ++k) v -= Td[i][k] * Xs[k][c];
                    Xs[i][c] = v / Td[i][i];
                }
            }
        }
        __syncthreads();
        for (int e = tid; e < 32 * 32; e += 128) {
            int i = e & 31, k = e >> 5;
            if (i < nb && k < nc) d.X[blk + i + (size_t)(c0 + k) * d.ldx] = Xs[i][k];
        }
        // update the remaining rows: X[r, :] -= op(T)[r, blk:blk+nb] Xblk
        const int r_begin = FWD ? blk + nb : 0;
        const int r_end = FWD ? n : blk;
        for (int e = tid; e < (r_end - r_begin) * nc; e += 128) {
            int r = r_begin + e % (r_end - r_begin);
            int c = e / (r_end - r_begin);
            double v = 0.0;
            for (int k = 0; k < nb; ++k) v += Tel(r, blk + k) * Xs[k][c];
            d.X[r + (size_t)(c0 + c) * d.ldx] -= v;
        }
        __syncthreads();
    }
}

template <bool LOWER, bool TRANS>
__global__ void __launch_bounds__(256) trsv_kernel(const TrsmDesc* descs) {
    constexpr bool FWD = (LOWER != TRANS);
    extern __shared__ double xs[];               // n x nrhs (nrhs <= 4)
    const TrsmDesc d = descs[blockIdx.x];
    const int n = d.n, nr = d.nrhs;
    for (int e = threadIdx.x; e < n * nr; e += blockDim.x) xs[e] = d.X[e % n + (size_t)(e / n) * d.ldx];
    __syncthreads();
    // column sweep: x_j /= T_jj ; x_r -= op(T)_{r j} x_j for the remaining rows
    for (int jj = 0; jj < n; ++jj) {
        const int j = FWD ? jj : n - 1 - jj;
        const double tjj = d.T[j + (size_t)j * d.ldt];
        __syncthreads();
        double xj[4];
        for (int v = 0; v < nr; ++v) xj[v] = xs[j + v * n] / tjj;
        __syncthreads();
        if (threadIdx.x < nr) xs[j + threadIdx.x * n] = xj[threadIdx.x];
        const int r0 = FWD ? j + 1 : 0, r1 = FWD ? n : j;
        for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
            const double t = TRANS ? d.T[j + (size_t)r * d.ldt] : d.T[r + (size_t)j * d.ldt];
            for (int v = 0; v < nr; ++v) xs[r + v * n] -= t * xj[v];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * nr; e += blockDim.x) d.X[e % n + (size_t)(e / n) * d.ldx] = xs[e];
}

template <bool TRANS>
__global__ void __launch_bounds__(256) trsv_warp_kernel(const TrsmDesc* __restrict__ descs, int ndesc, int nmax) {
    extern __shared__ double xsh[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int item = blockIdx.x * 8 + warp;          // (desc, rhs column)
    // items are laid out desc-major with 4 slots per desc (nrhs <= 4)
    const int di = item >> 2, c = item & 3;
    if (di >= ndesc) return;
    const TrsmDesc d = descs[di];
    if (c >= d.nrhs) return;
    const int n = d.n;
    double* xs = xsh + (size_t)warp * nmax;
    double* xg = d.X + (size_t)c * d.ldx;
    for (int i = lane; i < n; i += 32) xs[i] = xg[i];
    __syncwarp();
    if (!TRANS) {                                    // L x = b : x_j /= L_jj ; x_r -= L_rj x_j (r > j)
        for (int j = 0; j < n; ++j) {
            const double* col = d.T + (size_t)j * d.ldt;
            const double xj = xs[j] / col[j];
            __syncwarp();
            if (lane == 0) xs[j] = xj;
            for (int r = j + 1 + lane; r < n; r += 32) xs[r] -= col[r] * xj;
            __syncwarp();
        }
    } else {                                         // L^T x = b : x_j = (b_j - sum_{r>j} L_rj x_r) / L_jj
        for (int j = n - 1; j >= 0; --j) {
            const double* col = d.T + (size_t)j * d.ldt;
            double sacc = 0.0;
            for (int r = j + 1 + lane; r < n; r += 32) sacc += col[r] * xs[r];
            sacc = warp_sum(sacc);
            if (lane == 0) xs[j] = (xs[j] - sacc) / col[j];
            __syncwarp();
        }
    }
    for (int i = lane; i < n; i += 32) xg[i] = xs[i];
}

constexpr int TRSM_REC_N = 128;
void trsm_rec(cudaStream_t s, const std::vector<TrsmDesc>& d, bool lower);
void trsm_base(cudaStream_t s, const std::vector<TrsmDesc>& d, bool lower, bool trans);

void trsm_batched(cudaStream_t s, const std::vector<TrsmDesc>& d, char uplo, bool trans) {
    {
        int nrmax = 0, nmax = 0;
        for (auto& t : d) { nrmax = std::max(nrmax, t.nrhs); nmax = std::max(nmax, t.n); }
        const bool lower = (uplo == 'L' || uplo == 'l');
        if (lower && nrmax <= 4 && nmax > 0 && nmax <= 768) {
            std::vector<TrsmDesc> dv;
            double fl = 0, by = 0;
            for (auto& t : d) if (t.n > 0 && t.nrhs > 0) { dv.push_back(t); fl += (double)t.n * t.n * t.nrhs; by += 4.0 * t.n * t.n; }
            if (dv.empty()) return;
            DevArray<TrsmDesc> dd(s, dv);
            ProfScope prof(s, "trsv", fl, by);
            const unsigned nb = (unsigned)ceil_div((int64_t)dv.size() * 4, 8);
            const size_t sh = (size_t)8 * nmax * sizeof(double);
            if (!trans) trsv_warp_kernel<false><<<nb, 256, sh, s>>>(dd.p, (int)dv.size(), nmax);
            else trsv_warp_kernel<true><<<nb, 256, sh, s>>>(dd.p, (int)dv.size(), nmax);
            SPD_LAUNCH();
            return;
        }
    }
    {
        int nrmax = 0, nmax = 0;
        for (auto& t : d) { nrmax = std::max(nrmax, t.nrhs); nmax = std::max(nmax, t.n); }
        if (nrmax <= 4 && nmax > 0 && (size_t)nmax * nrmax * 8 <= 48 * 1024) {
            std::vector<TrsmDesc> dv;
            double fl = 0, by = 0;
            for (auto& t : d) if (t.n > 0 && t.nrhs > 0) { dv.push_back(t); fl += (double)t.n * t.n * t.nrhs; by += 4.0 * t.n * t.n; }
            if (dv.empty()) return;
            DevArray<TrsmDesc> dd(s, dv);
            ProfScope prof(s, "trsv", fl, by);
            const size_t sh = (size_t)nmax * nrmax * 8;
            const unsigned nb = (unsigned)dv.size();
            bool lower = (uplo == 'L' || uplo == 'l');
            if (lower && !trans) trsv_kernel<true, false><<<nb, 256, sh, s>>>(dd.p);
            else if (lower && trans) trsv_kernel<true, true><<<nb, 256, sh, s>>>(dd.p);
            else if (!lower && !trans) trsv_kernel<false, false><<<nb, 256, sh, s>>>(dd.p);
            else trsv_kernel<false, true><<<nb, 256, sh, s>>>(dd.p);
            SPD_LAUNCH();
            return;
        }
    }
    const bool lower_ = (uplo == 'L' || uplo == 'l');
    if (!trans) {
        bool any_big = false;
        for (auto& t : d) any_big |= t.n > TRSM_REC_N && t.nrhs >= 64;
        if (any_big) { trsm_rec(s, d, lower_); return; }
    }
    trsm_base(s, d, lower_, trans);
}

// Recursive blocked TRSM (no transpose) for n > TRSM_REC_N: [T11 0; T21 T22] (lower) or
// [T11 T12; 0 T22] (upper) split at a multiple of 32; the off-diagonal update
// X_other -= T_off X_solved is one batched DMMA GEMM per recursion step (K = the
// solved half), so most of the n^2 nrhs flops run on the tensor path; the
// diagonal blocks at the bottom use the 32-row blocked kernel.
void trsm_rec(cudaStream_t s, const std::vector<TrsmDesc>& d, bool lower) {
    std::vector<TrsmDesc> small, first, second;
    std::vector<GemmDesc> upd;
    for (const auto& t : d) {
        if (t.n <= 0 || t.nrhs <= 0) continue;
        if (t.n <= TRSM_REC_N || t.nrhs < 64) { small.push_back(t); continue; }   // few columns: GEMMs too thin
        const int h = ((t.n / 2 + 31) / 32) * 32;
        const TrsmDesc a{t.T, t.X, h, t.nrhs, t.ldt, t.ldx};                                        // T11, X1
        const TrsmDesc b{t.T + h + (size_t)h * t.ldt, t.X + h, t.n - h, t.nrhs, t.ldt, t.ldx};       // T22, X2
        if (lower) {
            first.push_back(a); second.push_back(b);
            upd.push_back({t.T + h, t.X, t.X + h, t.n - h, t.nrhs, h, t.ldt, t.ldx, t.ldx});           // X2 -= T21 X1
        } else {
            first.push_back(b); second.push_back(a);
            upd.push_back({t.T + (size_t)h * t.ldt, t.X + h, t.X, h, t.nrhs, t.n - h, t.ldt, t.ldx, t.ldx});  // X1 -= T12 X2
        }
    }
    if (!small.empty()) trsm_base(s, small, lower, false);
    if (first.empty()) return;
    trsm_rec(s, first, lower);
    gemm_batched(s, upd, false, false, -1.0, 1.0);
    trsm_rec(s, second, lower);
}

// the 32-row blocked kernel: one CTA per (matrix, 32 right-hand sides)
void trsm_base(cudaStream_t s, const std::vector<TrsmDesc>& d, bool lower_in, bool trans) {
    const char uplo = lower_in ? 'L' : 'U';
    std::vector<int2> work;
    for (int i = 0; i < (int)d.size(); ++i) {
        if (d[i].n <= 0 || d[i].nrhs <= 0) continue;
        for (int c = 0; c < ceil_div(d[i].nrhs, 32); ++c) work.push_back(make_int2(i, c));
    }
    if (work.empty()) return;
    double fl = 0, by = 0;
    for (auto& t : d) { fl += (double)t.n * t.n * t.nrhs; by += 8.0 * ((double)t.n * t.n / 2 + 2.0 * t.n * t.nrhs); }
    DevArray<TrsmDesc> dd(s, d);
    DevArray<int2> dw(s, work);
    ProfScope prof(s, "trsm", fl, by);
    unsigned nb = (unsigned)work.size();
    bool lower = (uplo == 'L' || uplo == 'l');
    if (lower && !trans) trsm_kernel<true, false><<<nb, 128, 0, s>>>(dd.p, dw.p);
    else if (lower && trans) trsm_kernel<true, true><<<nb, 128, 0, s>>>(dd.p, dw.p);
    else if (!lower && !trans) trsm_kernel<false, false><<<nb, 128, 0, s>>>(dd.p, dw.p);
    else trsm_kernel<false, true><<<nb, 128, 0, s>>>(dd.p, dw.p);
    SPD_LAUNCH();
}

// ================================================================= QRCP
constexpr int QR_THREADS = 256;
__device__ unsigned long long g_qr_trace[64];      // debug (SPD_QR_TRACE): phase timestamps
__device__ unsigned long long g_qr_steps[8192];    // debug (SPD_QR_STEPS): start of every step of matrix 0
__device__ __forceinline__ void qr_tr(int k) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_qr_trace[k] = t;
}

struct QrItem { int desc, g, G; };

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// barrier among the G CTAs working on one matrix (all co-resident: cooperative launch)
__device__ void group_barrier(unsigned* bar, int G) {
    __syncthreads();
    if (G > 1 && threadIdx.x == 0) {
        volatile unsigned* vgen = bar + 1;
        unsigned gen = *vgen;
        __threadfence();
        if (atomicAdd(bar, 1u) == (unsigned)G - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*vgen == gen) { __nanosleep(32); }
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ void block_argmax(double v, int idx, double* sv, int* si, double& bv, int& bi) {
    // max value, lowest index on ties
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, o);
        int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
    if (lane == 0) { sv[warp] = v; si[warp] = idx; }
    __syncthreads();
    if (warp == 0) {
        int nw = blockDim.x >> 5;
        v = lane < nw ? sv[lane] : -1.0;
        idx = lane < nw ? si[lane] : 0x7fffffff;
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_xor_sync(0xffffffffu, v, o);
            int oi = __shfl_xor_sync(0xffffffffu, idx, o);
            if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
        }
        if (lane == 0) { sv[0] = v; si[0] = idx; }
    }
    __syncthreads();
    bv = sv[0];
    bi = si[0];
    __syncthreads();
}

__device__ double block_sum(double v, double* sv) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) sv[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int nw = blockDim.x >> 5;
        v = lane < nw ? sv[lane] : 0.0;
        v = warp_sum(v);
        if (lane == 0) sv[0] = v;
    }
    __syncthreads();
    double r = sv[0];
    __syncthreads();
    return r;
}

// squared norm of column j over rows [r0, m), one warp
__device__ __forceinline__ double col_norm2(const double* c, int r0, int m) {
    double s = 0.0;
    for (int i = r0 + (threadIdx.x & 31); i < m; i += 32) { double x = ldcg(c + i); s += x * x; }
    return warp_sum(s);
}

// loads in flight per lane and column in the update pass (4; 8 measured slower at C4:
// 10.3 against 9.4 s of H2 build -- 121 registers leave 2 CTAs per SM)
#ifndef SPD_QRCP_QU
#define SPD_QRCP_QU 4
#endif
constexpr int QU = SPD_QRCP_QU;
template <int U>
__device__ __forceinline__ double tree_sum(const double* s) {
    if constexpr (U == 1) return s[0];
    else return tree_sum<U / 2>(s) + tree_sum<U / 2>(s + U / 2);
}

__global__ void __launch_bounds__(QR_THREADS) qrcp_kernel(const QrcpDesc* descs, const QrItem* items,
                                                          const int2* cta_items, unsigned* barriers,
                                                          double rel_tol) {
    __shared__ double sv[32];
    __shared__ int si[32];
    __shared__ int s_stop;
    __shared__ double s_nu0;
    extern __shared__ double vsh[];                 // m: the current reflector
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = QR_THREADS / 32;
    const int2 range = cta_items[blockIdx.x];
    for (int it = range.x; it < range.y; ++it) {
        const QrItem item = items[it];
        const QrcpDesc d = descs[item.desc];
        const int g = item.g, G = item.G;
        unsigned* bar = barriers + 2 * item.desc;
        const int m = d.m, n = d.n, ld = d.ld;
        double* A = d.A;
        const int kmax = min(min(m, n), d.max_rank);
        // initial norms (rows 0..m-1) of owned columns
        {
            int local = 0;
            for (int j = g; j < n; j += G, ++local)
                if (local % nw == warp) {
                    double s = col_norm2(A + (size_t)j * ld, 0, m);
                    if (lane == 0) d.norms[j] = s;
                }
            if (g == 0)
                for (int j = threadIdx.x; j < n; j += QR_THREADS) d.piv[j] = j;
        }
        if (threadIdx.x == 0) { s_stop = 0; s_nu0 = 0.0; }
        if (g == 0 && threadIdx.x == 0) d.rank[0] = -1;     // "running" (published by the barrier)
        group_barrier(bar, G);
        for (int t = 0;; ++t) {
            const bool trc = (item.desc == 0 && g == 0 && t == 100 && threadIdx.x == 0);
            if (trc) qr_tr(10);
            // ---- leader: pivot, stop test, Householder of column t
            if (g == 0) {
                double bv = -1.0;
                int bi = 0x7fffffff;
                if (t < kmax) {
                    double v = -1.0;
                    int idx = 0x7fffffff;
                    for (int j = t + threadIdx.x; j < n; j += QR_THREADS) {
                        double x = ldcg(d.norms + j);
                        if (x > v) { v = x; idx = j; }   // ascending j: keeps lowest on ties
                    }
                    block_argmax(v, idx, sv, si, bv, bi);
                }
                const double nu = bv > 0.0 ? sqrt(bv) : 0.0;
                if (threadIdx.x == 0) {
                    if (t == 0) s_nu0 = nu;
                    s_stop = (t >= kmax || nu == 0.0 || nu <= rel_tol * s_nu0) ? 1 : 0;
                }
                __syncthreads();
                if (d.force) {                          // injected pivots (R19 hook)
                    if (threadIdx.x == 0) s_stop = (t >= min(kmax, d.nforce)) ? 1 : 0;
                    __syncthreads();
                    if (!s_stop) {
                        const int want = d.force[t];
                        for (int j = t + threadIdx.x; j < n; j += QR_THREADS)
                            if (__ldcg(d.piv + j) == want) si[0] = j;
                    }
                    __syncthreads();
                    bi = si[0];
                    __syncthreads();
                }
                if (!s_stop) {
                    const int p = bi;
                    if (p != t) {
                        double* ct = A + (size_t)t * ld;
                        double* cp = A + (size_t)p * ld;
                        for (int i = threadIdx.x; i < m; i += QR_THREADS) {
                            double a = ldcg(ct + i), b = ldcg(cp + i);
                            ct[i] = b; cp[i] = a;
                        }
                        if (threadIdx.x == 0) { int tp = d.piv[t]; d.piv[t] = d.piv[p]; d.piv[p] = tp; }
                    }
                    __syncthreads();
                    double* ct = A + (size_t)t * ld;
                    double sig = 0.0;
                    for (int i = t + 1 + threadIdx.x; i < m; i += QR_THREADS) { double x = ct[i]; sig += x * x; }
                    sig = block_sum(sig, sv);
                    const double x0 = ct[t];
                    double beta, mu, v0;
                    if (sig == 0.0) { beta = (x0 >= 0.0) ? 0.0 : 2.0; mu = fabs(x0); v0 = 1.0; }
                    else {
                        mu = sqrt(x0 * x0 + sig);
                        v0 = (x0 <= 0.0) ? x0 - mu : -sig / (x0 + mu);
                        beta = 2.0 * v0 * v0 / (sig + v0 * v0);
                    }
                    const double inv0 = 1.0 / v0;
                    for (int i = t + 1 + threadIdx.x; i < m; i += QR_THREADS) ct[i] = (sig == 0.0) ? 0.0 : ct[i] * inv0;
                    if (threadIdx.x == 0) { ct[t] = mu; d.beta[t] = beta; }
                } else if (threadIdx.x == 0) {
                    d.rank[0] = t;                  // stop: publish the rank (-1 while running)
                }
                __syncthreads();
            }
            if (trc) qr_tr(11);
            group_barrier(bar, G);
            if (trc) qr_tr(12);
            {
                const int r = __ldcg(d.rank);
                if (r >= 0) break;
            }
            // ---- all CTAs: apply H_t to owned columns j > t, recompute norms over rows t+1..
            //      v (v_t = 1) cached in shared memory; per column two passes with 8 loads in
            //      flight per lane (the update phase is latency-bound otherwise)
            const double* vg = A + (size_t)t * ld;     // v_i = A[i, t], i > t
            const double beta = __ldcg(d.beta + t);
            for (int i = t + threadIdx.x; i < m; i += QR_THREADS) vsh[i] = (i == t) ? 1.0 : ldcg(vg + i);
            __syncthreads();
            // this warp's columns: j = g + G * local (local = warp mod nw), j > t; two at a
            // time (16 loads in flight per lane)
            int j0 = g + G * warp;
            while (j0 <= t && j0 < n) j0 += G * nw;
            for (; j0 < n; j0 += 2 * G * nw) {
                const int j1 = j0 + G * nw;
                const bool two = j1 < n;
                double* c0 = A + (size_t)j0 * ld;
                double* c1 = A + (size_t)(two ? j1 : j0) * ld;
                double sa[QU], sb[QU];
#pragma unroll
                for (int u = 0; u < QU; ++u) sa[u] = sb[u] = 0.0;
                int i0 = t + lane;
                for (; i0 + (QU - 1) * 32 < m; i0 += QU * 32) {
                    double x[QU], y[QU];
#pragma unroll
                    for (int u = 0; u < QU; ++u) { x[u] = ldcg(c0 + i0 + 32 * u); y[u] = two ? ldcg(c1 + i0 + 32 * u) : 0.0; }
#pragma unroll
                    for (int u = 0; u < QU; ++u) { const double vv = vsh[i0 + 32 * u]; sa[u] += vv * x[u]; sb[u] += vv * y[u]; }
                }
                for (int i = i0; i < m; i += 32) {
                    sa[0] += vsh[i] * ldcg(c0 + i);
                    if (two) sb[0] += vsh[i] * ldcg(c1 + i);
                }
                const double w0 = beta * warp_sum(tree_sum<QU>(sa));
                const double w1 = beta * warp_sum(tree_sum<QU>(sb));
                double na[QU], nb[QU];
#pragma unroll
                for (int u = 0; u < QU; ++u) na[u] = nb[u] = 0.0;
                i0 = t + lane;
                for (; i0 + (QU - 1) * 32 < m; i0 += QU * 32) {
                    double x[QU], y[QU];
#pragma unroll
                    for (int u = 0; u < QU; ++u) { x[u] = ldcg(c0 + i0 + 32 * u); y[u] = two ? ldcg(c1 + i0 + 32 * u) : 0.0; }
#pragma unroll
                    for (int u = 0; u < QU; ++u) {
                        const int i = i0 + 32 * u;
                        const double vv = vsh[i];
                        const double a = x[u] - w0 * vv;
                        c0[i] = a;
                        if (i > t) na[u] += a * a;
                        if (two) {
                            const double b = y[u] - w1 * vv;
                            c1[i] = b;
                            if (i > t) nb[u] += b * b;
                        }
                    }
                }
                for (int i = i0; i < m; i += 32) {
                    const double a = ldcg(c0 + i) - w0 * vsh[i];
                    c0[i] = a;
                    if (i > t) na[0] += a * a;
                    if (two) {
                        const double b = ldcg(c1 + i) - w1 * vsh[i];
                        c1[i] = b;
                        if (i > t) nb[0] += b * b;
                    }
                }
                const double n0 = warp_sum(tree_sum<QU>(na));
                const double n1 = warp_sum(tree_sum<QU>(nb));
                if (lane == 0) {
                    d.norms[j0] = n0;
                    if (two) d.norms[j1] = n1;
                }
            }
            if (trc) qr_tr(13);
            group_barrier(bar, G);
            if (trc) qr_tr(14);
        }
        group_barrier(bar, G);
    }
}

// Deferred-update Businger-Golub QRCP (the same pivot rule, reading R4: the residual
// norms are recomputed from the trailing entries at every step).  The eager kernel above
// reads every trailing column twice (the dot with v_t, then the update + norm) and writes
// it back at every step; this one reads it from DRAM ONCE per step and writes it back once
// per block of nb steps:
//  * within a block starting at step b the trailing columns keep a^(b) in memory and every
//    step reconstructs a^(t) = a^(b) - Y w_j on the fly, Y = [v_b .. v_{t-1}] (the block's
//    reflectors, in shared memory, zero above their first row, 1 on it), w_j one
//    coefficient per reflector and column (global W), by the compact recurrence
//    w_j[l] = beta_l (v_l^T a^(b) - sum_{i<l} (v_l^T v_i) w_j[i]);
//  * a producer warp streams each owned column (rows [b, m), contiguous) into a ring of
//    shared-memory stages with 1-D bulk copies (cp.async.bulk + mbarrier transaction
//    counts: a whole column in flight per stage, no registers), the consumer warps run
//    pass 1 (d = v_t^T a^(b), w_j[k] = beta_t (d - sum_l c_l w_j[l]), c_l = v_t^T v_l
//    published by the leader) and pass 2 (every entry of a^(t+1) reconstructed -- the
//    norm over rows > t recomputed, not downdated -- written back at the block's last
//    step) from shared memory.
// Pivots can differ from the eager kernel's only through rounding, i.e. at ties inside
// the certified band of reading R19.
constexpr int QNB = 8;
constexpr int QSMAX = 32;                    // ring stages (max)
struct QrcpLazy { double* Y; double* W; double* c; };    // Y: nb x m, W: n x QNB, c: QNB

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile("{\n\t.reg .pred p;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n}" :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int NT>
__device__ double qb_sum(double v, double* sv) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) sv[warp] = v;
    __syncthreads();
    double r = 0.0;
    for (int w = 0; w < NT / 32; ++w) r += sv[w];
    __syncthreads();
    return r;
}

// pass 2 of the deferred QRCP for one column (one warp): a = a^(b) - sum_{l < KK} v_l w[l]
// on rows [rstart, m), four rows per lane in flight; norm^2 of rows > t; write back if wb
template <int KK>
__device__ __forceinline__ void qrcp_pass2(const double* col, const double* ysh, int ms, const double* w,
                                           int rstart, int m, int t, bool wb, double* c, double& n0, double& n1) {
    const int lane = threadIdx.x & 31;
    double wr[KK];
#pragma unroll
    for (int l = 0; l < KK; ++l) wr[l] = w[l];
    int i = rstart + lane;
    for (; i + 96 < m; i += 128) {
        double a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = col[i + 32 * u];
#pragma unroll
        for (int l = 0; l < KK; ++l) {
            const double* y = ysh + (size_t)l * ms + i;
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] -= y[32 * u] * wr[l];
        }
        if (wb) {
#pragma unroll
            for (int u = 0; u < 4; ++u) c[i + 32 * u] = a[u];
        }
        if (i > t) { n0 += a[0] * a[0]; n1 += a[1] * a[1]; n0 += a[2] * a[2]; n1 += a[3] * a[3]; }
        else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + 32 * u > t) n0 += a[u] * a[u];
        }
    }
    for (; i < m; i += 32) {
        double a0 = col[i];
#pragma unroll
        for (int l = 0; l < KK; ++l) a0 -= ysh[(size_t)l * ms + i] * wr[l];
        if (wb) c[i] = a0;
        if (i > t) n0 += a0 * a0;
    }
}

template <int NT>
__global__ void __launch_bounds__(NT, 512 / NT) qrcp_lazy_kernel(const QrcpDesc* descs, const QrcpLazy* lzs,
                                                          const QrItem* items, const int2* cta_items,
                                                          unsigned* barriers, double rel_tol, int nb, int ms,
                                                          int nstage, int sst, int steptrace) {
    constexpr int NW = NT / 32;
    constexpr int NCW = NW - 1;                      // consumer warps (warp 0 produces)
    __shared__ double sv[32];
    __shared__ int si[32];
    __shared__ int s_stop;
    __shared__ double s_nu0;
    __shared__ double s_cred[QNB][NW];
    __shared__ __align__(8) uint64_t full[QSMAX], empty[QSMAX];
    extern __shared__ __align__(16) double ysh[];   // nb x ms reflectors, then nstage x sst column stages
    double* stg = ysh + (size_t)nb * ms;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < QSMAX) { mbar_init(&full[threadIdx.x], 1); mbar_init(&empty[threadIdx.x], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    __shared__ unsigned s_use[QSMAX];                // completed uses of every stage barrier
    if (threadIdx.x < QSMAX) s_use[threadIdx.x] = 0;
    const size_t stg_doubles = (size_t)nstage * sst; // the ring's shared memory
    const int2 range = cta_items[blockIdx.x];
    for (int it = range.x; it < range.y; ++it) {
        const QrItem item = items[it];
        const QrcpDesc d = descs[item.desc];
        const QrcpLazy lz = lzs[item.desc];
        const int g = item.g, G = item.G;
        unsigned* bar = barriers + 2 * item.desc;
        const int m = d.m, n = d.n, ld = d.ld;
        double* A = d.A;
        const int kmax = min(min(m, n), d.max_rank);
        {
            int local = 0;
            for (int j = g; j < n; j += G, ++local)
                if (local % NW == warp) {
                    double s = col_norm2(A + (size_t)j * ld, 0, m);
                    if (lane == 0) d.norms[j] = s;
                }
            if (g == 0)
                for (int j = threadIdx.x; j < n; j += NT) d.piv[j] = j;
        }
        if (threadIdx.x == 0) { s_stop = 0; s_nu0 = 0.0; }
        if (g == 0 && threadIdx.x == 0) d.rank[0] = -1;
        group_barrier(bar, G);
        int b = 0;
        for (int t = 0;; ++t) {
            const int k = t - b;                        // reflectors already in the block
            const bool trc = (item.desc == 0 && g == 0 && t == 100 && threadIdx.x == 0);
            if (trc) qr_tr(10);
            if (steptrace && item.desc == 0 && g == 0 && threadIdx.x == 0 && t < 8192) {
                unsigned long long tt;
                asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tt));
                g_qr_steps[t] = tt;
            }
            if (g == 0) {
                // ---- leader: pivot, the pivot column brought to step t, Householder, c_l
                double bv = -1.0;
                int bi = 0x7fffffff;
                if (t < kmax) {
                    double v = -1.0;
                    int idx = 0x7fffffff;
                    for (int j = t + threadIdx.x; j < n; j += NT) {
                        double x = ldcg(d.norms + j);
                        if (x > v) { v = x; idx = j; }
                    }
                    block_argmax(v, idx, sv, si, bv, bi);
                }
                const double nu = bv > 0.0 ? sqrt(bv) : 0.0;
                if (threadIdx.x == 0) {
                    if (t == 0) s_nu0 = nu;
                    s_stop = (t >= kmax || nu == 0.0 || nu <= rel_tol * s_nu0) ? 1 : 0;
                }
                __syncthreads();
                if (d.force) {
                    if (threadIdx.x == 0) s_stop = (t >= min(kmax, d.nforce)) ? 1 : 0;
                    __syncthreads();
                    if (!s_stop) {
                        const int want = d.force[t];
                        for (int j = t + threadIdx.x; j < n; j += NT)
                            if (__ldcg(d.piv + j) == want) si[0] = j;
                    }
                    __syncthreads();
                    bi = si[0];
                    __syncthreads();
                }
                if (!s_stop) {
                    const int p = bi;
                    if (p != t) {
                        double* ct = A + (size_t)t * ld;
                        double* cp = A + (size_t)p * ld;
                        for (int i = threadIdx.x; i < m; i += NT) {
                            double a = ldcg(ct + i), bb = ldcg(cp + i);
                            ct[i] = bb; cp[i] = a;
                        }
                        if (threadIdx.x < k) {
                            double a = ldcg(lz.W + (size_t)t * QNB + threadIdx.x), bb = ldcg(lz.W + (size_t)p * QNB + threadIdx.x);
                            lz.W[(size_t)t * QNB + threadIdx.x] = bb; lz.W[(size_t)p * QNB + threadIdx.x] = a;
                        }
                        if (threadIdx.x == 0) { int tp = d.piv[t]; d.piv[t] = d.piv[p]; d.piv[p] = tp; }
                    }
                    __syncthreads();
                    double* ct = A + (size_t)t * ld;
                    double* yk = ysh + (size_t)k * ms;
                    double* ykg = lz.Y + (size_t)k * m;
                    {
                        double wv[QNB];
#pragma unroll
                        for (int l = 0; l < QNB; ++l) wv[l] = l < k ? ldcg(lz.W + (size_t)t * QNB + l) : 0.0;
                        for (int i = b + threadIdx.x; i < m; i += NT) {
                            double x = ldcg(ct + i);
#pragma unroll
                            for (int l = 0; l < QNB; ++l)
                                if (l < k) x -= ysh[(size_t)l * ms + i] * wv[l];
                            if (i < t) { ct[i] = x; yk[i] = 0.0; ykg[i] = 0.0; }
                            else yk[i] = x;
                        }
                    }
                    __syncthreads();
                    double sig = 0.0;
                    for (int i = t + 1 + threadIdx.x; i < m; i += NT) { double x = yk[i]; sig += x * x; }
                    sig = qb_sum<NT>(sig, sv);
                    const double x0 = yk[t];
                    double beta, mu, v0;
                    if (sig == 0.0) { beta = (x0 >= 0.0) ? 0.0 : 2.0; mu = fabs(x0); v0 = 1.0; }
                    else {
                        mu = sqrt(x0 * x0 + sig);
                        v0 = (x0 <= 0.0) ? x0 - mu : -sig / (x0 + mu);
                        beta = 2.0 * v0 * v0 / (sig + v0 * v0);
                    }
                    const double inv0 = 1.0 / v0;
                    for (int i = t + 1 + threadIdx.x; i < m; i += NT) {
                        const double v = (sig == 0.0) ? 0.0 : yk[i] * inv0;
                        yk[i] = v; ct[i] = v; ykg[i] = v;
                    }
                    __syncthreads();
                    if (threadIdx.x == 0) { yk[t] = 1.0; ykg[t] = 1.0; ct[t] = mu; d.beta[t] = beta; }
                    __syncthreads();
                    if (k > 0) {
                        double cp[QNB];
#pragma unroll
                        for (int l = 0; l < QNB; ++l) cp[l] = 0.0;
                        for (int i = t + threadIdx.x; i < m; i += NT) {
                            const double v = yk[i];
#pragma unroll
                            for (int l = 0; l < QNB; ++l)
                                if (l < k) cp[l] += v * ysh[(size_t)l * ms + i];
                        }
#pragma unroll
                        for (int l = 0; l < QNB; ++l)
                            if (l < k) { const double r = warp_sum(cp[l]); if (lane == 0) s_cred[l][warp] = r; }
                        __syncthreads();
                        if (threadIdx.x < k) {
                            double r = 0.0;
                            for (int w = 0; w < NW; ++w) r += s_cred[threadIdx.x][w];
                            lz.c[threadIdx.x] = r;
                        }
                    }
                } else if (threadIdx.x == 0) {
                    d.rank[0] = t;
                }
                __syncthreads();
            }
            if (trc) qr_tr(11);
            group_barrier(bar, G);
            if (trc) qr_tr(12);
            const int r = __ldcg(d.rank);
            if (r >= 0 && k == 0) break;
            if (r < 0 && g != 0) {                     // the step's reflector into shared memory
                double* yk = ysh + (size_t)k * ms;
                const double* ykg = lz.Y + (size_t)k * m;
                for (int i = b + threadIdx.x; i < m; i += NT) yk[i] = ldcg(ykg + i);
                __syncthreads();
            }
            // ---- column phase: owned columns j = g + G q >= jfirst, streamed through the ring
            const int kk = r >= 0 ? k : k + 1;          // reflectors applied in pass 2
            const bool wb = r >= 0 || kk == nb;         // write back (block end or stop)
            const int jfirst = r >= 0 ? t : t + 1;
            const int q0 = jfirst > g ? (jfirst - g + G - 1) / G : 0;
            const int ncol = n > g + G * q0 ? (n - 1 - g - G * q0) / G + 1 : 0;
            const int b0 = b & ~1, me = m & ~1;         // 16-byte aligned bulk copies: rows [b0, me)
            const unsigned bytes = me > b0 ? (unsigned)(me - b0) * 8u : 0u;
            // this step's ring: stages of the current column length (all drained between
            // steps), ncw consumer warps with spc >= 2 stages each where they fit (a consumer
            // computes on one stage while its next column streams into the other)
            const int cst = ((m - b0 + 2) + 1) & ~1;    // doubles per stage
            const int nfit = min(QSMAX, (int)(stg_doubles / cst));
            const int ncw = max(1, min(NCW, nfit / 2));
            const int spc = max(1, min(nfit / ncw, QSMAX / ncw));
            if (warp == 0) {
                if (lane == 0)
                    for (int q = 0; q < ncol; ++q) {
                        // column q -> consumer c = q mod ncw, its x-th column of the step; consumer
                        // c owns the stages c + ncw i, i < spc, used in turn
                        const int c = q % ncw, x = q / ncw;
                        const int st = c + ncw * (x % spc);
                        const unsigned use = s_use[st] + x / spc;
                        if (use > 0) mbar_wait(&empty[st], (use - 1) & 1);
                        mbar_expect_tx(&full[st], bytes);
                        const int j = g + G * (q0 + q);
                        if (bytes) bulk_g2s(stg + (size_t)st * cst, A + (size_t)j * ld + b0, bytes, &full[st]);
                    }
            } else if (warp <= ncw) {
                const double beta = r >= 0 ? 0.0 : __ldcg(d.beta + t);
                double cl[QNB];
#pragma unroll
                for (int l = 0; l < QNB; ++l) cl[l] = (r < 0 && l < k) ? __ldcg(lz.c + l) : 0.0;
                const double* yk = ysh + (size_t)k * ms;
                const int rstart = wb ? b : t + 1;
                int x = 0;
                for (int q = warp - 1; q < ncol; q += ncw, ++x) {
                    const int st = (warp - 1) + ncw * (x % spc);
                    const unsigned use = s_use[st] + x / spc;
                    const int j = g + G * (q0 + q);
                    double* c = A + (size_t)j * ld;
                    double* col = stg + (size_t)st * cst - b0;     // col[i] = row i
                    double w[QNB];
#pragma unroll
                    for (int l = 0; l < QNB; ++l) w[l] = l < k ? __ldcg(lz.W + (size_t)j * QNB + l) : 0.0;
                    mbar_wait(&full[st], use & 1);
                    if ((m & 1) && lane == 0) col[m - 1] = ldcg(c + m - 1);
                    __syncwarp();
                    if (r < 0) {
                        // pass 1: v_t^T a^(b) over rows >= t
                        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                        int i = t + lane;
                        for (; i + 96 < m; i += 128) {
                            s0 += yk[i] * col[i];
                            s1 += yk[i + 32] * col[i + 32];
                            s2 += yk[i + 64] * col[i + 64];
                            s3 += yk[i + 96] * col[i + 96];
                        }
                        for (; i < m; i += 32) s0 += yk[i] * col[i];
                        double d0 = warp_sum((s0 + s1) + (s2 + s3));
#pragma unroll
                        for (int l = 0; l < QNB; ++l)
                            if (l < k) d0 -= cl[l] * w[l];
                        d0 *= beta;
#pragma unroll
                        for (int l = 0; l < QNB; ++l)
                            if (l == k) w[l] = d0;
                        if (lane == 0) lz.W[(size_t)j * QNB + k] = d0;
                    }
                    // pass 2: a^(t+1) = a^(b) - sum_{l < kk} v_l w[l]; norm over rows > t
                    // (kk a compile-time count: no predicated-off multiply-adds)
                    double n0 = 0.0, n1 = 0.0;
                    switch (kk) {
                        case 1: qrcp_pass2<1>(col, ysh, ms, w, rstart, m, t, wb, c, n0, n1); break;
                        case 2: qrcp_pass2<2>(col, ysh, ms, w, rstart, m, t, wb, c, n0, n1); break;
                        case 3: qrcp_pass2<3>(col, ysh, ms, w, rstart, m, t, wb, c, n0, n1); break;
                        case 4: qrcp_pass2<4>(col, ysh, ms, w, rstart, m, t, wb, c, n0, n1); break;
                        case 5: qrcp_pass2<5>(col, ysh, ms, w, rstart, m, t, wb, c, n0, n1); break;
                        case 6: qrcp_pass2<6>(col, ysh, ms, w, rstart, m, t, wb, c, n0, n1); break;
                        case 7: qrcp_pass2<7>(col, ysh, ms, w, rstart, m, t, wb, c, n0, n1); break;
                        case 8: qrcp_pass2<8>(col, ysh, ms, w, rstart, m, t, wb, c, n0, n1); break;
                        default: break;
                    }
                    if (r < 0) {
                        const double nn = warp_sum(n0 + n1);
                        if (lane == 0) d.norms[j] = nn;
                    }
                    fence_proxy_async();                       // generic smem accesses before the next bulk copy
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[st]);
                }
            }
            __syncthreads();
            if (threadIdx.x < ncw * spc) {              // uses of stage st = c + ncw i this step
                const int c = threadIdx.x % ncw, i = threadIdx.x / ncw;
                const int nc = ncol > c ? (ncol - c + ncw - 1) / ncw : 0;
                if (nc > i) s_use[threadIdx.x] += (nc - i + spc - 1) / spc;
            }
            __syncthreads();
            if (trc) qr_tr(13);
            group_barrier(bar, G);
            if (trc) qr_tr(14);
            if (r >= 0) break;
            if (wb) b = t + 1;
        }
        group_barrier(bar, G);
    }
}

// Small matrices (m n <= ~24k doubles: the SPD-HSS sketches 200 x 110, the leaf-level H2
// triangles 128 x 128): one CTA per matrix with the matrix in shared memory -- the same
// Businger-Golub steps (recomputed norms, lowest index on ties), but every step is
// separated by CTA barriers only, not by group barriers through global memory.
__global__ void __launch_bounds__(256) qrcp_smem_kernel(const QrcpDesc* __restrict__ descs, double rel_tol) {
    extern __shared__ double smq[];
    __shared__ double sv[32];
    __shared__ int si[32];
    const QrcpDesc d = descs[blockIdx.x];
    const int m = d.m, n = d.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    double* As = smq;                                // m x n, ld m
    double* nrm = smq + (size_t)m * n;
    int* pv = (int*)(nrm + n);
    for (int e = tid; e < m * n; e += blockDim.x) As[e] = d.A[e % m + (size_t)(e / m) * d.ld];
    for (int j = tid; j < n; j += blockDim.x) pv[j] = j;
    __syncthreads();
    for (int j = warp; j < n; j += nw) {
        double sacc = 0.0;
        for (int i = lane; i < m; i += 32) { const double x = As[i + (size_t)j * m]; sacc += x * x; }
        sacc = warp_sum(sacc);
        if (lane == 0) nrm[j] = sacc;
    }
    __syncthreads();
    const int kmax = min(min(m, n), d.max_rank);
    double nu0 = 0.0;
    int rank = kmax;
    for (int t = 0; t < kmax; ++t) {
        double v = -1.0;
        int idx = 0x7fffffff;
        for (int j = t + tid; j < n; j += blockDim.x) {
            const double x = nrm[j];
            if (x > v) { v = x; idx = j; }             // ascending j: lowest index on ties
        }
        double bv;
        int bi;
        block_argmax(v, idx, sv, si, bv, bi);
        const double nu = bv > 0.0 ? sqrt(bv) : 0.0;
        if (t == 0) nu0 = nu;
        if (d.force) {                                  // injected pivots (R19 hook)
            if (t >= d.nforce) { rank = t; break; }
            const int want = d.force[t];
            for (int j = t + tid; j < n; j += blockDim.x)
                if (pv[j] == want) si[0] = j;
            __syncthreads();
            bi = si[0];
            __syncthreads();
        } else if (nu == 0.0 || nu <= rel_tol * nu0) { rank = t; break; }
        const int p = bi;
        if (p != t) {
            for (int i = tid; i < m; i += blockDim.x) {
                const double a = As[i + (size_t)t * m];
                As[i + (size_t)t * m] = As[i + (size_t)p * m];
                As[i + (size_t)p * m] = a;
            }
            if (tid == 0) {
                const int tp = pv[t]; pv[t] = pv[p]; pv[p] = tp;
                const double tn = nrm[t]; nrm[t] = nrm[p]; nrm[p] = tn;
            }
        }
        __syncthreads();
        double* ct = As + (size_t)t * m;
        double sig = 0.0;
        for (int i = t + 1 + tid; i < m; i += blockDim.x) { const double x = ct[i]; sig += x * x; }
        sig = block_sum(sig, sv);
        const double x0 = ct[t];
        double beta, mu, v0;
        if (sig == 0.0) { beta = (x0 >= 0.0) ? 0.0 : 2.0; mu = fabs(x0); v0 = 1.0; }
        else {
            mu = sqrt(x0 * x0 + sig);
            v0 = (x0 <= 0.0) ? x0 - mu : -sig / (x0 + mu);
            beta = 2.0 * v0 * v0 / (sig + v0 * v0);
        }
        const double inv0 = 1.0 / v0;
        for (int i = t + 1 + tid; i < m; i += blockDim.x) ct[i] = (sig == 0.0) ? 0.0 : ct[i] * inv0;
        __syncthreads();
        if (tid == 0) { ct[t] = mu; d.beta[t] = beta; }
        // columns j > t: w = beta v^T a_j (v_t = 1), a_j -= w v, norms over rows > t
        for (int j = t + 1 + warp; j < n; j += nw) {
            double* cj = As + (size_t)j * m;
            double sacc = lane == 0 ? cj[t] : 0.0;
            for (int i = t + 1 + lane; i < m; i += 32) sacc += ct[i] * cj[i];
            const double w = beta * warp_sum(sacc);
            double nn = 0.0;
            for (int i = t + 1 + lane; i < m; i += 32) { const double a = cj[i] - w * ct[i]; cj[i] = a; nn += a * a; }
            nn = warp_sum(nn);
            if (lane == 0) { cj[t] -= w; nrm[j] = nn; }
        }
        __syncthreads();
    }
    for (int e = tid; e < m * n; e += blockDim.x) d.A[e % m + (size_t)(e / m) * d.ld] = As[e];
    for (int j = tid; j < n; j += blockDim.x) { d.piv[j] = pv[j]; d.norms[j] = nrm[j]; }
    if (tid == 0) d.rank[0] = rank;
}

__global__ void gather_ranks_kernel(const QrcpDesc* __restrict__ d, int n, int* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = *d[i].rank;
}

// algorithmic work of the QRCPs just enqueued (profiling only; ranks read back): step t of
// the Businger-Golub QRCP with recomputed norms (R4) must read every entry of the trailing
// (m-t) x (n-t) block once (the norms of the updated columns) -- 8 B per entry, the
// algorithmic bytes -- and does 6 flops per entry (dot, update, norm).  The write-back of
// the updated block is an implementation cost: every step in the eager kernel (16 B per
// entry of DRAM traffic), once per nb steps in the deferred kernel (8 + 8/nb B).
static void qrcp_prof_exact(cudaStream_t s, const std::vector<QrcpDesc>& d, const QrcpDesc* dd) {
    if (!prof_on()) return;
    DBuf<int> rk(d.size());
    gather_ranks_kernel<<<ceil_div((int64_t)d.size(), 256), 256, 0, s>>>(dd, (int)d.size(), rk.p);
    std::vector<int> r = rk.download(s);
    double by = 0.0, fl = 0.0;
    for (size_t i = 0; i < d.size(); ++i)
        for (int t = 0; t <= std::min(r[i], std::min(d[i].m, d[i].n) - 1); ++t) {   // + the stopping step's norms
            const double e = (double)(d[i].m - t) * (d[i].n - t);
            by += 8.0 * e;
            fl += 6.0 * e;
        }
    prof_update_last("qrcp", fl, by);
}

// CTA shape of the deferred kernel for matrices of up to m rows: 256 threads, two CTAs per
// SM (more, finer groups) up to 1024 rows; 512 threads, one CTA per SM (the whole shared
// memory for one ring of long columns) beyond; SPD_QRCP_NT overrides
static int qrcp_nt(int m) {
    static const int env = getenv("SPD_QRCP_NT") ? atoi(getenv("SPD_QRCP_NT")) : 0;
    if (env == 256 || env == 512) return env;
    return m <= 1024 ? 256 : 512;
}
int qrcp_slots(int m) {
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        SPD_CUDA(cudaGetDevice(&dev));
        SPD_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    if (getenv("SPD_QRCP_EAGER")) return 3 * nsm;
    return qrcp_nt(m) == 256 ? 2 * nsm : nsm;
}

void qrcp_batched(cudaStream_t s, const std::vector<QrcpDesc>& d, double rel_tol) {
    if (d.empty()) return;
    {
        size_t need = 0;
        for (auto& q : d) need = std::max(need, sizeof(double) * ((size_t)q.m * q.n + q.n) + sizeof(int) * q.n);
        if (need <= 200 * 1024 && !getenv("SPD_QRCP_GROUP")) {
            static size_t set = 0;
            if (need > 48 * 1024 && need > set) {
                SPD_CUDA(cudaFuncSetAttribute(qrcp_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                set = 200 * 1024;
            }
            double fl = 0;
            for (auto& q : d) fl += 4.0 * q.m * q.n * std::min(std::min(q.m, q.n), q.max_rank);
            DevArray<QrcpDesc> dd(s, d);
            {
                ProfScope prof(s, "qrcp", fl, 0);
                for (size_t off = 0; off < d.size(); off += 65535) {
                    qrcp_smem_kernel<<<(unsigned)std::min<size_t>(65535, d.size() - off), 256, need, s>>>(dd.p + off, rel_tol);
                    SPD_LAUNCH();
                }
            }
            qrcp_prof_exact(s, d, dd.p);
            return;
        }
    }
    int dev = 0;
    SPD_CUDA(cudaGetDevice(&dev));
    int nsm = 0, per_sm = 0;
    SPD_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    int mmax = 1;
    for (auto& q : d) mmax = std::max(mmax, q.m);
    // deferred-update kernel (default; SPD_QRCP_EAGER=1: the read+write-per-step kernel):
    // nb reflectors per block (SPD_QRCP_NB, default 4) in shared memory next to a ring of
    // column stages (one column of <= mmax rows each); one CTA of NT threads per SM.  Needs
    // 16-byte aligned columns (bulk copies) and >= 2 stages, else the eager kernel.
    static const bool eager_env = getenv("SPD_QRCP_EAGER") != nullptr;
    static const int nb_env = getenv("SPD_QRCP_NB") ? atoi(getenv("SPD_QRCP_NB")) : 2;
    // CTA shape: 512 threads, one CTA per SM (the whole shared memory for one ring), or
    // 256 threads, two CTAs per SM (twice the CTAs to share among the matrices: finer groups)
    const int nt_env = qrcp_nt(mmax);
    const int ms = (mmax + 1) & ~1;                  // reflector row stride (even: 16-byte stages)
    const int sst = ((mmax + 2) + 1) & ~1;           // doubles per column stage
    const size_t budget = nt_env == 256 ? 110 * 1024 : 220 * 1024;
    bool aligned = true;
    for (auto& q : d) aligned = aligned && ((uintptr_t)q.A % 16 == 0) && (q.ld % 2 == 0);
    // (the kernel re-plans the ring every step for the current column length; here: at
    // least two full-length stages must fit next to the reflectors)
    int nb = std::max(1, std::min(QNB, nb_env)), nstage = 0;
    for (; nb >= 1; --nb) {
        const size_t ybytes = sizeof(double) * (size_t)nb * ms;
        nstage = ybytes < budget ? (int)((budget - ybytes) / (sizeof(double) * sst)) : 0;
        if (nstage >= 2) break;
    }
    const bool eager = eager_env || !aligned || nb < 1 || nstage < 2;
    const void* lazy_fn = nt_env == 256 ? (const void*)qrcp_lazy_kernel<256> : (const void*)qrcp_lazy_kernel<512>;
    const int lazy_nt = nt_env == 256 ? 256 : 512;
    const size_t qsmem = eager ? sizeof(double) * (size_t)mmax
                               : sizeof(double) * ((size_t)nb * ms + (size_t)nstage * sst);
    SPD_REQUIRE(qsmem <= 220 * 1024, "qrcp: matrix too tall");
    SPD_CUDA(cudaFuncSetAttribute(eager ? (const void*)qrcp_kernel : lazy_fn,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(qsmem, 48 * 1024)));
    SPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, eager ? (const void*)qrcp_kernel : lazy_fn,
                                                           eager ? QR_THREADS : lazy_nt, qsmem));
    const int cap = std::max(1, nsm * std::max(1, per_sm));
    // work estimate per matrix ~ m * n * min(m, n, max_rank)
    std::vector<double> work(d.size());
    double total = 0.0;
    for (size_t i = 0; i < d.size(); ++i) {
        double k = std::max(1, std::min(std::min(d[i].m, d[i].n), d[i].max_rank));
        work[i] = (double)std::max(d[i].m, 1) * std::max(d[i].n, 1) * k;
        total += work[i];
    }
    DevArray<QrcpDesc> dd(s, d);
    // per-matrix scratch of the deferred kernel: Y (nb x m), W (n x QNB), c (QNB)
    size_t lz_total = 0;
    if (!eager)
        for (auto& q : d) lz_total += (size_t)nb * q.m + (size_t)q.n * QNB + QNB;
    DBuf<double> lzbuf(std::max<size_t>(1, lz_total));
    std::vector<QrcpLazy> lzv;
    if (!eager) {
        size_t off = 0;
        for (auto& q : d) {
            QrcpLazy z;
            z.Y = lzbuf.p + off; off += (size_t)nb * q.m;
            z.W = lzbuf.p + off; off += (size_t)q.n * QNB;
            z.c = lzbuf.p + off; off += QNB;
            lzv.push_back(z);
        }
    }
    DevArray<QrcpLazy> dlz(s, lzv);
    unsigned* bars = nullptr;
    SPD_CUDA(cudaMallocAsync((void**)&bars, sizeof(unsigned) * 2 * d.size(), s));
    SPD_CUDA(cudaMemsetAsync(bars, 0, sizeof(unsigned) * 2 * d.size(), s));
    // L2-resident rounds (env SPD_QRCP_L2MB = budget in MB, 0 = one round): matrices in
    // rounds whose working sets fit the budget, each round with all CTAs, so the per-step
    // re-reads of the trailing matrices hit L2 instead of HBM
    const char* l2e = getenv("SPD_QRCP_L2MB");
    const double l2b = l2e ? atof(l2e) * 1e6 : 0.0;
    std::vector<std::vector<int>> rounds;
    if (l2b > 0.0) {
        std::vector<int> order(d.size());
        for (size_t i = 0; i < d.size(); ++i) order[i] = (int)i;
        std::sort(order.begin(), order.end(), [&](int a, int b) { return work[a] > work[b]; });
        double acc = 0.0;
        for (int i : order) {
            const double b = 8.0 * d[i].m * d[i].n;
            if (rounds.empty() || acc + b > l2b || (int)rounds.back().size() >= cap) { rounds.push_back({}); acc = 0.0; }
            rounds.back().push_back(i);
            acc += b;
        }
    } else {
        rounds.push_back({});
        for (size_t i = 0; i < d.size(); ++i) rounds.back().push_back((int)i);
    }
    double fl = 0, by = 0;
    for (size_t i = 0; i < d.size(); ++i) { fl += 4.0 * work[i]; by += 8.0 * d[i].m * d[i].n; }
    {
        ProfScope prof(s, "qrcp", fl, by);     // exact counts filled in by qrcp_prof_exact (profiling)
        for (const auto& rd : rounds) {
        double rtotal = 0.0;
        for (int i : rd) rtotal += work[i];
        std::vector<QrItem> items;
        std::vector<int2> cta;
        if ((int)rd.size() >= cap) {
            // one CTA per matrix, CTAs loop over matrices (largest first, greedy balance)
            std::vector<int> order(rd);
            std::sort(order.begin(), order.end(), [&](int a, int b) { return work[a] > work[b]; });
            std::vector<std::vector<int>> bins(cap);
            std::vector<double> load(cap, 0.0);
            for (int i : order) {
                int b = (int)(std::min_element(load.begin(), load.end()) - load.begin());
                bins[b].push_back(i);
                load[b] += work[i];
            }
            for (int b = 0; b < cap; ++b) {
                int begin = (int)items.size();
                for (int i : bins[b]) items.push_back({i, 0, 1});
                cta.push_back(make_int2(begin, (int)items.size()));
            }
        } else {
            // CTAs per matrix: one each, then every spare CTA to the matrix whose time
            // work / G is largest (greedy min-max; proportional rounding left near-equal
            // matrices with G and G + 1 CTAs, i.e. the slowest at up to twice the rest)
            const int gmax = l2b > 0.0 ? 128 : 64;
            std::vector<int> Gs(d.size(), 1);
            {
                std::priority_queue<std::pair<double, int>> pq;
                for (int i : rd) pq.push({work[i], i});
                for (int spare = cap - (int)rd.size(); spare > 0 && !pq.empty(); --spare) {
                    const int i = pq.top().second;
                    pq.pop();
                    if (Gs[i] >= std::max(1, std::min(d[i].n, gmax))) { ++spare; continue; }
                    ++Gs[i];
                    pq.push({work[i] / Gs[i], i});
                }
            }
            for (int i : rd) {
                const int G = Gs[i];
                for (int g = 0; g < G; ++g) {
                    cta.push_back(make_int2((int)items.size(), (int)items.size() + 1));
                    items.push_back({i, g, G});
                }
            }
        }
        DevArray<QrItem> di(s, items);
        DevArray<int2> dc(s, cta);
        const QrcpDesc* a0 = dd.p;
        const QrItem* a1 = di.p;
        const int2* a2 = dc.p;
        double tol = rel_tol;
        if (eager) {
            void* args[] = {(void*)&a0, (void*)&a1, (void*)&a2, (void*)&bars, (void*)&tol};
            SPD_CUDA(cudaLaunchCooperativeKernel((void*)qrcp_kernel, dim3((unsigned)cta.size()), dim3(QR_THREADS),
                                                 args, qsmem, s));
        } else {
            const QrcpLazy* a5 = dlz.p;
            int nbv = nb, msv = ms, nsv = nstage, sstv = sst;
            static const int steptr = getenv("SPD_QR_STEPS") ? 1 : 0;
            int stv = steptr;
            void* args[] = {(void*)&a0, (void*)&a5, (void*)&a1, (void*)&a2, (void*)&bars, (void*)&tol, (void*)&nbv,
                            (void*)&msv, (void*)&nsv, (void*)&sstv, (void*)&stv};
            SPD_CUDA(cudaLaunchCooperativeKernel(lazy_fn, dim3((unsigned)cta.size()), dim3(lazy_nt),
                                                 args, qsmem, s));
        }
        count_launch();
        }
    }
    static const bool trace = getenv("SPD_QR_TRACE") != nullptr;
    if (trace) {
        unsigned long long tr[16];
        SPD_CUDA(cudaStreamSynchronize(s));
        SPD_CUDA(cudaMemcpyFromSymbol(tr, g_qr_trace, sizeof(tr), 10 * sizeof(unsigned long long)));
        fprintf(stderr, "[qrcp trace] %zu mats, %zu rounds, m %d n %d: leader %.2f bar1 %.2f update %.2f bar2 %.2f us\n",
                d.size(), rounds.size(), d[0].m, d[0].n, (tr[1] - tr[0]) * 1e-3, (tr[2] - tr[1]) * 1e-3,
                (tr[3] - tr[2]) * 1e-3, (tr[4] - tr[3]) * 1e-3);
    }
    if (getenv("SPD_QR_STEPS") && !eager) {
        static std::vector<unsigned long long> st(8192);
        SPD_CUDA(cudaStreamSynchronize(s));
        SPD_CUDA(cudaMemcpyFromSymbol(st.data(), g_qr_steps, sizeof(unsigned long long) * 8192));
        int rk = 0;
        SPD_CUDA(cudaMemcpy(&rk, d[0].rank, sizeof(int), cudaMemcpyDeviceToHost));
        fprintf(stderr, "[qrcp steps] %zu mats m %d rank %d:", d.size(), d[0].m, rk);
        for (int t = 0; t + 50 < std::min(rk, 8192); t += 50)
            fprintf(stderr, " %d:%.1f", t, (st[t + 50] - st[t]) * 1e-3 / 50);
        fprintf(stderr, " us/step\n");
    }
    SPD_CUDA(cudaFreeAsync(bars, s));
    qrcp_prof_exact(s, d, dd.p);
}

// ================================================================= unpivoted blocked QR
constexpr int QB = 32;
struct PanelDesc {
    double* A; int m, n, ld;     // full matrix
    int p, jb;                   // panel columns [p, p + jb)
    double* V; int ldv;          // (m - p) x jb explicit unit-lower reflectors
    double* T;                   // jb x jb (ld QB) compact-WY factor, H_0..H_{jb-1} = I - V T V^T
};

// one CTA per panel: Householder column by column (warp per column for the
// updates, so only two block barriers per column), then T from V^T V.
__global__ void __launch_bounds__(256) panel_qr_kernel(const PanelDesc* descs) {
    const PanelDesc d = descs[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = 8;
    const int L = d.m - d.p;                 // panel rows
    double* P = d.A + d.p + (size_t)d.p * d.ld;   // panel origin
    __shared__ double s_beta[QB], s_v0, s_mu, s_sig;
    __shared__ double G[QB][QB + 1];         // V^T V
    for (int j = 0; j < d.jb; ++j) {
        double* col = P + (size_t)j * d.ld;
        if (warp == 0) {
            double sg = 0.0;
            for (int i = j + 1 + lane; i < L; i += 32) { double x = col[i]; sg += x * x; }
            sg = warp_sum(sg);
            if (lane == 0) {
                const double x0 = col[j];
                double beta, mu, v0;
                if (sg == 0.0) { beta = (x0 >= 0.0) ? 0.0 : 2.0; mu = fabs(x0); v0 = 1.0; }
                else {
                    mu = sqrt(x0 * x0 + sg);
                    v0 = (x0 <= 0.0) ? x0 - mu : -sg / (x0 + mu);
                    beta = 2.0 * v0 * v0 / (sg + v0 * v0);
                }
                s_beta[j] = beta; s_v0 = v0; s_mu = mu; s_sig = sg;
            }
        }
        __syncthreads();
        const double inv0 = (s_sig == 0.0) ? 0.0 : 1.0 / s_v0;
        double* v = d.V + (size_t)j * d.ldv;
        for (int i = threadIdx.x; i < L; i += blockDim.x) {
            double vi = (i < j) ? 0.0 : (i == j ? 1.0 : col[i] * inv0);
            v[i] = vi;
        }
        __syncthreads();
        if (threadIdx.x == 0) col[j] = s_mu;
        const double beta = s_beta[j];
        for (int c = j + 1 + warp; c < d.jb; c += nw) {
            double* cc = P + (size_t)c * d.ld;
            double w = 0.0;
            for (int i = j + lane; i < L; i += 32) w += v[i] * cc[i];
            w = warp_sum(w) * beta;
            for (int i = j + lane; i < L; i += 32) cc[i] -= w * v[i];
        }
        __syncthreads();
    }
    // G = V^T V (upper part), T recurrence: T_jj = beta_j, T[:j, j] = -beta_j T[:j,:j] (V^T v_j)[:j]
    for (int pr = warp; pr < d.jb * d.jb; pr += nw) {
        const int a = pr % d.jb, b = pr / d.jb;
        if (a >= b) continue;
        const double* va = d.V + (size_t)a * d.ldv;
        const double* vb = d.V + (size_t)b * d.ldv;
        double s = 0.0;
        for (int i = b + lane; i < L; i += 32) s += va[i] * vb[i];
        s = warp_sum(s);
        if (lane == 0) G[a][b] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double* T = d.T;
        for (int j = 0; j < d.jb; ++j) {
            const double beta = s_beta[j];
            for (int a = 0; a < j; ++a) {
                double s = 0.0;
                for (int b = a; b < j; ++b) s += T[a + b * QB] * G[b][j];
                T[a + j * QB] = -beta * s;
            }
            T[j + j * QB] = beta;
            for (int a = j + 1; a < QB; ++a) T[a + j * QB] = 0.0;
        }
    }
}

// Cluster panel QR: a cluster of QCL CTAs per panel; CTA g keeps rows
// [g*rp, (g+1)*rp) of the panel in shared memory.  ONE cluster barrier per column:
// before the reflector of column j is known, every CTA forms the partial sums over
// its rows i > j of  A_ij^2 (sigma),  A_ij A_ic (c > j)  and  V_ia A_ij (a < j)  and
// publishes them with the row-j values it owns; after the barrier every CTA adds
// the QCL partials (lane q reads CTA q, xor-butterfly: bitwise identical everywhere)
// and derives the Householder scalars, w_c = A_jc + d_c / v0 for the update and
// V^T v_j = V_j. + g / v0 for the next column of the compact-WY T (T_jj = beta_j,
// T[:j, j] = -beta_j T[:j, :j] V^T v_j; Golub-Van Loan 5.1.2), without a second pass.
namespace cg = cooperative_groups;

__device__ __forceinline__ void qr_tr0(int k) {        // CTA 0 only
    if (blockIdx.x == 0 && threadIdx.x == 0) qr_tr(k);
}

template <int QCL, int PW>
__global__ void __launch_bounds__(512) panel_qr_cluster_kernel(const PanelDesc* descs, int rp) {
    cg::cluster_group cluster = cg::this_cluster();
    const int g = (int)cluster.block_rank();
    const PanelDesc d = descs[blockIdx.x / QCL];
    extern __shared__ double sm[];                    // rp x PW panel slice (col-major, ld rp)
    constexpr int NP = 2 * PW + 2;                    // partials per column
    __shared__ double part[2][NP];                    // [0..PW): A_ij A_ic (c = j: sigma), [PW..2QB): V_ia A_ij,
                                                      // [2QB]: x0 (row-j owner), row-j values in rowv
    __shared__ double rowv[2][2 * PW];                // row j: A_jc (c > j) and V_ja (a < j), owner CTA only
    __shared__ double T[PW][PW + 1];
    __shared__ double vtv[PW];
    __shared__ double wc[PW];
    __shared__ double tot[NP + 2 * PW];               // their sums
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int L = d.m - d.p, jb = d.jb;
    const int r0 = g * rp, nr = max(0, min(rp, L - r0));
    double* P = d.A + d.p + (size_t)d.p * d.ld;
    qr_tr0(0);
    // panel slice -> smem with asynchronous copies (all in flight at once)
    for (int c = 0; c < jb; ++c)
        for (int i = threadIdx.x; i < rp; i += blockDim.x)
            cp_async8(sm + i + c * rp, i < nr ? P + r0 + i + (size_t)c * d.ld : P, i < nr);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    qr_tr0(1);
    for (int j = 0; j < jb; ++j) {
        if (j == 1) qr_tr0(2);
        if (j == 16) qr_tr0(3);
        const int buf = j & 1;
        const double* colj = sm + j * rp;
        // ---- partial sums over my rows i > j (warp w: entries e = w, w + 8, ...)
        //      e < PW: column c = j + e (c == j: sigma);  PW <= e < PW + j: reflector a = e - PW
        for (int e = warp; e < PW + j; e += (int)(blockDim.x >> 5)) {
            double acc = 0.0;
            const double* other = e < PW ? (j + e < jb ? sm + (j + e) * rp : nullptr) : sm + (e - PW) * rp;
            if (other)
                for (int i = lane; i < nr; i += 32)
                    if (r0 + i > j) acc += colj[i] * other[i];
            acc = warp_sum(acc);
            if (lane == 0) part[buf][e] = acc;
        }
        // row-j values (owner of row j)
        const bool own = j >= r0 && j < r0 + nr;
        if (own) {
            const int lj = j - r0;
            for (int c = threadIdx.x; c < jb; c += blockDim.x) rowv[buf][c] = sm[lj + c * rp];          // A_jc
            for (int a = threadIdx.x; a < j; a += blockDim.x) rowv[buf][PW + a] = sm[lj + a * rp];      // V_ja
        } else {
            for (int c = threadIdx.x; c < jb; c += blockDim.x) rowv[buf][c] = 0.0;
            for (int a = threadIdx.x; a < j; a += blockDim.x) rowv[buf][PW + a] = 0.0;
        }
        cluster.sync();
        // ---- sum every entry over the CTAs in rank order (same bits in every CTA):
        //      thread e issues its QCL remote (DSMEM) loads at once
        {
            constexpr int NE = NP + 2 * PW;
            for (int e = threadIdx.x; e < NE; e += blockDim.x) {
                const double* base = e < NP ? &part[buf][e] : &rowv[buf][e - NP];
                double v[QCL];
#pragma unroll
                for (int q = 0; q < QCL; ++q) v[q] = *cluster.map_shared_rank(base, q);
                double t = 0.0;
#pragma unroll
                for (int q = 0; q < QCL; ++q) t += v[q];
                tot[e] = t;
            }
            __syncthreads();
        }
        const double sig = tot[0], x0 = tot[NP + j];
        double beta, mu, v0;
        if (sig == 0.0) { beta = (x0 >= 0.0) ? 0.0 : 2.0; mu = fabs(x0); v0 = 1.0; }
        else {
            mu = sqrt(x0 * x0 + sig);
            v0 = (x0 <= 0.0) ? x0 - mu : -sig / (x0 + mu);
            beta = 2.0 * v0 * v0 / (sig + v0 * v0);
        }
        const double inv0 = (sig == 0.0) ? 0.0 : 1.0 / v0;
        // w_c = A_jc + d_c / v0 (c > j);  V^T v_j [a] = V_ja + g_a / v0 (a < j)
        for (int c = j + 1 + threadIdx.x; c < jb; c += blockDim.x) wc[c] = tot[NP + c] + tot[c - j] * inv0;
        for (int a = threadIdx.x; a < j; a += blockDim.x) vtv[a] = tot[NP + PW + a] + tot[PW + a] * inv0;
        __syncthreads();
        // ---- T column j (warp 0; identical in every CTA, CTA 0 stores it)
        if (warp == 0) {
            double t = 0.0;
            if (lane < j)
                for (int b = lane; b < j; ++b) t += T[lane][b] * vtv[b];
            __syncwarp();
            if (lane < j) T[lane][j] = -beta * t;
            if (lane == j) T[j][j] = beta;
            if (lane > j && lane < PW) T[lane][j] = 0.0;
        }
        // ---- update my rows: column j -> v (mu at row j), columns c > j -= beta w_c v
        double* colw = sm + j * rp;
        for (int i = threadIdx.x; i < nr; i += blockDim.x) {
            const int gi = r0 + i;
            const double vi = gi < j ? 0.0 : (gi == j ? 1.0 : colw[i] * inv0);
            for (int c = j + 1; c < jb; ++c) sm[i + c * rp] -= beta * wc[c] * vi;
            if (gi > j) colw[i] = vi;
            else if (gi == j) colw[i] = mu;
            d.V[(size_t)j * d.ldv + gi] = vi;
        }
        __syncthreads();
    }
    qr_tr0(4);
    // write the R part (rows <= column) back; the rest of the slice is scratch
    for (int c = 0; c < jb; ++c)
        for (int i = threadIdx.x; i < nr; i += blockDim.x)
            if (r0 + i <= c) P[r0 + i + (size_t)c * d.ld] = sm[i + c * rp];
    if (g == 0)
        for (int e = threadIdx.x; e < PW * PW; e += blockDim.x) d.T[e] = T[e % PW][e / PW];
    qr_tr0(5);
    qr_tr0(6);
    cluster.sync();                                   // keep smem alive for remote readers
}

template <int PW>
static void launch_panels_pw(cudaStream_t s, const std::vector<PanelDesc>& pd, int p) {
        if (pd.empty()) return;
        {
            DevArray<PanelDesc> dp(s, pd);
            double pb = 0;
            int Lmax = 0;
            for (auto& q : pd) { pb += 8.0 * (q.m - q.p) * q.jb * (q.jb + 2); Lmax = std::max(Lmax, q.m - q.p); }
            // cluster of 8 CTAs (portable) when the panel slice fits 180 KB, else 16 (non-portable)
            // (env SPD_QR_QCL8_KB: largest 8-CTA slice in KB, default 208: the 6144-row proxy
            // panels run as 8-CTA clusters of one CTA per SM, measured 1 % faster than 16 x 2)
            static const int q8kb = getenv("SPD_QR_QCL8_KB") ? atoi(getenv("SPD_QR_QCL8_KB")) : 208;
            const int qcl = ceil_div(Lmax, 8) * PW * (int)sizeof(double) <= q8kb * 1024 ? 8 : 16;
            const int rp = ceil_div(Lmax, qcl);
            const size_t sh = (size_t)rp * PW * sizeof(double);
            ProfScope prof(s, "qr_panel", 0, pb);
            if (sh <= 208 * 1024) {
                static bool attr = false;   // per PW instantiation
                if (!attr) {
                    SPD_CUDA(cudaFuncSetAttribute(panel_qr_cluster_kernel<8, PW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 208 * 1024));
                    SPD_CUDA(cudaFuncSetAttribute(panel_qr_cluster_kernel<16, PW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024));
                    SPD_CUDA(cudaFuncSetAttribute(panel_qr_cluster_kernel<16, PW>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                    attr = true;
                }
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3((unsigned)pd.size() * qcl);
                cfg.blockDim = dim3(512);
                cfg.dynamicSmemBytes = sh;
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = qcl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                if (qcl == 8) SPD_CUDA(cudaLaunchKernelEx(&cfg, panel_qr_cluster_kernel<8, PW>, (const PanelDesc*)dp.p, rp));
                else SPD_CUDA(cudaLaunchKernelEx(&cfg, panel_qr_cluster_kernel<16, PW>, (const PanelDesc*)dp.p, rp));
                count_launch();
                static const bool trace = getenv("SPD_QR_TRACE") != nullptr;
                if (trace && p == 0) {
                    unsigned long long tr[8];
                    SPD_CUDA(cudaStreamSynchronize(s));
                    SPD_CUDA(cudaMemcpyFromSymbol(tr, g_qr_trace, sizeof(tr)));
                    fprintf(stderr, "[qr trace] panels %zu qcl %d rp %d: load %.1f col0 %.1f cols1-15 %.1f cols16-31 %.1f "
                            "gram %.1f T %.1f us\n", pd.size(), qcl, rp, (tr[1] - tr[0]) * 1e-3, (tr[2] - tr[1]) * 1e-3,
                            (tr[3] - tr[2]) * 1e-3, (tr[4] - tr[3]) * 1e-3, (tr[5] - tr[4]) * 1e-3, (tr[6] - tr[5]) * 1e-3);
                }
            } else {
                SPD_REQUIRE(PW == QB, "qr panel: slice too tall for the cluster kernel");
                panel_qr_kernel<<<(unsigned)pd.size(), 256, 0, s>>>(dp.p);
                SPD_LAUNCH();
            }
        }
    }

static void launch_panels(cudaStream_t s, const std::vector<PanelDesc>& pd, int p, int pw = QB) {
    if (pw == 16) launch_panels_pw<16>(s, pd, p);
    else launch_panels_pw<QB>(s, pd, p);
}

// Blocks of NP panels (NP x 32 columns): panel s is updated by the reflectors of panels
// 0..s-1 of its block (combined compact-WY factor T_{0:s}), factored, and T is extended
// (Schreiber-Van Loan: T_{0:s+1} = [T_{0:s}, -T_{0:s} V_{0:s}^T V_s T_s; 0, T_s]); the
// rest of the trailing matrix gets ONE rank-(32 NP) update per block, so its traffic is
// 1/NP of the column-by-panel scheme and the far GEMMs have K = 32 NP.
static void qr_blocked_np(cudaStream_t s, const std::vector<QrDesc>& d, int NP, int PW = QB) {
    const int KB = NP * PW;
    int nmax = 0;
    size_t vtot = 0, wtot = 0;
    std::vector<size_t> voff(d.size()), woff(d.size());
    for (size_t i = 0; i < d.size(); ++i) {
        nmax = std::max(nmax, d[i].n);
        voff[i] = vtot; vtot += (size_t)d[i].m * KB;
        woff[i] = wtot; wtot += (size_t)KB * std::max(d[i].n, PW);
    }
    const size_t nd = d.size();
    DBuf<double> V(vtot), T(nd * KB * KB), Ts(nd * PW * PW), S(nd * KB * PW), X(nd * KB * PW), W(wtot), W2(wtot);
    for (int p = 0; p < nmax; p += KB) {
        V.zero(s);                                    // rows above each panel's start must be 0
        T.zero(s);
        std::vector<int> kacc(nd, 0);                 // reflector columns of the block so far
        std::vector<int> done(nd, 0);                 // columns of the block already handled
        for (int sp = 0; sp < NP; ++sp) {
            std::vector<GemmDesc> u1, u2, u3, e1, e2, e3;
            std::vector<PanelDesc> pd;
            std::vector<CopyDesc> cp;
            for (size_t i = 0; i < nd; ++i) {
                const QrDesc& q = d[i];
                const int kk = std::min(q.n, q.m);
                const int ps = p + done[i];
                if (ps >= q.n || done[i] < sp * PW) continue;       // block ended early for this matrix
                const int ncols = std::min(PW, q.n - ps);
                const int jb = std::max(0, std::min(PW, kk - ps));
                const int K = kacc[i], L = q.m - p;
                double* Vb = V.p + voff[i];
                double* Tb = T.p + i * KB * KB;
                double* As = q.A + p + (size_t)ps * q.ld;              // rows from p
                if (K > 0) {                                            // in-block update of panel sp
                    u1.push_back({Vb, As, W.p + woff[i], K, ncols, L, q.m, q.ld, KB});
                    u2.push_back({Tb, W.p + woff[i], W2.p + woff[i], K, ncols, K, KB, KB, KB});
                    u3.push_back({Vb, W2.p + woff[i], As, L, ncols, K, q.m, KB, q.ld});
                }
                done[i] += ncols;
                if (jb <= 0) continue;
                double* Vs = Vb + (size_t)K * q.m + (ps - p);
                pd.push_back({q.A, q.m, q.n, q.ld, ps, jb, Vs, q.m, Ts.p + i * PW * PW});
                if (K > 0) {                                            // extend T
                    const int Ls = q.m - ps;
                    e1.push_back({Vb + (ps - p), Vs, S.p + i * KB * PW, K, jb, Ls, q.m, q.m, KB});
                    e2.push_back({Tb, S.p + i * KB * PW, X.p + i * KB * PW, K, jb, K, KB, KB, KB});
                    e3.push_back({X.p + i * KB * PW, Ts.p + i * PW * PW, Tb + (size_t)K * KB, K, jb, jb, KB, PW, KB});
                }
                cp.push_back({Ts.p + i * PW * PW, Tb + K + (size_t)K * KB, jb, jb, PW, KB, 0});
                kacc[i] = K + jb;
            }
            gemm_batched(s, u1, true, false, 1.0, 0.0);
            gemm_batched(s, u2, true, false, 1.0, 0.0);
            gemm_batched(s, u3, false, false, -1.0, 1.0);
            launch_panels(s, pd, p + sp * PW, PW);
            gemm_batched(s, e1, true, false, 1.0, 0.0);
            gemm_batched(s, e2, false, false, 1.0, 0.0);
            gemm_batched(s, e3, false, false, -1.0, 0.0);
            copy_batched(s, cp, 1.0, false);
        }
        // far columns: one rank-K update with the block's combined factor
        std::vector<GemmDesc> g1, g2, g3;
        for (size_t i = 0; i < nd; ++i) {
            const QrDesc& q = d[i];
            const int pf = p + done[i], nt = q.n - pf, K = kacc[i], L = q.m - p;
            if (nt <= 0 || K <= 0 || p >= q.n) continue;
            double* Af = q.A + p + (size_t)pf * q.ld;
            g1.push_back({V.p + voff[i], Af, W.p + woff[i], K, nt, L, q.m, q.ld, KB});
            g2.push_back({T.p + i * KB * KB, W.p + woff[i], W2.p + woff[i], K, nt, K, KB, KB, KB});
            g3.push_back({V.p + voff[i], W2.p + woff[i], Af, L, nt, K, q.m, KB, q.ld});
        }
        gemm_batched(s, g1, true, false, 1.0, 0.0);
        gemm_batched(s, g2, true, false, 1.0, 0.0);
        gemm_batched(s, g3, false, false, -1.0, 1.0);
    }
}

// The matrices of a batch in two independent halves on two streams: one half's panels
// (latency-bound, few SMs busy) overlap the other half's trailing-update GEMMs.
// (measured at C4: 9.84 s of H2 build against 9.50 s on one stream -- the halves' smaller
// GEMM launches lose more than the overlap gains; kept behind env SPD_QR_2S=1)
static void qr_blocked_np_2s(cudaStream_t s, const std::vector<QrDesc>& d, int NP, int PW) {
    if (d.size() < 8 || !getenv("SPD_QR_2S")) {
        qr_blocked_np(s, d, NP, PW);
        SPD_CUDA(cudaStreamSynchronize(s));
        return;
    }
    static thread_local cudaStream_t s2 = nullptr;
    static thread_local cudaEvent_t ev[2];
    if (!s2) {
        SPD_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        SPD_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
        SPD_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    }
    std::vector<QrDesc> a, b;
    for (size_t i = 0; i < d.size(); ++i) (i & 1 ? b : a).push_back(d[i]);
    SPD_CUDA(cudaEventRecord(ev[0], s));
    SPD_CUDA(cudaStreamWaitEvent(s2, ev[0], 0));
    qr_blocked_np(s, a, NP, PW);
    {
        AllocStreamScope sc(s2);                      // the half's temporaries are ordered on s2
        qr_blocked_np(s2, b, NP, PW);
    }
    SPD_CUDA(cudaEventRecord(ev[1], s2));
    SPD_CUDA(cudaStreamWaitEvent(s, ev[1], 0));
    SPD_CUDA(cudaStreamSynchronize(s));
}

void qr_unpivoted_batched(cudaStream_t s, const std::vector<QrDesc>& d) {
    if (d.empty()) return;
    // default: 16-column panels in blocks of NP = 4 (64-column compact-WY trailing updates):
    // the panel's per-column latency is set by the cluster barrier and reductions, not by its
    // width, so half-width panels double the panels in flight (measured C4 H2 build 9.76 ->
    // 9.38 s).  env SPD_QR_PW=32 / SPD_QR_NP select the 32-column variants (A/B).
    const int pw = getenv("SPD_QR_PW") ? atoi(getenv("SPD_QR_PW")) : 16;
    const int np = getenv("SPD_QR_NP") ? atoi(getenv("SPD_QR_NP")) : (pw == 16 ? 4 : 2);
    if (pw == 16) { qr_blocked_np_2s(s, d, std::max(1, std::min(8, np)), 16); return; }
    if (np >= 1 && np <= 8 && np != 2) { qr_blocked_np_2s(s, d, np, QB); return; }
    // Panels are taken in pairs A = [p, p + 32), B = [p + 32, p + 64): A is factored, its
    // reflectors update B's columns only, B is factored, and the rest of the trailing
    // matrix gets ONE update with the combined 64-column compact-WY factor
    //   I - [V_A V_B] [T_A, -T_A (V_A^T V_B) T_B; 0, T_B] [V_A V_B]^T
    // (Schreiber-Van Loan), halving the trailing-matrix traffic of the 32-wide scheme.
    constexpr int QB2 = 2 * QB;
    int nmax = 0;
    size_t vtot = 0, wtot = 0;
    std::vector<size_t> voff(d.size()), woff(d.size());
    for (size_t i = 0; i < d.size(); ++i) {
        nmax = std::max(nmax, d[i].n);
        voff[i] = vtot; vtot += (size_t)d[i].m * QB2;
        woff[i] = wtot; wtot += (size_t)QB2 * d[i].n;
    }
    const size_t nd = d.size();
    DBuf<double> V(vtot), TA(nd * QB * QB), TB(nd * QB * QB), TAB(nd * QB2 * QB2), S(nd * QB * QB),
        X(nd * QB * QB), W(wtot), W2(wtot);
    double fl = 0;
    for (auto& q : d) fl += 2.0 * q.m * q.n * q.n - 2.0 / 3.0 * q.n * q.n * q.n;
    for (int p = 0; p < nmax; p += QB2) {
        V.zero(s);                                    // V_B's rows above its panel must be 0
        TAB.zero(s);
        std::vector<PanelDesc> pa, pb;
        std::vector<GemmDesc> n1, n2, n3, gs, gx, gt, g1, g2, g3;
        std::vector<CopyDesc> cp;
        std::vector<int> jbA(nd, 0), jbB(nd, 0);
        for (size_t i = 0; i < nd; ++i) {
            const QrDesc& q = d[i];
            const int kk = std::min(q.n, q.m);
            if (p >= kk) continue;
            jbA[i] = std::min(QB, kk - p);
            jbB[i] = jbA[i] == QB ? std::max(0, std::min(QB, kk - p - QB)) : 0;
            pa.push_back({q.A, q.m, q.n, q.ld, p, jbA[i], V.p + voff[i], q.m, TA.p + i * QB * QB});
            const int L = q.m - p;
            const int pB = p + jbA[i];
            const int nbB = std::min(QB, q.n - pB);     // B's columns (also when B is not factored)
            if (nbB > 0) {                              // B columns -= V_A T_A^T V_A^T B
                double* Ab = q.A + p + (size_t)pB * q.ld;
                n1.push_back({V.p + voff[i], Ab, W.p + woff[i], jbA[i], nbB, L, q.m, q.ld, QB2});
                n2.push_back({TA.p + i * QB * QB, W.p + woff[i], W2.p + woff[i], jbA[i], nbB, jbA[i], QB, QB2, QB2});
                n3.push_back({V.p + voff[i], W2.p + woff[i], Ab, L, nbB, jbA[i], q.m, QB2, q.ld});
            }
            if (jbB[i] > 0)
                pb.push_back({q.A, q.m, q.n, q.ld, pB, jbB[i], V.p + voff[i] + (size_t)QB * q.m + QB, q.m,
                              TB.p + i * QB * QB});
            const int pf = pB + nbB, nt = q.n - pf;     // far columns
            if (nt <= 0) continue;
            double* Af = q.A + p + (size_t)pf * q.ld;
            const int K = jbA[i] + jbB[i];
            if (jbB[i] > 0) {                           // T_AB from T_A, T_B, V_A^T V_B
                gs.push_back({V.p + voff[i], V.p + voff[i] + (size_t)QB * q.m, S.p + i * QB * QB, QB, jbB[i], L,
                              q.m, q.m, QB});
                gx.push_back({TA.p + i * QB * QB, S.p + i * QB * QB, X.p + i * QB * QB, QB, jbB[i], QB, QB, QB, QB});
                gt.push_back({X.p + i * QB * QB, TB.p + i * QB * QB, TAB.p + i * QB2 * QB2 + (size_t)QB * QB2, QB,
                              jbB[i], jbB[i], QB, QB, QB2});
                cp.push_back({TA.p + i * QB * QB, TAB.p + i * QB2 * QB2, QB, QB, QB, QB2, 0});
                cp.push_back({TB.p + i * QB * QB, TAB.p + i * QB2 * QB2 + QB + (size_t)QB * QB2, jbB[i], jbB[i], QB,
                              QB2, 0});
            } else {
                cp.push_back({TA.p + i * QB * QB, TAB.p + i * QB2 * QB2, jbA[i], jbA[i], QB, QB2, 0});
            }
            // W = V^T A_far ; W2 = T^T W ; A_far -= V W2   (K = 64 combined, or A alone)
            g1.push_back({V.p + voff[i], Af, W.p + woff[i], K, nt, L, q.m, q.ld, QB2});
            g2.push_back({TAB.p + i * QB2 * QB2, W.p + woff[i], W2.p + woff[i], K, nt, K, QB2, QB2, QB2});
            g3.push_back({V.p + voff[i], W2.p + woff[i], Af, L, nt, K, q.m, QB2, q.ld});
        }
        launch_panels(s, pa, p);
        gemm_batched(s, n1, true, false, 1.0, 0.0);
        gemm_batched(s, n2, true, false, 1.0, 0.0);
        gemm_batched(s, n3, false, false, -1.0, 1.0);
        launch_panels(s, pb, p + QB);
        gemm_batched(s, gs, true, false, 1.0, 0.0);
        gemm_batched(s, gx, false, false, 1.0, 0.0);
        gemm_batched(s, gt, false, false, -1.0, 0.0);
        copy_batched(s, cp, 1.0, false);
        gemm_batched(s, g1, true, false, 1.0, 0.0);
        gemm_batched(s, g2, true, false, 1.0, 0.0);
        gemm_batched(s, g3, false, false, -1.0, 1.0);
    }
    SPD_CUDA(cudaStreamSynchronize(s));
}

// R of tall matrices whose panels do not fit the 16-CTA cluster (m > 16 x 720 rows, e.g.
// the RPY proxy matrices with 3 dofs per proxy point): one level of TSQR -- row blocks
// factored separately, then the QR of their stacked triangles.  R is unique up to row
// signs, which neither the column pivots of the following QRCP nor R11^{-1} R12 see.
void qr_tall_batched(cudaStream_t s, const std::vector<QrDesc>& d) {
    static const int MAXROWS = getenv("SPD_TSQR_ROWS") ? atoi(getenv("SPD_TSQR_ROWS"))
                                                        : 16 * ((180 * 1024) / (QB * (int)sizeof(double)));
    std::vector<QrDesc> direct, blocks, stacks;
    struct Big { QrDesc q; int nb; int64_t soff; };
    std::vector<Big> big;
    int64_t stot = 0;
    for (const auto& q : d) {
        const int nb = ceil_div(q.m, MAXROWS);
        if (nb <= 1 || (int64_t)nb * q.n > MAXROWS || ceil_div(q.m, nb) < q.n) { direct.push_back(q); continue; }
        big.push_back({q, nb, stot});
        stot += (int64_t)nb * q.n * q.n;
    }
    if (!direct.empty()) qr_unpivoted_batched(s, direct);
    if (big.empty()) return;
    DBuf<double> S(std::max<int64_t>(1, stot));
    S.zero(s);
    std::vector<CopyDesc> up, back;
    std::vector<MatDesc> low;
    for (const auto& b : big) {
        const int rb = ceil_div(b.q.m, b.nb), n = b.q.n, ls = b.nb * n;
        for (int k = 0; k < b.nb; ++k) {
            const int r0 = k * rb, rows = std::min(rb, b.q.m - r0);
            blocks.push_back({b.q.A + r0, rows, n, b.q.ld});
            up.push_back({b.q.A + r0, S.p + b.soff + (int64_t)k * n, n, n, b.q.ld, ls, 0});   // block's R
            low.push_back({S.p + b.soff + (int64_t)k * n, n, n, ls});
        }
        stacks.push_back({S.p + b.soff, ls, n, ls});
        back.push_back({S.p + b.soff, b.q.A, n, n, ls, b.q.ld, 0});
    }
    qr_unpivoted_batched(s, blocks);
    copy_batched(s, up, 1.0, false);
    zero_lower_batched(s, low);                      // keep the triangles only
    qr_unpivoted_batched(s, stacks);
    copy_batched(s, back, 1.0, false);               // R (upper n x n) back into the top rows
}

// ================================================================= FORM Q
__global__ void __launch_bounds__(256) formq_kernel(const FormQDesc* descs) {
    const FormQDesc d = descs[blockIdx.x];
    const int r = *d.rank;
    const int m = d.m;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = warp; j < r; j += nw)
        for (int i = lane; i < m; i += 32) d.Q[i + (size_t)j * d.ldq] = (i == j) ? 1.0 : 0.0;
    __syncthreads();
    for (int t = r - 1; t >= 0; --t) {
        const double* v = d.A + (size_t)t * d.lda;
        const double beta = d.beta[t];
        for (int j = t + warp; j < r; j += nw) {
            double* q = d.Q + (size_t)j * d.ldq;
            double s = (lane == 0) ? q[t] : 0.0;
            for (int i = t + 1 + lane; i < m; i += 32) s += v[i] * q[i];
            s = warp_sum(s) * beta;
            if (lane == 0) q[t] -= s;
            for (int i = t + 1 + lane; i < m; i += 32) q[i] -= s * v[i];
        }
        __syncthreads();
    }
}

void formq_batched(cudaStream_t s, const std::vector<FormQDesc>& d) {
    if (d.empty()) return;
    DevArray<FormQDesc> dd(s, d);
    ProfScope prof(s, "formq", 0, 0);
    formq_kernel<<<(unsigned)d.size(), 256, 0, s>>>(dd.p);
    SPD_LAUNCH();
}

// ================================================================= copies
__global__ void copy_kernel(const CopyDesc* descs, double alpha, int accumulate) {
    const CopyDesc d = descs[blockIdx.y];
    const int64_t total = (int64_t)d.m * d.n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(e % d.m), j = (int)(e / d.m);
        double v = d.trans ? d.A[j + (size_t)i * d.lda] : d.A[i + (size_t)j * d.lda];
        double* c = d.C + i + (size_t)j * d.ldc;
        *c = accumulate ? *c + alpha * v : alpha * v;
    }
}

void copy_batched(cudaStream_t s, const std::vector<CopyDesc>& d, double alpha, bool accumulate) {
    if (d.empty()) return;
    DevArray<CopyDesc> dd(s, d);
    ProfScope prof(s, "copy", 0, 0);
    for (size_t off = 0; off < d.size(); off += 65535) {
        unsigned ny = (unsigned)std::min<size_t>(65535, d.size() - off);
        copy_kernel<<<dim3(8, ny), 256, 0, s>>>(dd.p + off, alpha, accumulate ? 1 : 0);
        SPD_LAUNCH();
    }
}

__global__ void add_identity_kernel(const MatDesc* descs) {
    const MatDesc d = descs[blockIdx.x];
    for (int i = threadIdx.x; i < min(d.m, d.n); i += blockDim.x) d.A[i + (size_t)i * d.ld] += 1.0;
}
void set_identity_plus(cudaStream_t s, const std::vector<MatDesc>& d) {
    if (d.empty()) return;
    DevArray<MatDesc> dd(s, d);
    add_identity_kernel<<<(unsigned)d.size(), 128, 0, s>>>(dd.p);
    SPD_LAUNCH();
}

__global__ void zero_lower_kernel(const MatDesc* descs) {
    const MatDesc d = descs[blockIdx.x];
    for (int j = 0; j < d.n; ++j)
        for (int i = j + 1 + threadIdx.x; i < d.m; i += blockDim.x) d.A[i + (size_t)j * d.ld] = 0.0;
}
void zero_lower_batched(cudaStream_t s, const std::vector<MatDesc>& d) {
    if (d.empty()) return;
    DevArray<MatDesc> dd(s, d);
    zero_lower_kernel<<<(unsigned)d.size(), 256, 0, s>>>(dd.p);
    SPD_LAUNCH();
}

__global__ void zero_upper_kernel(const MatDesc* descs) {
    const MatDesc d = descs[blockIdx.x];
    for (int j = 1; j < d.n; ++j)
        for (int i = threadIdx.x; i < min(j, d.m); i += blockDim.x) d.A[i + (size_t)j * d.ld] = 0.0;
}
void zero_upper_batched(cudaStream_t s, const std::vector<MatDesc>& d) {
    if (d.empty()) return;
    DevArray<MatDesc> dd(s, d);
    zero_upper_kernel<<<(unsigned)d.size(), 128, 0, s>>>(dd.p);
    SPD_LAUNCH();
}

}  // namespace spd
