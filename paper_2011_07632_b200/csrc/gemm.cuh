// gemm.cuh -- pipelined FP64 DMMA GEMM tile kernel (sm_100a), shared by dense.cu.
//
// C = alpha op(A) op(B) + beta C on one BM x BN output tile per CTA, K in chunks of
// 16 through a STAGES-deep cp.async (LDGSTS) shared-memory ring, warp tiles of
// WM x WN computed with mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; tcgen05 has no f64
// kind, so this is the FP64 tensor path on Blackwell).  Shared-memory layouts are
// chosen per operand so that the fragment loads are 2 wavefronts (optimal for a
// 256-byte warp access) and the global reads are along the contiguous dimension:
//   A col-major (m contiguous):  As[k][BM + 8]      A^T (k contiguous): As[m][BK + 4]
//   B col-major (k contiguous):  Bs[n][BK + 4]      B^T (n contiguous): Bs[k][BN + 8]
// Copies are 8-byte cp.async with zero fill past the edges (any ld / alignment).
#pragma once
#include "common.cuh"

namespace spd {

struct TileRef {
    int desc, tm, tn;
    int kb, ke;            // K range of this tile
    double* P; int ldp;    // split-K: raw partial tile goes to P (ld ldp); nullptr: C = alpha acc + beta C
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" :: "r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" :: "n"(N)); }

template <int BM, int BN, bool TA, bool TB>
struct GemmSmem {
    static constexpr int BK = 16;
    static constexpr int A_LD = TA ? BK + 4 : BM + 8;
    static constexpr int B_LD = TB ? BN + 8 : BK + 4;
    static constexpr int A_ELEMS = TA ? BM * A_LD : BK * A_LD;
    static constexpr int B_ELEMS = TB ? BK * B_LD : BN * B_LD;
};

// PRE: the C tile (beta != 0) is loaded at kernel start, so its read latency overlaps
// the A/B loads (short-K updates such as the rank-32 trailing update of the blocked QR)
template <int BM, int BN, int WM, int WN, int STAGES, bool TA, bool TB, bool PRE = false>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
gemm_pipe_kernel(const GemmDesc* __restrict__ descs, const TileRef* __restrict__ tiles, double alpha, double beta) {
    using SM = GemmSmem<BM, BN, TA, TB>;
    constexpr int BK = SM::BK, NWN = BN / WN, NT = (BM / WM) * (BN / WN) * 32;
    constexpr int FM = WM / 8, FN = WN / 8;
    extern __shared__ double smem[];
    double* As = smem;
    double* Bs = smem + STAGES * SM::A_ELEMS;
    const TileRef tr = tiles[blockIdx.x];
    const GemmDesc d = descs[tr.desc];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int wm = warp / NWN, wn = warp % NWN;
    const int m0 = tr.tm * BM, n0 = tr.tn * BN;
    const int kb = tr.kb, ke = tr.ke;
    const int nk = ke > kb ? (ke - kb + BK - 1) / BK : 0;

    auto load_stage = [&](int st, int k0) {
        double* as = As + st * SM::A_ELEMS;
        double* bs = Bs + st * SM::B_ELEMS;
#pragma unroll
        for (int e = tid; e < BM * BK; e += NT) {
            int m, k;
            if (TA) { k = e % BK; m = e / BK; } else { m = e % BM; k = e / BM; }
            const int gm = m0 + m, gk = k0 + k;
            const bool ok = gm < d.m && gk < ke;
            const double* src = TA ? d.A + (size_t)gm * d.lda + gk : d.A + gm + (size_t)gk * d.lda;
            cp_async8(TA ? as + m * SM::A_LD + k : as + k * SM::A_LD + m, ok ? src : d.A, ok);
        }
#pragma unroll
        for (int e = tid; e < BN * BK; e += NT) {
            int n, k;
            if (TB) { n = e % BN; k = e / BN; } else { k = e % BK; n = e / BK; }
            const int gn = n0 + n, gk = k0 + k;
            const bool ok = gn < d.n && gk < ke;
            const double* src = TB ? d.B + gn + (size_t)gk * d.ldb : d.B + gk + (size_t)gn * d.ldb;
            cp_async8(TB ? bs + k * SM::B_LD + n : bs + n * SM::B_LD + k, ok ? src : d.B, ok);
        }
    };

    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double cpre[PRE ? FM : 1][PRE ? FN : 1][2];
    if (PRE) {
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int gi = m0 + wm * WM + i * 8 + g;
                    const int gj = n0 + wn * WN + j * 8 + 2 * q + h;
                    cpre[PRE ? i : 0][PRE ? j : 0][h] = (gi < d.m && gj < d.n && !tr.P) ? d.C[gi + (size_t)gj * d.ldc] : 0.0;
                }
    }

#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nk) load_stage(st, kb + st * BK);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int kn = kt + STAGES - 1;
            if (kn < nk) load_stage(kn % STAGES, kb + kn * BK);
            cp_async_commit();
        }
        const double* as = As + (kt % STAGES) * SM::A_ELEMS;
        const double* bs = Bs + (kt % STAGES) * SM::B_ELEMS;
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            const int k = ks * 4 + q;
            double af[FM], bf[FN];
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                const int m = wm * WM + i * 8 + g;
                af[i] = TA ? as[m * SM::A_LD + k] : as[k * SM::A_LD + m];
            }
#pragma unroll
            for (int j = 0; j < FN; ++j) {
                const int n = wn * WN + j * 8 + g;
                bf[j] = TB ? bs[k * SM::B_LD + n] : bs[n * SM::B_LD + k];
            }
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int gi = m0 + wm * WM + i * 8 + g;
                const int gj = n0 + wn * WN + j * 8 + 2 * q + h;
                if (gi < d.m && gj < d.n) {
                    if (tr.P) {
                        tr.P[gi + (size_t)gj * tr.ldp] = acc[i][j][h];
                    } else {
                        double* c = d.C + gi + (size_t)gj * d.ldc;
                        const double cold = PRE ? cpre[PRE ? i : 0][PRE ? j : 0][h] : (beta == 0.0 ? 0.0 : *c);
                        *c = (beta == 0.0 ? 0.0 : beta * cold) + alpha * acc[i][j][h];
                    }
                }
            }
}

// Persistent variant for short-K updates C = alpha A B + beta C (the blocked QR's rank-64
// trailing updates: K = 64 is only four 16-deep chunks, so a one-tile CTA spends most of
// its life filling and draining its pipeline).  Each CTA walks the tiles
// blockIdx.x, blockIdx.x + gridDim.x, ... and its cp.async ring of (tile, k-chunk) stages
// runs ACROSS tile boundaries: the next tile's first chunks (and its C values, loaded into
// registers) are in flight while the current tile finishes.  Same per-tile arithmetic and
// summation order as gemm_pipe_kernel (bitwise-equal C).  No split-K (tr.P unused).
template <int BM, int BN, int WM, int WN, int STAGES, bool TA, bool TB>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
gemm_persist_kernel(const GemmDesc* __restrict__ descs, const TileRef* __restrict__ tiles, int ntiles, double alpha,
                    double beta) {
    using SM = GemmSmem<BM, BN, TA, TB>;
    constexpr int BK = SM::BK, NWN = BN / WN, NT = (BM / WM) * (BN / WN) * 32;
    constexpr int FM = WM / 8, FN = WN / 8;
    extern __shared__ double smem[];
    double* As = smem;
    double* Bs = smem + STAGES * SM::A_ELEMS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int wm = warp / NWN, wn = warp % NWN;
    // the producer cursor (tile, chunk) runs STAGES - 1 chunks ahead of the consumer
    int pt = blockIdx.x, pc = 0;
    auto nchunks = [&](int t) { const TileRef& r = tiles[t]; return r.ke > r.kb ? (r.ke - r.kb + BK - 1) / BK : 0; };
    auto produce = [&](int st) {
        while (pt < ntiles && pc >= nchunks(pt)) { pt += gridDim.x; pc = 0; }
        if (pt < ntiles) {
            const TileRef tr = tiles[pt];
            const GemmDesc d = descs[tr.desc];
            const int m0 = tr.tm * BM, n0 = tr.tn * BN, k0 = tr.kb + pc * BK, ke = tr.ke;
            double* as = As + st * SM::A_ELEMS;
            double* bs = Bs + st * SM::B_ELEMS;
#pragma unroll
            for (int e = tid; e < BM * BK; e += NT) {
                int m, k;
                if (TA) { k = e % BK; m = e / BK; } else { m = e % BM; k = e / BM; }
                const int gm = m0 + m, gk = k0 + k;
                const bool ok = gm < d.m && gk < ke;
                const double* s = TA ? d.A + (size_t)gm * d.lda + gk : d.A + gm + (size_t)gk * d.lda;
                cp_async8(TA ? as + m * SM::A_LD + k : as + k * SM::A_LD + m, ok ? s : d.A, ok);
            }
#pragma unroll
            for (int e = tid; e < BN * BK; e += NT) {
                int n, k;
                if (TB) { n = e % BN; k = e / BN; } else { k = e % BK; n = e / BK; }
                const int gn = n0 + n, gk = k0 + k;
                const bool ok = gn < d.n && gk < ke;
                const double* s = TB ? d.B + gn + (size_t)gk * d.ldb : d.B + gk + (size_t)gn * d.ldb;
                cp_async8(TB ? bs + k * SM::B_LD + n : bs + n * SM::B_LD + k, ok ? s : d.B, ok);
            }
            ++pc;
        }
        cp_async_commit();
    };
    double acc[FM][FN][2], cpre[FM][FN][2];
    auto load_c = [&](int t) {                   // C values of tile t into registers (beta != 0)
        const TileRef tr = tiles[t];
        const GemmDesc d = descs[tr.desc];
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int gi = tr.tm * BM + wm * WM + i * 8 + g;
                    const int gj = tr.tn * BN + wn * WN + j * 8 + 2 * q + h;
                    cpre[i][j][h] = (beta != 0.0 && gi < d.m && gj < d.n) ? d.C[gi + (size_t)gj * d.ldc] : 0.0;
                }
    };
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) produce(st);
    int slot = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int nk = nchunks(t);
        load_c(t);
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int kt = 0; kt < nk; ++kt) {
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            produce((slot + STAGES - 1) % STAGES);
            const double* as = As + slot * SM::A_ELEMS;
            const double* bs = Bs + slot * SM::B_ELEMS;
            slot = (slot + 1) % STAGES;
#pragma unroll
            for (int ks = 0; ks < BK / 4; ++ks) {
                const int k = ks * 4 + q;
                double af[FM], bf[FN];
#pragma unroll
                for (int i = 0; i < FM; ++i) {
                    const int m = wm * WM + i * 8 + g;
                    af[i] = TA ? as[m * SM::A_LD + k] : as[k * SM::A_LD + m];
                }
#pragma unroll
                for (int j = 0; j < FN; ++j) {
                    const int n = wn * WN + j * 8 + g;
                    bf[j] = TB ? bs[k * SM::B_LD + n] : bs[n * SM::B_LD + k];
                }
#pragma unroll
                for (int i = 0; i < FM; ++i)
#pragma unroll
                    for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
        }
        const TileRef tr = tiles[t];
        const GemmDesc d = descs[tr.desc];
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int gi = tr.tm * BM + wm * WM + i * 8 + g;
                    const int gj = tr.tn * BN + wn * WN + j * 8 + 2 * q + h;
                    if (gi < d.m && gj < d.n)
                        d.C[gi + (size_t)gj * d.ldc] = (beta == 0.0 ? 0.0 : beta * cpre[i][j][h]) + alpha * acc[i][j][h];
                }
    }
    cp_async_wait<0>();
}

template <int BM, int BN, int WM, int WN, int STAGES, bool TA, bool TB>
constexpr size_t gemm_pipe_smem() {   // (independent of PRE)
    using SM = GemmSmem<BM, BN, TA, TB>;
    return sizeof(double) * (size_t)STAGES * (SM::A_ELEMS + SM::B_ELEMS);
}

}  // namespace spd
