// kblock.cu -- on-the-fly kernel-block x multi-vector products (product path).
//
// Y_e += K(P_t, P_s) X_e for every (target t, source s) entry e, where P_t, P_s
// are point sets (tree-order points for near-field leaf blocks, skeleton points
// for Type-3 couplings, PAPER.md eqn:uniformbasis_h2 with B^{H2}_ij =
// K(X_{J_i}, X_{J_j}) never stored -- north star "evaluated on the fly").
// The kernel tile is evaluated in registers/shared memory and contracted with
// FP64 DMMA (mma.sync m8n8k4).  Owner-computes: a CTA owns a (target rows x
// columns) tile and accumulates over all its entries, flushing when the output
// pointer changes, so there are no atomics and the summation order is fixed.
#include "common.cuh"
#include "kblock.cuh"
#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace spd {

constexpr int KB_M = 64, KB_K = 16;   // simple kernel: 64-row tiles, 16-source chunks

// work item: target row tile tm, column tile tn, entries [eb, ee) of the target;
// pslot >= 0: the tile is a segment of a split target, its sum goes to partial slot
// pslot (64 x NC, ld 64) and kb_reduce_kernel adds the segments in order into Y
struct KbWork { int target, tm, tn, eb, ee, pslot; };

template <int KID>
__device__ __forceinline__ double kval(const KernelParams& kp, double r2) {
    if (KID == SPD_K_GAUSSIAN) return exp(-r2 * kp.inv_l2);
    if (KID == SPD_K_MATERN32) { const double t = sqrt(r2) * kp.sqrt3_inv_l; return (1.0 + t) * exp(-t); }
    if (KID == SPD_K_EXPONENTIAL) return exp(-sqrt(r2) * kp.inv_l);
    return rsqrt(r2 + kp.l2);
}

// CTA tile: KB_M target rows x NC columns, NC/32 * 2 warps (each 32 x 32 = 4x4 DMMA
// m8n8k4 blocks).  Per source chunk of 16 points: the 64x16 kernel tile is
// evaluated once into shared memory (shared by all column warps) and contracted
// with the 16 x NC slice of X; the next chunk's X slice and coordinates are
// prefetched into registers while the current chunk is evaluated/contracted.
// sources per chunk of the kblock kernel: 32 for the 160-column tile (half the barriers per
// flop; one CTA per SM), 16 otherwise
__host__ __device__ constexpr int kb_chunk(int NC) { return NC == 160 ? 32 : 16; }
__host__ __device__ constexpr int kb_smem_bytes(int NC) {
    return (int)sizeof(double) * (kb_chunk(NC) * (KB_M + 8) + NC * (kb_chunk(NC) + 4) + 4 * kb_chunk(NC));
}

template <class F>
static void kb_attr(F* f, int bytes) {
    if (bytes > 48 * 1024) SPD_CUDA(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

template <int KID, int NC>
__global__ void __launch_bounds__(2 * NC, NC == 32 ? 6 : (NC == 160 ? 1 : 256 / NC)) kblock_kernel(
    KernelParams kp, double shift, int d, const KbBlock* __restrict__ blocks,
    const KbTarget* __restrict__ targets, const KbEntry* __restrict__ entries,
    const KbWork* __restrict__ work, double* __restrict__ partial) {
    constexpr int NT = 2 * NC;                  // threads
    constexpr int KK = kb_chunk(NC);            // sources per chunk (32 for the 160-column tile)
    constexpr int WN = NC / 32;                 // warps along columns
    constexpr int XPT = KK * NC / NT;         // X values per thread per chunk (= 8)
    constexpr int EST = NT / KB_M;              // kernel-tile columns kc = tid / 64 + EST u (NC / 32 of them)
    extern __shared__ double kbsm[];              // dynamic: Ks | Xs | Sx (kb_smem_bytes)
    double (*Ks)[KB_M + 8] = reinterpret_cast<double (*)[KB_M + 8]>(kbsm);               // row stride = 8 (mod 16) doubles: fragment reads in 2 wavefronts
    double (*Xs)[KK + 4] = reinterpret_cast<double (*)[KK + 4]>(kbsm + KK * (KB_M + 8));  // kc contiguous: conflict-free writes and reads
    double (*Sx)[KK] = reinterpret_cast<double (*)[KK]>(kbsm + KK * (KB_M + 8) + NC * (KK + 4));   // coordinates (RPY: + component row)
    const KbWork wk = work[blockIdx.x];
    const KbTarget tg = targets[wk.target];
    const KbBlock tb = blocks[tg.blk];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, q = lane & 3, wm = warp / WN, wn = warp % WN;
    double* part = wk.pslot >= 0 ? partial + (size_t)wk.pslot * KB_M * NC : nullptr;
    const int r0 = wk.tm * KB_M, c0 = wk.tn * NC;
    const int nrows = min(KB_M, tb.n - r0);
    const int er = tid & (KB_M - 1), ec0 = tid / KB_M;
    double rx[4] = {0.0, 0.0, 0.0, 0.0};
    if (er < nrows)
        for (int a = 0; a < d; ++a) rx[a] = tb.x[(size_t)a * tb.ds + r0 + er];
    const int64_t rid = tb.id0 >= 0 ? tb.id0 + r0 + er : -1;

    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    double xr[XPT], sr = 0.0;
    for (int e = wk.eb; e < wk.ee; ++e) {
        const KbEntry en = entries[e];
        if (c0 < en.ncols) {
            const KbBlock sb = blocks[en.src];
            const int ncols = min(NC, en.ncols - c0);
            const bool use_shift = (shift != 0.0) && rid >= 0 && sb.id0 >= 0;
            auto load = [&](int k0) {
                const int nk = min(KK, sb.n - k0);
#pragma unroll
                for (int u = 0; u < XPT; ++u) {
                    const int idx = tid + u * NT;
                    const int kk = idx % KK, j = idx / KK;
                    xr[u] = (kk < nk && j < ncols) ? __ldg(en.X + k0 + kk + (size_t)(c0 + j) * en.ldx) : 0.0;
                }
                if (tid < KK * 4) {
                    const int a = tid / KK, c = tid % KK;
                    sr = (a < d && c < nk) ? __ldg(sb.x + (size_t)a * sb.ds + k0 + c) : 0.0;
                }
            };
            load(0);
            for (int k0 = 0; k0 < sb.n; k0 += KK) {
                const int nk = min(KK, sb.n - k0);
                __syncthreads();
#pragma unroll
                for (int u = 0; u < XPT; ++u) {
                    const int idx = tid + u * NT;
                    Xs[idx / KK][idx % KK] = xr[u];
                }
                if (tid < KK * 4) Sx[tid / KK][tid % KK] = sr;
                __syncthreads();
                if (k0 + KK < sb.n) load(k0 + KK);          // prefetch the next chunk
                if (en.kmode == 0) {
#pragma unroll
                    for (int kc = ec0; kc < KK; kc += EST) {
                        const double d0 = rx[0] - Sx[0][kc], d1 = rx[1] - Sx[1][kc], d2 = rx[2] - Sx[2][kc];
                        double kv;
                        if constexpr (KID == SPD_K_RPY) kv = rpy_entry(kp, d0, d1, d2, (int)rx[3], (int)Sx[3][kc]);
                        else kv = kval<KID>(kp, d0 * d0 + d1 * d1 + d2 * d2);
                        if (use_shift && rid == sb.id0 + k0 + kc) kv += shift;
                        Ks[kc][er] = (er < nrows && kc < nk) ? kv : 0.0;
                    }
                } else {                          // stored block (symmetric store): loads only
                    const int r = r0 + er;
                    constexpr int EPT = (KK + EST - 1) / EST;
                    double kv[EPT];
#pragma unroll
                    for (int c = 0; c < EPT; ++c) {
                        const int kc = ec0 + c * EST, cc = k0 + kc;
                        const double* a = en.kmode == 1
                            ? en.kst + (size_t)(r >> 5) * 32 * en.kld + (size_t)cc * 32 + (r & 31)
                            : en.kst + (size_t)(cc >> 5) * 32 * en.kld + (size_t)r * 32 + (cc & 31);
                        kv[c] = (kc < KK && er < nrows && kc < nk) ? __ldg(a) : 0.0;
                    }
#pragma unroll
                    for (int c = 0; c < EPT; ++c)
                        if (ec0 + c * EST < KK) Ks[ec0 + c * EST][er] = kv[c];
                }
                __syncthreads();
#pragma unroll
                for (int ks = 0; ks < KK / 4; ++ks) {
                    double af[4], bf[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) af[a] = Ks[ks * 4 + q][wm * 32 + a * 8 + g];
#pragma unroll
                    for (int b = 0; b < 4; ++b) bf[b] = Xs[wn * 32 + b * 8 + g][ks * 4 + q];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
                }
            }
        }
        const bool flush = (e + 1 == wk.ee) || entries[e + 1].Y != en.Y;
        if (flush) {
            if (part) {                       // segment of a split target: raw tile to its slot
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            int i = wm * 32 + a * 8 + g, j = wn * 32 + b * 8 + 2 * q + h;
                            part[i + (size_t)j * KB_M] = acc[a][b][h];
                        }
            } else if (c0 < en.ncols) {
                const int ncols = min(NC, en.ncols - c0);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            int i = wm * 32 + a * 8 + g, j = wn * 32 + b * 8 + 2 * q + h;
                            if (i < nrows && j < ncols) en.Y[r0 + i + (size_t)(c0 + j) * en.ldy] += acc[a][b][h];
                        }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        }
    }
}

// ---------------------------------------------------------------- TMA-staged variant
// The same tile, work list and summation order as kblock_kernel; the X slice of every
// source chunk (KK sources x NC columns) is staged by the tensor-memory accelerator
// instead of a register prefetch: one elected thread issues cp.async.bulk.tensor.2d of
// 16 x NC boxes (128-byte swizzle, rows past the buffer zero-filled) into a two-stage
// shared-memory ring whose mbarrier carries the transaction count, one chunk ahead of
// the evaluation.  Entries whose X buffer has no tensor map (tmi < 0: an odd leading
// dimension, too many buffers) fill the same swizzled stage with plain loads.
__device__ __forceinline__ unsigned kb_su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void kb_mbar_init(uint64_t* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(kb_su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void kb_mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(kb_su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void kb_mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile("{\n\t.reg .pred p;\n"
                 "KBW_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra KBW_%=;\n}" :: "r"(kb_su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void kb_tma2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(kb_su32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(kb_su32(bar))
                 : "memory");
}
// element (column j, source kk < 16) of a 16 x NC sub-tile in the TMA 128-byte swizzle:
// column j is a 128-byte row, its 16-byte chunk index XOR (j mod 8)
__device__ __forceinline__ int kb_swz(int j, int kk) { return j * 16 + ((((kk >> 1) ^ (j & 7)) << 1) | (kk & 1)); }

// sources per chunk of the TMA kernel = the register kernel's.  A box must start at a
// 16-byte aligned row (an odd starting row faults), so a stage holds KK / 16 + 1 sub-tiles:
// a chunk starting at an odd row is loaded from the row before it, one sub-tile more, and
// read with a one-row offset.
__host__ __device__ constexpr int kb_tma_chunk(int NC) { return kb_chunk(NC); }
__host__ __device__ constexpr int kb_tma_nsub(int NC) { return kb_tma_chunk(NC) / 16 + 1; }
__host__ __device__ constexpr int kb_tma_smem_bytes(int NC) {
    return 1024 + (int)sizeof(double) * (2 * kb_tma_nsub(NC) * 16 * NC + kb_tma_chunk(NC) * (KB_M + 8) + 4 * kb_tma_chunk(NC));
}

template <int KID, int NC, bool MIX>
__global__ void __launch_bounds__(2 * NC, NC == 32 ? 6 : (NC == 160 ? 1 : 256 / NC)) kblock_tma_kernel(
    KernelParams kp, double shift, int d, const KbBlock* __restrict__ blocks,
    const KbTarget* __restrict__ targets, const KbEntry* __restrict__ entries,
    const KbWork* __restrict__ work, double* __restrict__ partial, const __grid_constant__ KbTma tm) {
    constexpr int NT = 2 * NC;
    constexpr int KK = kb_tma_chunk(NC);
    constexpr int WN = NC / 32;
    constexpr int EST = NT / KB_M;
    constexpr int NSUB = kb_tma_nsub(NC);
    constexpr int XST = NSUB * 16 * NC;           // doubles per stage (NSUB sub-tiles of 16 x NC)
    extern __shared__ unsigned char kbraw[];
    double* const Xst = reinterpret_cast<double*>(kbraw + ((1024u - (kb_su32(kbraw) & 1023u)) & 1023u));
    double (*Ks)[KB_M + 8] = reinterpret_cast<double (*)[KB_M + 8]>(Xst + 2 * XST);
    double (*Sx)[KK] = reinterpret_cast<double (*)[KK]>(Xst + 2 * XST + KK * (KB_M + 8));
    __shared__ __align__(8) uint64_t full[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        kb_mbar_init(&full[0], 1);
        kb_mbar_init(&full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const KbWork wk = work[blockIdx.x];
    const KbTarget tg = targets[wk.target];
    const KbBlock tb = blocks[tg.blk];
    const int g = lane >> 2, q = lane & 3, wm = warp / WN, wn = warp % WN;
    double* part = wk.pslot >= 0 ? partial + (size_t)wk.pslot * KB_M * NC : nullptr;
    const int r0 = wk.tm * KB_M, c0 = wk.tn * NC;
    const int nrows = min(KB_M, tb.n - r0);
    const int er = tid & (KB_M - 1), ec0 = tid / KB_M;
    double rx[4] = {0.0, 0.0, 0.0, 0.0};
    if (er < nrows)
        for (int a = 0; a < d; ++a) rx[a] = tb.x[(size_t)a * tb.ds + r0 + er];
    const int64_t rid = tb.id0 >= 0 ? tb.id0 + r0 + er : -1;

    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    constexpr int XPT = KK * NC / NT;             // X values per thread per chunk (entries without a map)
    unsigned cc = 0, use0 = 0, use1 = 0;          // chunk counter, TMA completions per stage
    double xr[MIX ? XPT : 1], sr = 0.0;          // MIX: some entries have no tensor map
    for (int e = wk.eb; e < wk.ee; ++e) {
        const KbEntry en = entries[e];
        if (c0 < en.ncols) {
            const KbBlock sb = blocks[en.src];
            const int ncols = min(NC, en.ncols - c0);
            const bool use_shift = (shift != 0.0) && rid >= 0 && sb.id0 >= 0;
            const bool tma = !MIX || en.tmi >= 0;
            const int dl = tma ? (en.tr & 1) : 0;      // row offset of the chunk in its stage
            auto issue = [&](int k0, unsigned c) {      // one thread: the chunk's boxes
                double* dst = Xst + (c & 1) * XST;
                const int nsub = KK / 16 + dl;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                kb_mbar_expect(&full[c & 1], (unsigned)nsub * tm.box_bytes[en.tmi]);
                for (int sub = 0; sub < nsub; ++sub)
                    kb_tma2d(dst + sub * 16 * NC, &tm.map[en.tmi], en.tr - dl + k0 + 16 * sub, c0, &full[c & 1]);
            };
            auto load_sx = [&](int k0) {                // + the X slice of entries without a map
                const int nk = min(KK, sb.n - k0);
                if constexpr (MIX) if (!tma) {
#pragma unroll
                    for (int u = 0; u < XPT; ++u) {
                        const int idx = tid + u * NT;
                        const int kk = idx % KK, j = idx / KK;
                        xr[u] = (kk < nk && j < ncols) ? __ldg(en.X + k0 + kk + (size_t)(c0 + j) * en.ldx) : 0.0;
                    }
                }
                if (tid < KK * 4) {
                    const int a = tid / KK, c = tid % KK;
                    sr = (a < d && c < nk) ? __ldg(sb.x + (size_t)a * sb.ds + k0 + c) : 0.0;
                }
            };
            if (tma && tid == 0) issue(0, cc);
            load_sx(0);
            for (int k0 = 0; k0 < sb.n; k0 += KK) {
                const int nk = min(KK, sb.n - k0);
                __syncthreads();
                if constexpr (MIX) if (!tma) {            // prefetched registers into the swizzled stage
                    double* dst = Xst + (cc & 1) * XST;
#pragma unroll
                    for (int u = 0; u < XPT; ++u) {
                        const int idx = tid + u * NT;
                        const int kk = idx % KK, j = idx / KK;
                        dst[(kk >> 4) * 16 * NC + kb_swz(j, kk & 15)] = xr[u];
                    }
                }
                if (tid < KK * 4) Sx[tid / KK][tid % KK] = sr;
                __syncthreads();
                if (k0 + KK < sb.n) {                     // stage the next chunk
                    if (tma && tid == 0) issue(k0 + KK, cc + 1);
                    load_sx(k0 + KK);
                }
                if (en.kmode == 0) {
#pragma unroll
                    for (int kc = ec0; kc < KK; kc += EST) {
                        const double d0 = rx[0] - Sx[0][kc], d1 = rx[1] - Sx[1][kc], d2 = rx[2] - Sx[2][kc];
                        double kv;
                        if constexpr (KID == SPD_K_RPY) kv = rpy_entry(kp, d0, d1, d2, (int)rx[3], (int)Sx[3][kc]);
                        else kv = kval<KID>(kp, d0 * d0 + d1 * d1 + d2 * d2);
                        if (use_shift && rid == sb.id0 + k0 + kc) kv += shift;
                        Ks[kc][er] = (er < nrows && kc < nk) ? kv : 0.0;
                    }
                } else {
                    const int r = r0 + er;
                    constexpr int EPT = (KK + EST - 1) / EST;
                    double kv[EPT];
#pragma unroll
                    for (int c = 0; c < EPT; ++c) {
                        const int kc = ec0 + c * EST, cq = k0 + kc;
                        const double* a = en.kmode == 1
                            ? en.kst + (size_t)(r >> 5) * 32 * en.kld + (size_t)cq * 32 + (r & 31)
                            : en.kst + (size_t)(cq >> 5) * 32 * en.kld + (size_t)r * 32 + (cq & 31);
                        kv[c] = (kc < KK && er < nrows && kc < nk) ? __ldg(a) : 0.0;
                    }
#pragma unroll
                    for (int c = 0; c < EPT; ++c)
                        if (ec0 + c * EST < KK) Ks[ec0 + c * EST][er] = kv[c];
                }
                __syncthreads();
                if (tma) {
                    if (cc & 1) kb_mbar_wait(&full[1], use1++ & 1);
                    else kb_mbar_wait(&full[0], use0++ & 1);
                }
                const double* xs = Xst + (cc & 1) * XST;
#pragma unroll
                for (int ks = 0; ks < KK / 4; ++ks) {
                    double af[4], bf[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) af[a] = Ks[ks * 4 + q][wm * 32 + a * 8 + g];
                    const int kq = ks * 4 + q + dl;
                    const int xo = (kq >> 4) * 16 * NC + ((((kq & 15) >> 1) ^ g) << 1) + (kq & 1);
#pragma unroll
                    for (int b = 0; b < 4; ++b) bf[b] = xs[xo + (wn * 32 + b * 8 + g) * 16];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
                }
                ++cc;
            }
        }
        const bool flush = (e + 1 == wk.ee) || entries[e + 1].Y != en.Y;
        if (flush) {
            if (part) {
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            int i = wm * 32 + a * 8 + g, j = wn * 32 + b * 8 + 2 * q + h;
                            part[i + (size_t)j * KB_M] = acc[a][b][h];
                        }
            } else if (c0 < en.ncols) {
                const int ncols = min(NC, en.ncols - c0);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            int i = wm * 32 + a * 8 + g, j = wn * 32 + b * 8 + 2 * q + h;
                            if (i < nrows && j < ncols) en.Y[r0 + i + (size_t)(c0 + j) * en.ldy] += acc[a][b][h];
                        }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        }
    }
}

// split targets: Y[tile] += sum of its segments' partial tiles, in segment order
struct KbRed { double* Y; int ldy, nrows, ncols, p0, np; };
template <int NC>
__global__ void kb_reduce_kernel(const KbRed* __restrict__ red, const double* __restrict__ partial) {
    const KbRed r = red[blockIdx.x];
    for (int e = threadIdx.x; e < KB_M * NC; e += blockDim.x) {
        const int i = e % KB_M, j = e / KB_M;
        if (i >= r.nrows || j >= r.ncols) continue;
        double s = 0.0;
        for (int p = 0; p < r.np; ++p) s += partial[(size_t)(r.p0 + p) * KB_M * NC + e];
        r.Y[i + (size_t)j * r.ldy] += s;
    }
}

// ---------------------------------------------------------------- narrow products (k <= 4)
// Eval-bound path (PCG matvec): lane = target row (32-row tile), the 8 warps of a
// CTA take the entries of one output group round-robin; a warp walks its entry's
// source points 32 at a time, broadcasting each point's coordinates and values
// by shuffles, so every kernel entry is evaluated exactly once; partial sums of
// the warps are reduced in shared memory before one read-modify-write of Y.

template <int KID, int NV>
__global__ void __launch_bounds__(256) kblock_vec_kernel(
    KernelParams kp, double shift, int d, const KbBlock* __restrict__ blocks,
    const KbTarget* __restrict__ targets, const KbEntry* __restrict__ entries,
    const int2* __restrict__ work) {
    __shared__ double red[8][32][NV];
    const int2 wk = work[blockIdx.x];
    const KbTarget tg = targets[wk.x];
    const KbBlock tb = blocks[tg.blk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r0 = wk.y * 32;
    const int row = r0 + lane;
    const bool valid = row < tb.n;
    double rx0 = 0.0, rx1 = 0.0, rx2 = 0.0;
    int rc = 0;                                  // RPY: component of the row dof
    if (valid) {
        rx0 = tb.x[row];
        if (d > 1) rx1 = tb.x[tb.ds + row];
        if (d > 2) rx2 = tb.x[2 * tb.ds + row];
        if (KID == SPD_K_RPY) rc = (int)tb.x[3 * tb.ds + row];
    }
    const int64_t rid = tb.id0 >= 0 ? tb.id0 + row : -1;
    int g0 = tg.e_begin;
    while (g0 < tg.e_end) {
        int g1 = g0 + 1;
        while (g1 < tg.e_end && entries[g1].Y == entries[g0].Y) ++g1;
        double acc[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = 0.0;
        for (int e = g0 + warp; e < g1; e += 8) {
            const KbEntry en = entries[e];
            const KbBlock sb = blocks[en.src];
            const int nc = min(en.ncols, NV);
            const bool sh = shift != 0.0 && rid >= 0 && sb.id0 >= 0;
            for (int c0 = 0; c0 < sb.n; c0 += 32) {
                const int c = c0 + lane;
                double sx0 = 0.0, sx1 = 0.0, sx2 = 0.0, xv[NV];
                int sc = 0;
                if (c < sb.n) {
                    sx0 = sb.x[c];
                    if (d > 1) sx1 = sb.x[sb.ds + c];
                    if (d > 2) sx2 = sb.x[2 * sb.ds + c];
                    if (KID == SPD_K_RPY) sc = (int)sb.x[3 * sb.ds + c];
                }
#pragma unroll
                for (int v = 0; v < NV; ++v) xv[v] = (c < sb.n && v < nc) ? en.X[c + (size_t)v * en.ldx] : 0.0;
                const int cnt = min(32, sb.n - c0);
                for (int q = 0; q < cnt; ++q) {
                    const double y0 = __shfl_sync(0xffffffffu, sx0, q);
                    const double y1 = __shfl_sync(0xffffffffu, sx1, q);
                    const double y2 = __shfl_sync(0xffffffffu, sx2, q);
                    const double df0 = rx0 - y0, df1 = rx1 - y1, df2 = rx2 - y2;
                    double kv;
                    if constexpr (KID == SPD_K_RPY)
                        kv = rpy_entry(kp, df0, df1, df2, rc, __shfl_sync(0xffffffffu, sc, q));
                    else kv = kval<KID>(kp, df0 * df0 + df1 * df1 + df2 * df2);
                    if (sh && rid == sb.id0 + c0 + q) kv += shift;
#pragma unroll
                    for (int v = 0; v < NV; ++v) acc[v] += kv * __shfl_sync(0xffffffffu, xv[v], q);
                }
            }
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) red[warp][lane][v] = acc[v];
        __syncthreads();
        if (warp == 0 && valid) {
            const KbEntry en = entries[g0];
            const int nc = min(en.ncols, NV);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (v >= nc) break;
                double sum = 0.0;
                for (int w = 0; w < 8; ++w) sum += red[w][lane][v];
                en.Y[row + (size_t)v * en.ldy] += sum;
            }
        }
        __syncthreads();
        g0 = g1;
    }
}

template <int KID>
static void launch_vec(cudaStream_t s, unsigned nb, int nv, const KernelParams& kp, double shift, int d,
                       const KbBlock* b, const KbTarget* t, const KbEntry* e, const int2* w) {
    if (nv == 1) kblock_vec_kernel<KID, 1><<<nb, 256, 0, s>>>(kp, shift, d, b, t, e, w);
    else kblock_vec_kernel<KID, 4><<<nb, 256, 0, s>>>(kp, shift, d, b, t, e, w);
}

static void kblock_vec(cudaStream_t s, const KernelParams& kp, double shift, int d,
                       const std::vector<KbBlock>& blocks, const std::vector<KbTarget>& targets,
                       const std::vector<KbEntry>& entries, int maxc) {
    std::vector<int2> work;
    double fl = 0, by = 0;
    for (int t = 0; t < (int)targets.size(); ++t) {
        const KbTarget& tg = targets[t];
        if (tg.e_end <= tg.e_begin) continue;
        for (int tm = 0; tm < ceil_div(blocks[tg.blk].n, 32); ++tm) work.push_back(make_int2(t, tm));
        for (int e = tg.e_begin; e < tg.e_end; ++e) {
            const double nr = blocks[tg.blk].n, ns = blocks[entries[e].src].n;
            fl += 2.0 * nr * ns * entries[e].ncols;
            by += 8.0 * (ns * (d + entries[e].ncols) + 2.0 * nr * entries[e].ncols);
        }
    }
    if (work.empty()) return;
    DevArray<KbBlock> db(s, blocks);
    DevArray<KbTarget> dt(s, targets);
    DevArray<KbEntry> de(s, entries);
    DevArray<int2> dw(s, work);
    ProfScope prof(s, "kblock_vec", fl, by);
    const unsigned nb = (unsigned)work.size();
    const int nv = maxc <= 1 ? 1 : 4;
    switch (kp.id) {
    case SPD_K_GAUSSIAN: launch_vec<SPD_K_GAUSSIAN>(s, nb, nv, kp, shift, d, db.p, dt.p, de.p, dw.p); break;
    case SPD_K_MATERN32: launch_vec<SPD_K_MATERN32>(s, nb, nv, kp, shift, d, db.p, dt.p, de.p, dw.p); break;
    case SPD_K_EXPONENTIAL: launch_vec<SPD_K_EXPONENTIAL>(s, nb, nv, kp, shift, d, db.p, dt.p, de.p, dw.p); break;
    case SPD_K_RPY: launch_vec<SPD_K_RPY>(s, nb, nv, kp, shift, d, db.p, dt.p, de.p, dw.p); break;
    default: launch_vec<SPD_K_IMQ>(s, nb, nv, kp, shift, d, db.p, dt.p, de.p, dw.p); break;
    }
    SPD_LAUNCH();
}

// Tensor maps for the TMA-staged kernel: the entries' X pointers are grouped into buffers
// (same leading dimension, every column block [X, X + n_src) inside one column of the
// group's base); a group gets a 2-D map (rows = the rows any entry reads, columns = the
// common width; 16 x NC boxes, 128-byte swizzle) when TMA can address it (16-byte
// aligned base and stride) and every chunk tail it loads lies inside rows some entry
// owns or past the map (zero fill) -- never uninitialised memory.  Returns the maps in use.
typedef CUresult (*kb_encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static kb_encode_fn kb_encoder() {
    static kb_encode_fn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (kb_encode_fn)p;
        else
            cudaGetLastError();
    }
    return fn;
}

static int kb_tma_maps(const std::vector<KbBlock>& blocks, std::vector<KbEntry>& ents, int NC, KbTma& tma) {
    for (auto& e : ents) { e.tmi = -1; e.tr = 0; }
    // default: TMA for the 32- and 160-column tiles; the 64 / 128-column tiles keep the register
    // prefetch (measured at C5: k = 64 110.2 ms with TMA against 107.1 ms, k = 256 379.8 against
    // 370.2 ms; C4 SPD-HSS build at w = 160 1.898 s against 1.915 s).  SPD_KB_TMA=1: every tile
    // through TMA, 0: none.
    const char* env = getenv("SPD_KB_TMA");
    if (env && atoi(env) == 0) return 0;
    if (!(env && atoi(env) == 1) && (NC == 64 || NC == 128)) return 0;
    kb_encode_fn enc = kb_encoder();
    if (!enc) return 0;
    const int KK = kb_tma_chunk(NC);
    std::vector<int> ord(ents.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int)i;
    std::sort(ord.begin(), ord.end(), [&](int a, int b) {
        if (ents[a].ldx != ents[b].ldx) return ents[a].ldx < ents[b].ldx;
        return ents[a].X < ents[b].X;
    });
    int nmap = 0, ngroup = 0;
    size_t i = 0;
    while (i < ord.size()) {
        // group: same ld, pointers within one column of the first one
        const KbEntry& f = ents[ord[i]];
        const int64_t ld = f.ldx;
        const double* base = f.X;
        size_t j = i;
        while (j < ord.size() && ents[ord[j]].ldx == ld && ents[ord[j]].X - base + blocks[ents[ord[j]].src].n <= ld) ++j;
        if (j == i) j = i + 1;                                 // a block longer than its column: no map
        const size_t gb = i, ge = j;
        i = j;
        ++ngroup;
        if (getenv("SPD_KB_TMA_MAPSEL") && !((atoll(getenv("SPD_KB_TMA_MAPSEL")) >> (ngroup - 1)) & 1)) continue;
        if (nmap >= KB_NTMA || (ld & 1) || ld <= 0) continue;
        const double* b16 = reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(base) & ~(uintptr_t)15);
        const int ncols = ents[ord[gb]].ncols;
        bool ok = true;
        int64_t rows = 0;
        std::vector<std::pair<int64_t, int64_t>> iv;          // rows owned by some entry
        for (size_t t = gb; t < ge; ++t) {
            const KbEntry& e = ents[ord[t]];
            if (e.ncols != ncols) { ok = false; break; }
            const int64_t r = e.X - b16, n = blocks[e.src].n;
            rows = std::max(rows, r + n);
            iv.push_back({r, r + n});
        }
        if (!ok || rows < 16 || rows > ld || rows >= (1LL << 31)) continue;    // box <= tensor

        std::sort(iv.begin(), iv.end());
        std::vector<std::pair<int64_t, int64_t>> mg;
        for (auto& v : iv) {
            if (!mg.empty() && v.first <= mg.back().second) mg.back().second = std::max(mg.back().second, v.second);
            else mg.push_back(v);
        }
        auto covered = [&](int64_t a, int64_t b) {            // [a, b) inside one merged interval
            if (a >= b) return true;
            auto it = std::upper_bound(mg.begin(), mg.end(), std::make_pair(a, INT64_MAX));
            if (it == mg.begin()) return false;
            --it;
            return it->first <= a && b <= it->second;
        };
        for (size_t t = gb; t < ge && ok; ++t) {
            const KbEntry& e = ents[ord[t]];
            const int64_t r = e.X - b16, n = blocks[e.src].n;
            const int64_t tail_end = std::min(rows, r + (int64_t)ceil_div((int)n, KK) * KK);
            ok = covered(r + n, tail_end);
        }
        if (!ok) continue;
        cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)ncols};
        cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
        // box columns: the tile's NC, or the buffer's width when narrower (a box wider than the
        // tensor faults); stage columns past it are never stored to Y (column-independent sums)
        const int bcols = std::min(NC, ncols);
        cuuint32_t box[2] = {16, (cuuint32_t)bcols};
        cuuint32_t es[2] = {1, 1};
        if (enc(&tma.map[nmap], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)b16, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            continue;
        tma.box_bytes[nmap] = 16u * (unsigned)bcols * (unsigned)sizeof(double);
        if (getenv("SPD_KB_TMA_TRACE")) {
            int nmin = 1 << 30, nmax = 0;
            for (size_t t = gb; t < ge; ++t) { nmin = std::min(nmin, blocks[ents[ord[t]].src].n); nmax = std::max(nmax, blocks[ents[ord[t]].src].n); }
            fprintf(stderr, "[kblock]   map %d (group %d): base %% 16 = %d, ld %lld, rows %lld, cols %d, box 16 x %d, %zu entries, src n %d..%d\n",
                    nmap, ngroup - 1, (int)(reinterpret_cast<uintptr_t>(base) & 15), (long long)ld, (long long)rows, ncols, bcols, ge - gb, nmin, nmax);
        }
        for (size_t t = gb; t < ge; ++t) {
            KbEntry& e = ents[ord[t]];
            e.tmi = nmap;
            e.tr = (int)(e.X - b16);
        }
        ++nmap;
    }
    return nmap;
}

bool kblock_plan(cudaStream_t s, const std::vector<KbBlock>& blocks, const std::vector<KbTarget>& targets,
                 const std::vector<KbEntry>& entries, KbPlan& plan) {
    plan = KbPlan();
    {
        int maxc = 0;
        for (auto& e : entries) maxc = std::max(maxc, e.ncols);
        if (maxc <= 4) return false;
    }
    int maxc_all = 0;
    for (auto& e : entries) maxc_all = std::max(maxc_all, e.ncols);
    // column tile matched to the width (k <= 160 in one tile: every kernel tile is evaluated
    // once per product; wider products take 128-column tiles)
    const int NC = maxc_all > 160 ? 128 : maxc_all > 128 ? 160 : maxc_all > 64 ? 128 : (maxc_all > 32 ? 64 : 32);
    // work items; a target whose entries (one output group) hold many more source
    // points than the average item is cut into segments at entry boundaries, so the
    // long top-level coupling lists spread over many CTAs (ordered reduction after)
    std::vector<long long> cost(targets.size(), 0);
    long long total_cost = 0, ntile_all = 0;
    for (int t = 0; t < (int)targets.size(); ++t) {
        for (int e = targets[t].e_begin; e < targets[t].e_end; ++e) cost[t] += blocks[entries[e].src].n;
        const long long tiles = (long long)ceil_div(blocks[targets[t].blk].n, KB_M);
        total_cost += cost[t] * tiles;
        ntile_all += tiles;
    }
    const long long seg = std::max<long long>(1024, total_cost / std::max<long long>(1, 148LL * 8));
    std::vector<KbWork> work;
    std::vector<KbRed> red;
    int nslot = 0;
    for (int t = 0; t < (int)targets.size(); ++t) {
        const KbTarget& tg = targets[t];
        if (tg.e_end <= tg.e_begin) continue;
        int maxc = 0;
        bool one_group = true;
        for (int e = tg.e_begin; e < tg.e_end; ++e) {
            maxc = std::max(maxc, entries[e].ncols);
            if (entries[e].Y != entries[tg.e_begin].Y || entries[e].ncols != entries[tg.e_begin].ncols) one_group = false;
        }
        const int nr = blocks[tg.blk].n;
        // segment boundaries
        std::vector<int> cuts{tg.e_begin};
        if (one_group && cost[t] > 2 * seg) {
            long long acc = 0;
            for (int e = tg.e_begin; e < tg.e_end; ++e) {
                acc += blocks[entries[e].src].n;
                if (acc >= seg && e + 1 < tg.e_end) { cuts.push_back(e + 1); acc = 0; }
            }
        }
        cuts.push_back(tg.e_end);
        const int nseg = (int)cuts.size() - 1;
        for (int tn = 0; tn < ceil_div(maxc, NC); ++tn)
            for (int tm = 0; tm < ceil_div(nr, KB_M); ++tm) {
                if (nseg == 1) { work.push_back({t, tm, tn, tg.e_begin, tg.e_end, -1}); continue; }
                const KbEntry& e0 = entries[tg.e_begin];
                red.push_back({e0.Y + tm * KB_M + (size_t)tn * NC * e0.ldy, e0.ldy, std::min(KB_M, nr - tm * KB_M),
                               std::min(NC, e0.ncols - tn * NC), nslot, nseg});
                for (int sg = 0; sg < nseg; ++sg) work.push_back({t, tm, tn, cuts[sg], cuts[sg + 1], nslot++});
            }
    }
    if (work.empty()) { plan.ok = true; return true; }
    // heaviest items first (crude LPT over the launch order)
    auto wcost = [&](const KbWork& w) {
        long long c = 0;
        for (int e = w.eb; e < w.ee; ++e) c += blocks[entries[e].src].n;
        return c;
    };
    std::vector<std::pair<long long, int>> order;
    for (int i = 0; i < (int)work.size(); ++i) order.push_back({-wcost(work[i]), i});
    std::stable_sort(order.begin(), order.end());
    {
        std::vector<KbWork> sorted;
        for (auto& o : order) sorted.push_back(work[o.second]);
        work.swap(sorted);
    }
    double fl = 0, by = 0;
    for (const auto& tg : targets)
        for (int e = tg.e_begin; e < tg.e_end; ++e) {
            const double nr = blocks[tg.blk].n, ns = blocks[entries[e].src].n, nc = entries[e].ncols;
            fl += 2.0 * nr * ns * nc;
            by += 8.0 * (ns * nc + 2.0 * nr * nc);
        }
    plan.NC = NC;
    std::vector<KbEntry> ents(entries);
    plan.ntma = kb_tma_maps(blocks, ents, NC, plan.tma);
    {
        // a launch whose entries mostly cannot be addressed by the (at most KB_NTMA) maps -- the level
        // loop's sandwiches, one X buffer per node -- runs the register-staged kernel: the mixed
        // kernel pays its staging branches for a handful of TMA entries (SPD_KB_TMA_MINSHARE, default 0.5)
        size_t nt = 0;
        for (auto& e : ents) nt += e.tmi >= 0;
        const char* ms = getenv("SPD_KB_TMA_MINSHARE");
        const double minshare = ms ? atof(ms) : 0.5;
        if (plan.ntma > 0 && (double)nt < minshare * (double)ents.size()) {
            for (auto& e : ents) { e.tmi = -1; e.tr = 0; }
            plan.ntma = 0;
        }
    }
    plan.tma_mix = false;
    for (auto& e : ents) plan.tma_mix |= e.tmi < 0;
    if (getenv("SPD_KB_TMA_TRACE")) {
        size_t nt = 0;
        for (auto& e : ents) nt += e.tmi >= 0;
        fprintf(stderr, "[kblock] NC %d: %d tensor maps, %zu of %zu entries TMA-staged\n", NC, plan.ntma, nt, ents.size());
    }
    plan.nwork = (int)work.size();
    plan.nred = (int)red.size();
    plan.fl = fl;
    plan.by = by;
    plan.partial.alloc(std::max<size_t>(1, (size_t)nslot * KB_M * NC));
    plan.b.upload(blocks, s);
    plan.t.upload(targets, s);
    plan.e.upload(ents, s);
    std::vector<char> wb(sizeof(KbWork) * work.size()), rb(sizeof(KbRed) * std::max<size_t>(1, red.size()));
    std::memcpy(wb.data(), work.data(), wb.size());
    if (!red.empty()) std::memcpy(rb.data(), red.data(), sizeof(KbRed) * red.size());
    plan.w.upload(wb, s);
    plan.r.upload(rb, s);
    plan.ok = true;
    return true;
}

void kblock_run(cudaStream_t s, const KernelParams& kp, double shift, int d, const KbPlan& plan) {
    if (!plan.ok || plan.nwork == 0) return;
    const int NC = plan.NC;
    const KbBlock* bp = plan.b.p;
    const KbTarget* tp = plan.t.p;
    const KbEntry* ep = plan.e.p;
    const KbWork* wp = (const KbWork*)plan.w.p;
    double* pp = plan.partial.p;
    ProfScope prof(s, "kblock_dmma", plan.fl, plan.by);
    const unsigned nb = (unsigned)plan.nwork;
#define SPD_KB_TMA_LAUNCH2(KID, MIX)                                                                          \
    if (NC == 160) { kb_attr(kblock_tma_kernel<KID, 160, MIX>, kb_tma_smem_bytes(160)); kblock_tma_kernel<KID, 160, MIX><<<nb, 320, kb_tma_smem_bytes(160), s>>>(kp, shift, d, bp, tp, ep, wp, pp, plan.tma); } \
    else if (NC == 128) { kb_attr(kblock_tma_kernel<KID, 128, MIX>, kb_tma_smem_bytes(128)); kblock_tma_kernel<KID, 128, MIX><<<nb, 256, kb_tma_smem_bytes(128), s>>>(kp, shift, d, bp, tp, ep, wp, pp, plan.tma); } \
    else if (NC == 64) { kb_attr(kblock_tma_kernel<KID, 64, MIX>, kb_tma_smem_bytes(64)); kblock_tma_kernel<KID, 64, MIX><<<nb, 128, kb_tma_smem_bytes(64), s>>>(kp, shift, d, bp, tp, ep, wp, pp, plan.tma); } \
    else { kb_attr(kblock_tma_kernel<KID, 32, MIX>, kb_tma_smem_bytes(32)); kblock_tma_kernel<KID, 32, MIX><<<nb, 64, kb_tma_smem_bytes(32), s>>>(kp, shift, d, bp, tp, ep, wp, pp, plan.tma); }
#define SPD_KB_TMA_LAUNCH(KID) if (plan.tma_mix) { SPD_KB_TMA_LAUNCH2(KID, true) } else { SPD_KB_TMA_LAUNCH2(KID, false) }
    if (plan.ntma > 0) {
        switch (kp.id) {
        case SPD_K_GAUSSIAN: SPD_KB_TMA_LAUNCH(SPD_K_GAUSSIAN); break;
        case SPD_K_MATERN32: SPD_KB_TMA_LAUNCH(SPD_K_MATERN32); break;
        case SPD_K_EXPONENTIAL: SPD_KB_TMA_LAUNCH(SPD_K_EXPONENTIAL); break;
        case SPD_K_RPY: SPD_KB_TMA_LAUNCH(SPD_K_RPY); break;
        default: SPD_KB_TMA_LAUNCH(SPD_K_IMQ); break;
        }
    } else {
#define SPD_KB_LAUNCH(KID)                                                                                    \
    if (NC == 160) { kb_attr(kblock_kernel<KID, 160>, kb_smem_bytes(160)); kblock_kernel<KID, 160><<<nb, 320, kb_smem_bytes(160), s>>>(kp, shift, d, bp, tp, ep, wp, pp); } \
    else if (NC == 128) { kb_attr(kblock_kernel<KID, 128>, kb_smem_bytes(128)); kblock_kernel<KID, 128><<<nb, 256, kb_smem_bytes(128), s>>>(kp, shift, d, bp, tp, ep, wp, pp); } \
    else if (NC == 64) kblock_kernel<KID, 64><<<nb, 128, kb_smem_bytes(64), s>>>(kp, shift, d, bp, tp, ep, wp, pp); \
    else kblock_kernel<KID, 32><<<nb, 64, kb_smem_bytes(32), s>>>(kp, shift, d, bp, tp, ep, wp, pp);
    switch (kp.id) {
    case SPD_K_GAUSSIAN: SPD_KB_LAUNCH(SPD_K_GAUSSIAN); break;
    case SPD_K_MATERN32: SPD_KB_LAUNCH(SPD_K_MATERN32); break;
    case SPD_K_EXPONENTIAL: SPD_KB_LAUNCH(SPD_K_EXPONENTIAL); break;
    case SPD_K_RPY: SPD_KB_LAUNCH(SPD_K_RPY); break;
    default: SPD_KB_LAUNCH(SPD_K_IMQ); break;
    }
    }
#undef SPD_KB_LAUNCH
#undef SPD_KB_TMA_LAUNCH
#undef SPD_KB_TMA_LAUNCH2
    SPD_LAUNCH();
    if (plan.nred > 0) {
        const KbRed* rp = (const KbRed*)plan.r.p;
        const unsigned nr = (unsigned)plan.nred;
        if (NC == 160) kb_reduce_kernel<160><<<nr, 256, 0, s>>>(rp, pp);
        else if (NC == 128) kb_reduce_kernel<128><<<nr, 256, 0, s>>>(rp, pp);
        else if (NC == 64) kb_reduce_kernel<64><<<nr, 256, 0, s>>>(rp, pp);
        else kb_reduce_kernel<32><<<nr, 256, 0, s>>>(rp, pp);
        SPD_LAUNCH();
    }
}

void kblock_apply(cudaStream_t s, const KernelParams& kp, double shift, int d,
                  const std::vector<KbBlock>& blocks, const std::vector<KbTarget>& targets,
                  const std::vector<KbEntry>& entries) {
    int maxc = 0;
    for (auto& e : entries) maxc = std::max(maxc, e.ncols);
    if (maxc == 0) return;
    if (maxc <= 4) { kblock_vec(s, kp, shift, d, blocks, targets, entries, maxc); return; }
    KbPlan plan;
    kblock_plan(s, blocks, targets, entries, plan);
    kblock_run(s, kp, shift, d, plan);
}

}  // namespace spd
