// common.cuh -- shared device/host helpers of libspdhss (product path).
// Independent of oracle/: nothing here is shared with the CPU oracle.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include <stdexcept>
#include "../../include/spdhss.h"

namespace spd {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    spd_status code;
    Error(spd_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void set_last_error(const std::string& m);

#define SPD_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw ::spd::Error(e_ == cudaErrorMemoryAllocation ? SPD_ENOMEM : SPD_ECUDA,\
                std::string(#call) + ": " + cudaGetErrorString(e_) + " @" __FILE__ ":" + \
                std::to_string(__LINE__));                                              \
    } while (0)
void count_launch();
void count_launches(long long n);          // e.g. the kernel nodes of one graph replay
#define SPD_LAUNCH() do { ::spd::count_launch(); SPD_CUDA(cudaGetLastError()); } while (0)
#define SPD_REQUIRE(cond, msg) do { if (!(cond)) throw ::spd::Error(SPD_EINVAL, msg); } while (0)

// ---------------------------------------------------------------- instrumentation
// Per-kernel-class CUDA events on the launching stream (enabled by spd_prof_enable;
// bench.py uses it for the roofline line).  flops / bytes are ALGORITHMIC counts.
struct ProfScope {
    int slot = -1;
    cudaStream_t s;
    bool ext = false;
    ProfScope(cudaStream_t st, const char* name, double flops, double bytes);
    ~ProfScope();
};
// debug: with env SPD_STAGES set, synchronize s and print the wall time since the last mark
void stage_mark(cudaStream_t s, const char* name, int level = 0);
// records created while capturing a graph are moved out and re-accumulated
// after every replay of that graph
struct ProfCaptured;
ProfCaptured* prof_capture_take(size_t first);   // records [first, end) of the list
size_t prof_mark();
void prof_update_last(const char* name, double flops, double bytes);   // latest record of that name
bool prof_on();                                   // the per-kernel-class profiler is enabled
void prof_accumulate(ProfCaptured* c);            // after a (synchronized) replay
void prof_release(ProfCaptured* c);

// ---------------------------------------------------------------- device memory
// Device buffers are stream-ordered (cudaMallocAsync / cudaFreeAsync from the
// device's default pool, which keeps freed memory cached up to a threshold), on
// the stream of the current library call (AllocStreamScope; the legacy stream
// when no call is active).  This keeps the many per-level allocations of the
// builds off the host's critical path (cudaMalloc/cudaFree synchronize).
cudaStream_t& alloc_stream();
void init_mem_pool();
size_t device_free_bytes();      // free device memory + the pool's unused reserve
struct AllocStreamScope {
    cudaStream_t prev;
    explicit AllocStreamScope(cudaStream_t s) : prev(alloc_stream()) { init_mem_pool(); alloc_stream() = s; }
    ~AllocStreamScope() { alloc_stream() = prev; }
};
template <class T>
struct DBuf {                       // owning device buffer
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; return *this; }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) SPD_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), alloc_stream()));
    }
    void release() { if (p) cudaFreeAsync(p, alloc_stream()); p = nullptr; n = 0; }
    void zero(cudaStream_t s) { if (n) SPD_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s)); }
    void upload(const std::vector<T>& h, cudaStream_t s) {
        if (h.size() != n) alloc(h.size());
        if (n) SPD_CUDA(cudaMemcpyAsync(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    std::vector<T> download(cudaStream_t s) const {
        std::vector<T> h(n);
        if (n) {
            SPD_CUDA(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
            SPD_CUDA(cudaStreamSynchronize(s));
        }
        return h;
    }
};

#if defined(__CUDACC__)
__host__ __device__
#endif
inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ---------------------------------------------------------------- kernel functions
// K as a function of r^2 (BASELINE.json forms, reading R13).
struct KernelParams {
    int id;
    double l, inv_l, inv_l2, sqrt3_inv_l, l2;
};
inline KernelParams make_kernel(const spd_kernel& k) {
    KernelParams p;
    p.id = k.id; p.l = k.l; p.inv_l = 1.0 / k.l; p.inv_l2 = 1.0 / (k.l * k.l);
    p.sqrt3_inv_l = 1.7320508075688772 / k.l; p.l2 = k.l * k.l;
    return p;
}
#if defined(__CUDACC__)
__device__ __forceinline__ double kernel_r2(const KernelParams& kp, double r2) {
    switch (kp.id) {
    case SPD_K_GAUSSIAN: return exp(-r2 * kp.inv_l2);
    case SPD_K_MATERN32: { double t = sqrt(r2) * kp.sqrt3_inv_l; return (1.0 + t) * exp(-t); }
    case SPD_K_EXPONENTIAL: return exp(-sqrt(r2) * kp.inv_l);
    default: return rsqrt(r2 + kp.l2);
    }
}

// RPY tensor entry (reading R28: 1/a on both near-branch
// terms) for r = x - y = (d0, d1, d2) and components ca, cb of the two dofs
__device__ __forceinline__ double rpy_entry(const KernelParams& kp, double d0, double d1, double d2, int ca,
                                            int cb) {
    const double r2 = d0 * d0 + d1 * d1 + d2 * d2;
    const double dl = ca == cb ? 1.0 : 0.0;
    if (r2 == 0.0) return dl * kp.inv_l;
    const double ra = ca == 0 ? d0 : (ca == 1 ? d1 : d2);
    const double rb = cb == 0 ? d0 : (cb == 1 ? d1 : d2);
    const double inv_r = 1.0 / sqrt(r2), r = r2 * inv_r;
    const double rr = ra * rb * (inv_r * inv_r);
    if (r >= 2.0 * kp.l)
        return 0.75 * inv_r * (dl + rr) + 1.5 * kp.l2 * (inv_r * inv_r * inv_r) * (dl * (1.0 / 3.0) - rr);
    const double t = r * kp.inv_l;
    return kp.inv_l * ((1.0 - 0.28125 * t) * dl + 0.09375 * t * rr);
}

// one kernel entry between point / dof rows x and y (coordinate a at x[a * xs]); d
// coordinates, for RPY (x, y, z, component)
__device__ __forceinline__ double kernel_entry(const KernelParams& kp, const double* x, int64_t xs, const double* y,
                                               int64_t ys, int d) {
    if (kp.id == SPD_K_RPY)
        return rpy_entry(kp, x[0] - y[0], x[xs] - y[ys], x[2 * xs] - y[2 * ys], (int)x[3 * xs], (int)y[3 * ys]);
    double r2 = 0.0;
    for (int a = 0; a < d; ++a) { const double df = x[a * xs] - y[a * ys]; r2 += df * df; }
    return kernel_r2(kp, r2);
}

// ---------------------------------------------------------------- DMMA m8n8k4 fp64
// Fragment layout (PTX ISA mma.m8n8k4 .f64): lane = 4*g + q (g = lane>>2, q = lane&3)
//   A (8x4, row):  a = A[g][q]      B (4x8, col): b = B[q][g]
//   C (8x8):       c0 = C[g][2q], c1 = C[g][2q+1]
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

#endif  // __CUDACC__

// ---------------------------------------------------------------- batched descriptors
struct GemmDesc {          // C = alpha op(A) op(B) + beta C ; column-major
    const double* A; const double* B; double* C;
    int m, n, k;
    int lda, ldb, ldc;
};
struct MatDesc {           // generic m x n matrix with leading dimension
    double* A; int m, n, ld;
};
struct TrsmDesc {          // X := op(T)^{-1} X, T n x n triangular, X n x nrhs
    const double* T; double* X; int n, nrhs, ldt, ldx;
};
struct QrcpDesc {          // pivoted QR of A (m x n) in place
    double* A; int m, n, ld;
    int max_rank;
    int* piv;              // n
    double* beta;          // min(m, n)
    int* rank;             // out (device)
    double* norms;         // scratch n
    // forced pivots (injection hook of reading R19, spd_h2_opts.inject_skeletons):
    // when non-null, step t < nforce takes the column whose ORIGINAL index is force[t]
    // (device) instead of the argmax, and the factorization stops after nforce steps
    const int* force = nullptr;
    int nforce = 0;
};

// host launchers (dense.cu)
void gemm_batched(cudaStream_t s, const std::vector<GemmDesc>& d, bool transA, bool transB,
                  double alpha, double beta);
// info[b] = 0 on success, else first failing column + 1; bad[b] = that pivot value
void potrf_batched(cudaStream_t s, const std::vector<MatDesc>& d, int* info_dev, double* bad_dev);
// uplo: 'L' lower / 'U' upper storage of T; trans: false -> T^{-1} X, true -> T^{-T} X
void trsm_batched(cudaStream_t s, const std::vector<TrsmDesc>& d, char uplo, bool trans);
void qrcp_batched(cudaStream_t s, const std::vector<QrcpDesc>& d, double rel_tol);
int qrcp_slots(int m);     // CTAs the QRCP of a large batch of m-row matrices runs at once (its balance unit)
// unpivoted blocked Householder QR (R factor only): on exit the upper triangle of
// A[:n, :n] holds R (n <= m); the rest of A is overwritten.  Panel width 32,
// compact-WY trailing updates on the DMMA GEMM.
struct QrDesc { double* A; int m, n, ld; };
void qr_unpivoted_batched(cudaStream_t s, const std::vector<QrDesc>& d);
void qr_tall_batched(cudaStream_t s, const std::vector<QrDesc>& d);      // + one-level TSQR for very tall m
// form Q[:, :r] (m x r, ld ldq) from the reflectors left in A by qrcp
struct FormQDesc { const double* A; const double* beta; const int* rank; double* Q; int m, n, lda, ldq; };
void formq_batched(cudaStream_t s, const std::vector<FormQDesc>& d);
// copy/transposed copy of sub-blocks: C[m x n] (+)= alpha * (trans ? A^T : A)
struct CopyDesc { const double* A; double* C; int m, n, lda, ldc; int trans; };
void copy_batched(cudaStream_t s, const std::vector<CopyDesc>& d, double alpha, bool accumulate);
void set_identity_plus(cudaStream_t s, const std::vector<MatDesc>& d);   // A += I, zero upper? no: A += I
void zero_upper_batched(cudaStream_t s, const std::vector<MatDesc>& d);
void zero_lower_batched(cudaStream_t s, const std::vector<MatDesc>& d);   // strictly lower part

// Descriptor arena: while a CUDA graph is being captured, descriptor arrays
// go to a persistent device arena (filled with a synchronous copy, legal in
// relaxed capture mode) and live as long as the graph.
struct DescArena {
    DBuf<char> buf;
    size_t off = 0;
    explicit DescArena(size_t bytes) : buf(bytes) {}
    void* take(size_t bytes) {
        size_t o = (off + 255) & ~(size_t)255;
        if (o + bytes > buf.n) throw Error(SPD_ENOMEM, "descriptor arena exhausted");
        off = o + bytes;
        return buf.p + o;
    }
};
DescArena*& desc_arena();                 // thread-local current arena (nullptr: none)

// descriptor arrays: stream-ordered device copy, freed after the launch
template <class T>
struct DevArray {
    T* p = nullptr;
    cudaStream_t s;
    bool owned = true;
    DevArray(cudaStream_t st, const std::vector<T>& h) : s(st) {
        if (h.empty()) return;
        if (DescArena* a = desc_arena()) {
            p = (T*)a->take(h.size() * sizeof(T));
            owned = false;
            SPD_CUDA(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
            return;
        }
        SPD_CUDA(cudaMallocAsync((void**)&p, h.size() * sizeof(T), s));
        SPD_CUDA(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    ~DevArray() { if (p && owned) cudaFreeAsync(p, s); }
};

}  // namespace spd
