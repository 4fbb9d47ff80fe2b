// pcg.cu -- preconditioned conjugate gradient (reading R15)
// with the H2 matvec as the operator and the SPD HSS solve as the preconditioner.
// x0 = 0; stop when ||r_k||_2 <= tol ||b||_2 (recursively updated residual) or
// at maxit.  All scalars live on the device; one iteration (H2 matvec, dots,
// updates, HSS solve) is captured once as a CUDA graph and replayed, and the
// host reads back only (p^T q, ||r||^2, r^T z) per iteration for the stop and
// breakdown tests.  Dot products use a fixed two-level reduction (deterministic).
#include "hss.hpp"
#include "comm.hpp"
#include <chrono>
#include <cmath>
#include <cstdlib>

namespace spd {

constexpr int RED_BLOCKS = 296, RED_THREADS = 256;
// device scalar slots
enum { S_RZ = 0, S_PQ = 1, S_ALPHA = 2, S_RR = 3, S_RZNEW = 4, S_BETA = 5, S_NSCAL = 8 };

__device__ double block_reduce(double v) {
    __shared__ double sh[RED_THREADS / 32];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    v = threadIdx.x < RED_THREADS / 32 ? sh[threadIdx.x] : 0.0;
    if (threadIdx.x < 32) v = warp_sum(v);
    return v;
}

__global__ void __launch_bounds__(RED_THREADS) dot_kernel(const double* a, const double* b, int64_t n, double* partial) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < n; i += (int64_t)RED_BLOCKS * RED_THREADS)
        s += a[i] * b[i];
    s = block_reduce(s);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}
// out = sum(partial); mode 1: also alpha = rz / pq ; mode 2: also beta = rz_new / rz, rz = rz_new
__global__ void finish_kernel(const double* partial, double* scal, int slot, int mode) {
    double v = threadIdx.x < RED_BLOCKS ? partial[threadIdx.x] : 0.0;
    if (threadIdx.x + 256 < RED_BLOCKS) v += partial[threadIdx.x + 256];
    v = block_reduce(v);
    if (threadIdx.x == 0) {
        scal[slot] = v;
        if (mode == 1) scal[S_ALPHA] = scal[S_RZ] / v;
        if (mode == 2) { scal[S_BETA] = v / scal[S_RZ]; scal[S_RZ] = v; }
    }
}
__global__ void __launch_bounds__(RED_THREADS) update_xr_kernel(double* x, double* r, const double* p, const double* q,
                                                                const double* scal, int64_t n, double* partial) {
    const double alpha = scal[S_ALPHA];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < n; i += (int64_t)RED_BLOCKS * RED_THREADS) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        s += ri * ri;
    }
    s = block_reduce(s);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}
__global__ void __launch_bounds__(RED_THREADS) resid_kernel(const double* b, const double* q, int64_t n, double* partial) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < n; i += (int64_t)RED_BLOCKS * RED_THREADS) {
        const double r = b[i] - q[i];
        s += r * r;
    }
    s = block_reduce(s);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}
__global__ void update_p_kernel(double* p, const double* z, const double* scal, int64_t n) {
    const double beta = scal[S_BETA];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = z[i] + beta * p[i];
}

struct PcgWork {
    DBuf<double> r, z, p, q, partial, scal;
    explicit PcgWork(int64_t N) : r(N), z(N), p(N), q(N), partial(RED_BLOCKS), scal(S_NSCAL) {}
};

static void dot_into(cudaStream_t s, PcgWork& w, const double* a, const double* b, int64_t n, int slot, int mode) {
    {
        ProfScope prof(s, "pcg_vec", 2.0 * n, 16.0 * n);
        dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(a, b, n, w.partial.p);
        SPD_LAUNCH();
        finish_kernel<<<1, RED_THREADS, 0, s>>>(w.partial.p, w.scal.p, slot, mode);
        SPD_LAUNCH();
    }
}

// one PCG iteration after the first: q = A p, alpha, x/r update, z = M r, beta, p update
static void apply_precond(spd_hss_s* M, int precond, PcgWork& w, int64_t N, cudaStream_t s) {
    if (!M) SPD_CUDA(cudaMemcpyAsync(w.z.p, w.r.p, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    else if (precond == PC_BJ) bj_solve_vec(M, w.r.p, w.z.p, M->bt.p, s);
    else hss_solve_tree(M, w.r.p, N, w.z.p, N, 1, s);
}

static void iteration_body(spd_h2_s* A, spd_hss_s* M, int precond, double* x, PcgWork& w, int64_t N,
                           cudaStream_t s) {
    // real communicator: the product is subtree-sharded (each rank its leaves' rows of q from
    // the stored blocks touching its nodes, then the owners' rows are broadcast); vectors,
    // dots and the preconditioner stay replicated (identical on every rank)
    h2_apply_tree(A, w.p.p, N, w.q.p, N, 1, s, comm_real(A->comm));
    dot_into(s, w, w.p.p, w.q.p, N, S_PQ, 1);
    {
        ProfScope prof(s, "pcg_vec", 4.0 * N, 40.0 * N);
        update_xr_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, w.r.p, w.p.p, w.q.p, w.scal.p, N, w.partial.p);
        SPD_LAUNCH();
        finish_kernel<<<1, RED_THREADS, 0, s>>>(w.partial.p, w.scal.p, S_RR, 0);
        SPD_LAUNCH();
    }
    apply_precond(M, precond, w, N, s);
    dot_into(s, w, w.r.p, w.z.p, N, S_RZNEW, 2);
    {
        ProfScope prof(s, "pcg_vec", 2.0 * N, 24.0 * N);
        update_p_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(w.p.p, w.z.p, w.scal.p, N);
        SPD_LAUNCH();
    }
}

static cudaStream_t pcg_private_stream() {
    struct Cache {
        int dev = -1; cudaStream_t s = nullptr;
    };
    static thread_local Cache c;
    int dev = 0;
    SPD_CUDA(cudaGetDevice(&dev));
    if (!c.s || c.dev != dev) {
        SPD_CUDA(cudaStreamCreateWithFlags(&c.s, cudaStreamNonBlocking));   // lives as long as the thread
        c.dev = dev;
    }
    return c.s;
}
static double* pcg_pinned_scalars() {
    static thread_local double* hs = nullptr;
    if (!hs) SPD_CUDA(cudaMallocHost(&hs, sizeof(double) * S_NSCAL));
    return hs;
}

void pcg_tree(spd_h2_s* A, spd_hss_s* M, const double* b, double* x, double tol, int maxit, spd_pcg_report* rep,
              cudaStream_t user, int precond) {
    const int64_t N = A->N;
    const auto t0 = std::chrono::steady_clock::now();
    stage_mark(user, nullptr);
    // private non-blocking stream (graph capture is illegal on the legacy stream), created
    // once per thread and device: creating / destroying it per solve costs up to
    // hundreds of ms at teardown when the driver reclaims its resources
    cudaStream_t s = pcg_private_stream();
    AllocStreamScope alloc_scope(s);           // workspaces are stream-ordered on s
    cudaEvent_t ev;
    SPD_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SPD_CUDA(cudaEventRecord(ev, user));
    SPD_CUDA(cudaStreamWaitEvent(s, ev, 0));
    struct Cleanup {
        cudaStream_t s, user; cudaEvent_t ev; cudaGraphExec_t ge = nullptr; cudaGraph_t g = nullptr;
        ProfCaptured* pc = nullptr;
        ~Cleanup() {
            cudaEventRecord(ev, s);
            cudaStreamWaitEvent(user, ev, 0);
            if (ge) cudaGraphExecDestroy(ge);
            if (g) cudaGraphDestroy(g);
            cudaStreamSynchronize(s);
            prof_release(pc);
            cudaEventDestroy(ev);
        }
    } cl{s, user, ev};
    PcgWork w(N);
    double* hs = pcg_pinned_scalars();          // pinned host scalars (per thread, reused)

    SPD_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * N, s));
    SPD_CUDA(cudaMemcpyAsync(w.r.p, b, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    dot_into(s, w, b, b, N, S_RR, 0);
    SPD_CUDA(cudaMemcpyAsync(hs, w.scal.p, sizeof(double) * S_NSCAL, cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    const double nb = std::sqrt(hs[S_RR]);
    rep->iters = 0; rep->converged = 0; rep->relres = 1.0; rep->seconds = 0.0; rep->relres_true = 1.0;
    if (nb == 0.0) { rep->converged = 1; rep->relres = 0.0; rep->relres_true = 0.0; return; }
    // true residual ||b - A x|| / ||b|| after the solve (one more H2 product)
    auto true_residual = [&]() {
        h2_apply_tree(A, x, N, w.q.p, N, 1, s, comm_real(A->comm));
        resid_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(b, w.q.p, N, w.partial.p);
        SPD_LAUNCH();
        finish_kernel<<<1, RED_THREADS, 0, s>>>(w.partial.p, w.scal.p, S_PQ, 0);
        SPD_LAUNCH();
        double v = 0.0;
        SPD_CUDA(cudaMemcpyAsync(&v, w.scal.p + S_PQ, sizeof(double), cudaMemcpyDeviceToHost, s));
        SPD_CUDA(cudaStreamSynchronize(s));
        rep->relres_true = std::sqrt(v) / nb;
    };
    // z = M r, p = z, rz = r^T z
    if (M && precond == PC_BJ) hss_solve_tree(M, w.r.p, N, w.z.p, N, 1, s);   // allocates the solve workspace
    apply_precond(M, precond, w, N, s);
    SPD_CUDA(cudaMemcpyAsync(w.p.p, w.z.p, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    dot_into(s, w, w.r.p, w.z.p, N, S_RZ, 0);
    SPD_CUDA(cudaMemcpyAsync(hs, w.scal.p, sizeof(double) * S_NSCAL, cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));

    stage_mark(s, "pcg init (r, z, p, rz)");
    h2_prepare(A, 1, s);
    stage_mark(s, "pcg h2_prepare");
    // persistent cooperative kernel for the whole loop (pcgk.cu); env SPD_PCG_GRAPH=1
    // selects the per-iteration CUDA graph below instead (per-kernel profiling)
    const bool sharded = comm_real(A->comm);
    if (!getenv("SPD_PCG_GRAPH") && !sharded) {     // (sharded: no collective inside the persistent kernel)
        PcgPersistent pk;
        if (pcg_persistent_prepare(pk, A, M, x, w.r.p, w.p.p, w.q.p, w.z.p, s, precond)) {
            stage_mark(s, "pcg persistent prepare");
            double out[4];
            pcg_persistent_run(pk, hs[S_RZ], nb, tol, maxit, out, s);
            stage_mark(s, "pcg persistent run");

            rep->iters = (int)out[1];
            rep->relres = std::sqrt(out[0]) / nb;
            rep->converged = out[2] != 0.0;
            if (out[3] == 1.0) throw Error(SPD_ENOTPD, "PCG breakdown: p^T A p <= 0");
            if (out[3] == 2.0) throw Error(SPD_ENOTPD, "PCG breakdown: r^T M^{-1} r <= 0");
            true_residual();
            rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            return;
        }
    }
    // capture one iteration as a graph (descriptors in a persistent arena)
    h2_apply_tree(A, w.p.p, N, w.q.p, N, 1, s, sharded);   // builds stored k=1 blocks outside the graph
    bool use_graph = maxit > 1 && !(sharded && A->comm->hosted);   // host-staged collectives cannot be captured
    long long graph_kernels = 0;          // kernel nodes per replay (launch accounting)
    DescArena arena((size_t)64 << 20);
    if (use_graph) {
        try {
            desc_arena() = &arena;
            const size_t mark = prof_mark();
            SPD_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
            try { iteration_body(A, M, precond, x, w, N, s); }
            catch (...) { cudaGraph_t g; cudaStreamEndCapture(s, &g); if (g) cudaGraphDestroy(g); throw; }
            SPD_CUDA(cudaStreamEndCapture(s, &cl.g));
            SPD_CUDA(cudaGraphInstantiate(&cl.ge, cl.g, 0));
            size_t nn = 0;
            SPD_CUDA(cudaGraphGetNodes(cl.g, nullptr, &nn));
            std::vector<cudaGraphNode_t> nodes(nn);
            if (nn) SPD_CUDA(cudaGraphGetNodes(cl.g, nodes.data(), &nn));
            for (auto nd : nodes) {
                cudaGraphNodeType ty;
                SPD_CUDA(cudaGraphNodeGetType(nd, &ty));
                if (ty == cudaGraphNodeTypeKernel) ++graph_kernels;
            }
            cl.pc = prof_capture_take(mark);
            desc_arena() = nullptr;
        } catch (const Error&) {
            desc_arena() = nullptr;
            cudaGetLastError();
            use_graph = false;           // fall back to direct launches (same kernels)
        }
    }
    for (int it = 1; it <= maxit; ++it) {
        if (use_graph) {
            SPD_CUDA(cudaGraphLaunch(cl.ge, s));
            count_launches(graph_kernels);
        } else {
            iteration_body(A, M, precond, x, w, N, s);
        }
        SPD_CUDA(cudaMemcpyAsync(hs, w.scal.p, sizeof(double) * S_NSCAL, cudaMemcpyDeviceToHost, s));
        SPD_CUDA(cudaStreamSynchronize(s));
        if (use_graph) prof_accumulate(cl.pc);
        if (!(hs[S_PQ] > 0.0)) throw Error(SPD_ENOTPD, "PCG breakdown: p^T A p = " + std::to_string(hs[S_PQ]));
        rep->iters = it;
        rep->relres = std::sqrt(hs[S_RR]) / nb;
        if (rep->relres <= tol) { rep->converged = 1; break; }
        if (!(hs[S_RZNEW] > 0.0)) throw Error(SPD_ENOTPD, "PCG breakdown: r^T M^{-1} r = " + std::to_string(hs[S_RZNEW]));
    }
    true_residual();
    rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace spd
