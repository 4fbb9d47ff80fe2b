// pcg.cu -- preconditioned conjugate gradient (reading R15)
// with the H2 matvec as the operator and the SPD HSS solve as the preconditioner.
// x0 = 0; stop when ||r_k||_2 <= tol ||b||_2 (recursively updated residual) or
// at maxit.  Dot products use a fixed two-level reduction (deterministic).
#include "hss.hpp"
#include <chrono>
#include <cmath>

namespace spd {

constexpr int RED_BLOCKS = 296, RED_THREADS = 256;

__device__ double block_reduce(double v) {
    __shared__ double sh[RED_THREADS / 32];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    v = threadIdx.x < RED_THREADS / 32 ? sh[threadIdx.x] : 0.0;
    if (threadIdx.x < 32) v = warp_sum(v);
    return v;
}

// partial[b] = sum a.b over block b's grid-stride slice
__global__ void __launch_bounds__(RED_THREADS) dot_kernel(const double* a, const double* b, int64_t n, double* partial) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < n; i += (int64_t)RED_BLOCKS * RED_THREADS)
        s += a[i] * b[i];
    s = block_reduce(s);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}
// x += alpha p ; r -= alpha q ; partial = r.r
__global__ void __launch_bounds__(RED_THREADS) update_xr_kernel(double* x, double* r, const double* p, const double* q,
                                                                const double* scal, int64_t n, double* partial) {
    const double alpha = scal[0];
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
// p = z + beta p
__global__ void update_p_kernel(double* p, const double* z, const double* scal, int64_t n) {
    const double beta = scal[1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = z[i] + beta * p[i];
}
// final sums of partials -> out[0]
__global__ void finish_kernel(const double* partial, double* out) {
    double v = threadIdx.x < RED_BLOCKS ? partial[threadIdx.x] : 0.0;
    if (threadIdx.x + 256 < RED_BLOCKS) v += partial[threadIdx.x + 256];
    v = block_reduce(v);
    if (threadIdx.x == 0) out[0] = v;
}

struct PcgState {
    DBuf<double> partial{RED_BLOCKS}, scal{4}, res{2};
};

static double dev_dot(cudaStream_t s, PcgState& st, const double* a, const double* b, int64_t n) {
    dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(a, b, n, st.partial.p);
    finish_kernel<<<1, RED_THREADS, 0, s>>>(st.partial.p, st.res.p);
    SPD_LAUNCH();
    double v;
    SPD_CUDA(cudaMemcpyAsync(&v, st.res.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    return v;
}

// all vectors in tree order, length N
void pcg_tree(spd_h2_s* A, spd_hss_s* M, const double* b, double* x, double tol, int maxit, spd_pcg_report* rep,
              cudaStream_t s) {
    const int64_t N = A->N;
    const auto t0 = std::chrono::steady_clock::now();
    DBuf<double> r(N), z(N), p(N), q(N);
    PcgState st;
    SPD_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * N, s));
    SPD_CUDA(cudaMemcpyAsync(r.p, b, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    const double nb = std::sqrt(dev_dot(s, st, b, b, N));
    rep->iters = 0; rep->converged = 0; rep->relres = 1.0;
    if (nb == 0.0) { rep->converged = 1; rep->relres = 0.0; return; }
    auto precond = [&](const double* in, double* out) {
        if (M) hss_solve_tree(M, in, N, out, N, 1, s);
        else SPD_CUDA(cudaMemcpyAsync(out, in, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    };
    precond(r.p, z.p);
    SPD_CUDA(cudaMemcpyAsync(p.p, z.p, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    double rz = dev_dot(s, st, r.p, z.p, N);
    for (int it = 1; it <= maxit; ++it) {
        h2_apply_tree(A, p.p, N, q.p, N, 1, s);
        const double pq = dev_dot(s, st, p.p, q.p, N);
        if (!(pq > 0.0)) throw Error(SPD_ENOTPD, "PCG breakdown: p^T A p = " + std::to_string(pq));
        double scal[2] = {rz / pq, 0.0};
        SPD_CUDA(cudaMemcpyAsync(st.scal.p, scal, sizeof(double), cudaMemcpyHostToDevice, s));
        update_xr_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, r.p, p.p, q.p, st.scal.p, N, st.partial.p);
        finish_kernel<<<1, RED_THREADS, 0, s>>>(st.partial.p, st.res.p);
        SPD_LAUNCH();
        double rr;
        SPD_CUDA(cudaMemcpyAsync(&rr, st.res.p, sizeof(double), cudaMemcpyDeviceToHost, s));
        SPD_CUDA(cudaStreamSynchronize(s));
        rep->iters = it;
        rep->relres = std::sqrt(rr) / nb;
        if (rep->relres <= tol) { rep->converged = 1; break; }
        precond(r.p, z.p);
        const double rz_new = dev_dot(s, st, r.p, z.p, N);
        if (!(rz_new > 0.0)) throw Error(SPD_ENOTPD, "PCG breakdown: r^T M^{-1} r = " + std::to_string(rz_new));
        scal[1] = rz_new / rz;
        SPD_CUDA(cudaMemcpyAsync(st.scal.p, scal, 2 * sizeof(double), cudaMemcpyHostToDevice, s));
        update_p_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(p.p, z.p, st.scal.p, N);
        SPD_LAUNCH();
        rz = rz_new;
    }
    SPD_CUDA(cudaStreamSynchronize(s));
    rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace spd
