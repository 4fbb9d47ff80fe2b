// hss.hpp -- SPD HSS handle (internal).  PAPER.md Alg. 4.
#pragma once
#include <unordered_map>
#include "h2.hpp"

namespace spd {

// per-level HSS data (level k nodes first..first+count-1)
struct HssLevel {
    int k = 0, first = 0, count = 0;
    std::vector<int> rank;          // r_i
    std::vector<int> m;             // rows of the node's basis: n_i (leaf) / r_c1 + r_c2 (nonleaf)
    std::vector<int64_t> off;       // row offset of node in the level's "rank space" (sum r)
    int64_t R = 0;                  // sum r_i
    // factors: leaf S_i (n x n) / nonleaf F_i (m x m), lower, col-major, ld = m
    std::vector<int64_t> F_off;
    DBuf<double> F;
    // explicit inverse factors S_i^{-1} / F_i^{-1} (lower, same layout as F) for the solve
    DBuf<double> Finv;
    // basis: leaf V_i (n x r) / nonleaf Vbar'_i (m x r), ld = m
    std::vector<int64_t> V_off;
    DBuf<double> V;
    // Phit: leaf Phi_i^T = S^{-T} V (n x r) / nonleaf P_i = F^{-T} Vbar' (m x r), ld = m
    DBuf<double> P;
    // transfer R_i = F Vbar' (nonleaf, m x r)
    DBuf<double> Rt;
    // (Phi_i U_i^{H2})^T : s_i x r_i, ld s_i
    std::vector<int64_t> PU_off;
    DBuf<double> PU;
    // B_ij (i < j) for Type-1 / Type-3 pairs at this level: r_i x r_j, ld r_i
    std::unordered_map<uint64_t, int64_t> B_off;
    DBuf<double> B;
    std::vector<int> piv;           // host copy of the QRCP pivots (w per node)
};

}  // namespace spd

struct spd_hss_s {
    uint32_t magic = 0x48535348u;    // 'HSSH'
    spd_h2_s* h2 = nullptr;
    int cap = 0, p = 0, w = 0;
    double tol = 0.0;
    std::vector<spd::HssLevel> lv;   // levels 1..L (level L: root factor only)
    double timings[16] = {0};
    int64_t shard_work[2] = {0, 0};  // nodes factorised by this process / nodes (sharding evidence)
    int64_t sketch_groups = 0;       // instrumentation: number of Y^(k) sketch groups
    // solve workspace
    int64_t ws_k = 0;
    spd::DBuf<double> bt, xt;
    // dense operator of the top of the solve recursion (levels > gt_level, root): the
    // linear map zh (level gt_level coefficients) -> xh; replaces 2 (L - 1 - gt_level) + 2
    // dependent single-vector phases by one GEMV (0: not built)
    int gt_level = 0;
    int64_t gt_R = 0;
    spd::DBuf<double> Gtop, gt_out;
    std::vector<spd::DBuf<double>> z, ub, zs;
};

namespace spd {
void hss_build_impl(spd_hss_s* H, const double* omega, uint64_t seed, cudaStream_t s);
// k = 1 fused per-level solve (hsolve.cu); z: N workspace, zl[l] / ub[l]: level workspaces
void hss_solve_vec(spd_hss_s* H, const double* b, double* x, double* z, const std::vector<double*>& zl,
                   const std::vector<double*>& zs, const std::vector<double*>& ub, cudaStream_t s);
void hss_solve_tree(spd_hss_s* H, const double* b, int64_t ldb, double* x, int64_t ldx, int k, cudaStream_t s);
// y = H x, the SPD-HSS matrix itself (tree order; x, y N x k, ld >= N; y overwritten)
void hss_apply_tree(spd_hss_s* H, const double* x, int64_t ldx, double* y, int64_t ldy, int k, cudaStream_t s);
void hss_query(const spd_hss_s* H, int what, void* buf, size_t bytes);
// precond: PC_HSS (the SPD-HSS solve), PC_BJ (block Jacobi from its leaf factors); M == nullptr: none
enum { PC_HSS = 0, PC_BJ = 1 };
void pcg_tree(spd_h2_s* A, spd_hss_s* M, const double* b, double* x, double tol, int maxit, spd_pcg_report* rep,
              cudaStream_t s, int precond = PC_HSS);
void bj_solve_vec(spd_hss_s* H, const double* b, double* x, double* z, cudaStream_t s);
// persistent (cooperative) PCG kernel, pcgk.cu
struct PcgPersistent {
    struct Impl;
    Impl* impl = nullptr;
    ~PcgPersistent();
};
bool pcg_persistent_prepare(PcgPersistent& pk, spd_h2_s* A, spd_hss_s* M, double* x, double* r, double* p, double* q,
                            double* z, cudaStream_t s, int precond = 0);
// out: ||r||^2, iterations, converged, error (1: p^T A p <= 0, 2: r^T M r <= 0)
void pcg_persistent_run(PcgPersistent& pk, double rz, double nb, double tol, int maxit, double out[4], cudaStream_t s);
const spd_hss_s* hss_if_hss(const void* handle);      // nullptr when handle is not an HSS
void philox_normal(cudaStream_t s, double* out, int64_t n, int w, uint64_t seed);   // Omega (R29)
const double* hss_timings(const spd_hss_s* H);
const int64_t* hss_shard_work(const spd_hss_s* H);
inline uint64_t pair_key(int i, int j) { return ((uint64_t)(uint32_t)i << 32) | (uint32_t)j; }
}  // namespace spd
