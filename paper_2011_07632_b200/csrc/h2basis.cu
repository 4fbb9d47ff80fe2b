// h2basis.cu -- single-vector H2 basis passes in interpolative form (k = 1).
//
// The nested interpolation matrices of the proxy-point ID (reading R4;
// eqn:nested P:218-226) have s_i identity rows: E_i[piv[k], k] = 1 for k < s_i
// and E_i[piv[s_i + c], :] = T_i[:, c]^T with T_i = R11^{-1} R12 (s_i x (n_c - s_i)).
// So the upward pass  xh_i = E_i^T x_c  is a gather plus T_i x_c[piv[s:]], and the
// downward pass  y_c += E_i yh_i  a scatter plus T_i^T yh_i: only T_i is read
// (at tol 1e-10 the leaf and lower-level ranks are close to n_c, so T_i is much
// smaller than E_i).  One launch per level; the work item is a 32-row tile.
#include "h2.hpp"
#include "phases.cuh"
#include <algorithm>

namespace spd {

__global__ void __launch_bounds__(PH_T) basis_up_kernel(const BasisItem* __restrict__ items) {
    extern __shared__ double sm[];
    basis_up_item(items[blockIdx.x], sm);
}
__global__ void __launch_bounds__(PH_T) basis_down_kernel(const BasisItem* __restrict__ items) {
    extern __shared__ double sm[];
    basis_down_item(items[blockIdx.x], sm);
}

// work items of the up pass, level 1..top (levels[l]); smax_out: largest n_c - s
std::vector<std::vector<BasisItem>> basis_up_plan(const spd_h2_s* h, const double* x, const std::vector<double*>& xh,
                                                  int top, int* ncmax_out, std::vector<double>* bytes,
                                                  const BasisFilter* f) {
    const TreeH& t = h->tree;
    std::vector<std::vector<BasisItem>> out(top + 1);
    int ncmax = 1;
    if (bytes) bytes->assign(top + 1, 0.0);
    for (int lk = 1; lk <= top; ++lk) {
        const H2Level& lv = h->lv[lk];
        for (int a = 0; a < lv.count; ++a) {
            const int sr = lv.rank[a];
            if (sr == 0 || (f && !f->keep(lk, lv.count, a))) continue;
            const int i = lv.first + a;
            const double* in;
            if (lk == 1) in = x + t.begin[i];
            else {
                const H2Level& pv = h->lv[lk - 1];
                in = xh[lk - 1] + pv.off[2 * i + 1 - pv.first];
            }
            const int nc = lv.ncand[a];
            ncmax = std::max(ncmax, nc - sr);
            if (bytes) (*bytes)[lk] += 8.0 * ((double)sr * (nc - sr) + nc + sr);
            for (int tl = 0; tl * 32 < sr; ++tl)
                out[lk].push_back({in, xh[lk] + lv.off[a], lv.T.p + lv.T_off[a], lv.piv.p + lv.piv_off[a], sr, nc, tl});
        }
    }
    if (ncmax_out) *ncmax_out = ncmax;
    return out;
}

// work items of the down pass, level 1..top (levels[l]); smax_out: largest s
std::vector<std::vector<BasisItem>> basis_down_plan(const spd_h2_s* h, const std::vector<double*>& yh, int top,
                                                    double* y, int* smax_out, std::vector<double>* bytes,
                                                    const BasisFilter* f) {
    const TreeH& t = h->tree;
    std::vector<std::vector<BasisItem>> out(top + 1);
    int smax = 1;
    if (bytes) bytes->assign(top + 1, 0.0);
    for (int lk = top; lk >= 1; --lk) {
        const H2Level& lv = h->lv[lk];
        for (int a = 0; a < lv.count; ++a) {
            const int sr = lv.rank[a];
            if (sr == 0 || (f && !f->keep(lk, lv.count, a))) continue;
            const int i = lv.first + a;
            double* o;
            if (lk == 1) o = y + t.begin[i];
            else {
                const H2Level& pv = h->lv[lk - 1];
                o = yh[lk - 1] + pv.off[2 * i + 1 - pv.first];
            }
            const int nc = lv.ncand[a];
            smax = std::max(smax, sr);
            if (bytes) (*bytes)[lk] += 8.0 * ((double)sr * (nc - sr) + 2.0 * nc + sr);
            const int ntile = std::max(ceil_div(sr, 32), ceil_div(nc - sr, 32));
            for (int tl = 0; tl < ntile; ++tl)
                out[lk].push_back({yh[lk] + lv.off[a], o, lv.T.p + lv.T_off[a], lv.piv.p + lv.piv_off[a], sr, nc, tl});
        }
    }
    if (smax_out) *smax_out = smax;
    return out;
}

// xh[l] = E^T [x_leaf | xh children] for levels 1..top (k = 1)
void h2_up_vec(const spd_h2_s* h, const double* x, const std::vector<double*>& xh, int top, cudaStream_t s,
               const BasisFilter* f) {
    int ncmax = 1;
    std::vector<double> by;
    auto plan = basis_up_plan(h, x, xh, top, &ncmax, &by, f);
    const size_t smem = sizeof(double) * (ncmax + PH_W * 32);
    if (smem > 48 * 1024)
        SPD_CUDA(cudaFuncSetAttribute(basis_up_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int lk = 1; lk <= top; ++lk) {
        if (plan[lk].empty()) continue;
        DevArray<BasisItem> di(s, plan[lk]);
        ProfScope prof(s, "basis_vec", 0, by[lk]);
        basis_up_kernel<<<(unsigned)plan[lk].size(), PH_T, smem, s>>>(di.p);
        SPD_LAUNCH();
    }
}

// children of level-l nodes += E yh[l] for l = top..2; y_leaf += E yh[1]  (k = 1)
void h2_down_vec(const spd_h2_s* h, const std::vector<double*>& yh, int top, double* y, cudaStream_t s,
                 const BasisFilter* f) {
    int smax = 1;
    std::vector<double> by;
    auto plan = basis_down_plan(h, yh, top, y, &smax, &by, f);
    const size_t smem = sizeof(double) * (smax + PH_W * 32);
    if (smem > 48 * 1024)
        SPD_CUDA(cudaFuncSetAttribute(basis_down_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int lk = top; lk >= 1; --lk) {
        if (plan[lk].empty()) continue;
        DevArray<BasisItem> di(s, plan[lk]);
        ProfScope prof(s, "basis_vec", 0, by[lk]);
        basis_down_kernel<<<(unsigned)plan[lk].size(), PH_T, smem, s>>>(di.p);
        SPD_LAUNCH();
    }
}

}  // namespace spd
