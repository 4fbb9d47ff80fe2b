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
#include <algorithm>

namespace spd {

struct BasisItem {
    const double* in;     // up: x_c (n_c) ; down: yh_i (s)
    double* out;          // up: xh_i (s)  ; down: y_c (n_c), accumulated
    const double* T;      // s x (n_c - s), ld s
    const int* piv;       // n_c
    int s, nc, tile;      // tile: 32-row tile of xh (up) / 32-column tile of T (down)
};

constexpr int BV_T = 512, BV_W = BV_T / 32;

// up: xh[k] = x[piv[k]] + sum_c T[k, c] x[piv[s + c]] for k in the tile (lane = k);
// warp w takes columns c = w (mod 16), 8 loads in flight per lane; the warp sums
// are added in warp order (deterministic)
__global__ void __launch_bounds__(BV_T) basis_up_kernel(const BasisItem* __restrict__ items) {
    extern __shared__ double xg[];                // gathered x[piv[s + c]], c < n_c - s
    __shared__ double red[BV_W][32];
    const BasisItem it = items[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = it.s, nr = it.nc - it.s;
    for (int c = threadIdx.x; c < nr; c += BV_T) xg[c] = it.in[it.piv[s + c]];
    __syncthreads();
    const int k = it.tile * 32 + lane;
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    if (k < s) {
        const double* p = it.T + k;
        int c = warp;
        for (; c + 7 * BV_W < nr; c += 8 * BV_W) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(p + (size_t)(c + u * BV_W) * s);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] += v[u] * xg[c + u * BV_W];
        }
        for (; c < nr; c += BV_W) acc[0] += __ldg(p + (size_t)c * s) * xg[c];
    }
    red[warp][lane] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    __syncthreads();
    if (warp == 0 && k < s) {
        double sum = it.in[it.piv[k]];
#pragma unroll
        for (int w = 0; w < BV_W; ++w) sum += red[w][lane];
        it.out[k] = sum;
    }
}

// down: y[piv[s + c]] += sum_k T[k, c] yh[k] for the tile's 32 columns c, and
// y[piv[k]] += yh[k] for k in [32 tile, 32 tile + 32).  Warp w takes the 32-row
// chunks q = w (mod 16) of T's tile: 32 coalesced loads (lane = row), scaled by
// yh, then a butterfly transpose-reduction leaves column c's partial in lane c.
__global__ void __launch_bounds__(BV_T) basis_down_kernel(const BasisItem* __restrict__ items) {
    extern __shared__ double yh[];
    __shared__ double red[BV_W][32];
    const BasisItem it = items[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = it.s, nr = it.nc - it.s;
    for (int k = threadIdx.x; k < s; k += BV_T) yh[k] = it.in[k];
    __syncthreads();
    const int k0 = it.tile * 32;
    if (warp == 0 && k0 + lane < s) it.out[it.piv[k0 + lane]] += yh[k0 + lane];
    const int c0 = k0, cn = min(32, nr - c0);
    if (cn <= 0) return;                         // whole CTA: no T columns in this tile
    double acc = 0.0;
    for (int q = warp; q * 32 < s; q += BV_W) {
        const int k = q * 32 + lane;
        const double y = k < s ? yh[k] : 0.0;
        const double* p = it.T + k + (size_t)c0 * s;
        double v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = (k < s && c < cn) ? __ldg(p + (size_t)c * s) : 0.0;
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] *= y;
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
        acc += v[0];
    }
    red[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && lane < cn) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < BV_W; ++w) sum += red[w][lane];
        it.out[it.piv[s + c0 + lane]] += sum;
    }
}

// xh[l] = E^T [x_leaf | xh children] for levels 1..top (k = 1)
void h2_up_vec(const spd_h2_s* h, const double* x, const std::vector<double*>& xh, int top, cudaStream_t s) {
    const TreeH& t = h->tree;
    for (int lk = 1; lk <= top; ++lk) {
        const H2Level& lv = h->lv[lk];
        std::vector<BasisItem> items;
        int ncmax = 1;
        double by = 0;
        for (int a = 0; a < lv.count; ++a) {
            const int sr = lv.rank[a];
            if (sr == 0) continue;
            const int i = lv.first + a;
            const double* in;
            if (lk == 1) in = x + t.begin[i];
            else {
                const H2Level& pv = h->lv[lk - 1];
                in = xh[lk - 1] + pv.off[2 * i + 1 - pv.first];
            }
            const int nc = lv.ncand[a];
            ncmax = std::max(ncmax, nc - sr);
            by += 8.0 * ((double)sr * (nc - sr) + nc + sr);
            for (int tl = 0; tl * 32 < sr; ++tl)
                items.push_back({in, xh[lk] + lv.off[a], lv.T.p + lv.T_off[a], lv.piv.p + lv.piv_off[a], sr, nc, tl});
        }
        if (items.empty()) continue;
        DevArray<BasisItem> di(s, items);
        const size_t smem = sizeof(double) * ncmax;
        if (smem > 48 * 1024)
            SPD_CUDA(cudaFuncSetAttribute(basis_up_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        ProfScope prof(s, "basis_vec", 0, by);
        basis_up_kernel<<<(unsigned)items.size(), BV_T, smem, s>>>(di.p);
        SPD_LAUNCH();
    }
}

// children of level-l nodes += E yh[l] for l = top..2; y_leaf += E yh[1]  (k = 1)
void h2_down_vec(const spd_h2_s* h, const std::vector<double*>& yh, int top, double* y, cudaStream_t s) {
    const TreeH& t = h->tree;
    for (int lk = top; lk >= 1; --lk) {
        const H2Level& lv = h->lv[lk];
        std::vector<BasisItem> items;
        int smax = 1;
        double by = 0;
        for (int a = 0; a < lv.count; ++a) {
            const int sr = lv.rank[a];
            if (sr == 0) continue;
            const int i = lv.first + a;
            double* out;
            if (lk == 1) out = y + t.begin[i];
            else {
                const H2Level& pv = h->lv[lk - 1];
                out = yh[lk - 1] + pv.off[2 * i + 1 - pv.first];
            }
            const int nc = lv.ncand[a];
            smax = std::max(smax, sr);
            by += 8.0 * ((double)sr * (nc - sr) + 2.0 * nc + sr);
            const int ntile = std::max(ceil_div(sr, 32), ceil_div(nc - sr, 32));
            for (int tl = 0; tl < ntile; ++tl)
                items.push_back({yh[lk] + lv.off[a], out, lv.T.p + lv.T_off[a], lv.piv.p + lv.piv_off[a], sr, nc, tl});
        }
        if (items.empty()) continue;
        DevArray<BasisItem> di(s, items);
        const size_t smem = sizeof(double) * smax;
        if (smem > 48 * 1024)
            SPD_CUDA(cudaFuncSetAttribute(basis_down_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        ProfScope prof(s, "basis_vec", 0, by);
        basis_down_kernel<<<(unsigned)items.size(), BV_T, smem, s>>>(di.p);
        SPD_LAUNCH();
    }
}

}  // namespace spd
