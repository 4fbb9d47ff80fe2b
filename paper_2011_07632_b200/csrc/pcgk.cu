// pcgk.cu -- persistent PCG: the whole iteration loop of PAPER.md P:1131-1132
// (reading R15) in ONE cooperative kernel.
//
// One PCG iteration is a chain of ~4L dependent phases (H2 up levels, symmetric
// near + coupling blocks, gather, H2 down levels, p^T q, x/r update + ||r||^2, HSS
// solve up levels / root / down levels, r^T z, p update), most of them a few
// microseconds of work.  Launched one kernel per phase (even from a CUDA graph) the
// iteration is dominated by launch latency; here every CTA (one per SM, 16 warps)
// loops over the iterations and over the phases, takes its share of each phase's
// work items (the same device bodies as the stand-alone kernels, phases.cuh) and
// meets the others at a grid barrier.  Dot products are reduced in a fixed order
// by every CTA redundantly, so all CTAs agree bitwise on alpha, beta and the stop
// test and no host round trip happens per iteration.
#include <cooperative_groups.h>
#include "hss.hpp"
#include "phases.cuh"
#include <algorithm>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <unordered_map>

namespace cg = cooperative_groups;

namespace spd {

constexpr int PK_MAXPH = 64;
constexpr int PK_MAXID = 16;       // fused identity levels at most
#ifndef PCG_CTAS
#define PCG_CTAS 2                 // CTAs per SM of the all-stored variant
#endif

struct PcgPlan {
    int64_t N;
    int maxit;
    double tol, nb;                // stop: sqrt(||r||^2) / ||b|| <= tol (as in pcg_tree)
    double *x, *r, *p, *q, *z;     // tree order
    double* part;                  // 3 x gridDim partial sums
    double* scal;                  // [0] rz (in); out: [1] relres^2 * bb, [2] iters, [3] converged, [4] error
    // H2 product q = A p
    int nup, ndn;                  // number of basis levels
    const BasisItem* up; int up_off[PK_MAXPH + 1];
    const BasisItem* dn; int dn_off[PK_MAXPH + 1];
    const SymPiece* pieces; int npieces;
    const double* vals; double* scratch;
    const SymGNode* gnodes; int ngnodes, nbig; const SymContrib* gcon; int nbmax;
    SymVecs xin; SymVecsOut yout;
    KernelParams kp; double shift; int d;
    // identity levels 1..nid (every node keeps all its candidates, T empty): their up passes
    // are gathers xh_l[k] = p[idb[..]] done in the first up phase together with level
    // nid + 1 (whose items read p through composed pivots), their down passes one phase
    // q[o] += yh_1[a_1(o)] + (... + yh_nid[a_nid(o)]) in the order of the level-by-level sums
    int nid, id_tot;
    const int* idb; int id_beg[PK_MAXID + 1];
    const int* ida;                // nid x N, -1: no coefficient
    // HSS solve z = M r
    int nhs;
    const HsNode* hs; const HsItem* hsi; int hs_off[PK_MAXPH + 1];
    unsigned char hs_cta[PK_MAXPH];   // 1: phase of CTA items (dense top operator), 0: warp items
    double* id_xh[PK_MAXID];
    double* id_yh[PK_MAXID];
    unsigned long long* trace;     // optional: globaltimer after every phase of iteration 2 (CTA 0)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double cta_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < PH_W ? red[lane] : 0.0;
        t = warp_sum(t);
    }
    __syncthreads();
    return t;      // valid in warp 0
}

// every CTA: sum of the gridDim partials in a fixed order (bitwise identical in all CTAs)
__device__ __forceinline__ double grid_total(const double* part, double* bc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) {
        double t = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) t += ldv(part + b);
        t = warp_sum(t);
        if (lane == 0) *bc = t;
    }
    __syncthreads();
    const double v = *bc;
    __syncthreads();
    return v;
}

// EVAL = false: every symmetric block is stored (no evaluation path compiled in, <= 128
// registers, two CTAs per SM); EVAL = true: some blocks are evaluated (one CTA per SM)
template <int KID, bool EVAL>
__global__ void __launch_bounds__(PH_T, EVAL ? 1 : PCG_CTAS) pcg_persistent_kernel(PcgPlan P) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    __shared__ double red[PH_W], bc;
    const int64_t N = P.N;
    const int64_t stride = (int64_t)gridDim.x * PH_T;
    const int64_t i0 = (int64_t)blockIdx.x * PH_T + threadIdx.x;
    double* part_pq = P.part;
    double* part_rr = P.part + gridDim.x;
    double* part_rz = P.part + 2 * gridDim.x;
    double rz = ldv(P.scal);
    int iters = 0, conv = 0, err = 0;
    double rr = 0.0;
    int nph = 0;
    auto sync = [&](int it) {
        grid.sync();
        if (P.trace && it == 2 && blockIdx.x == 0 && threadIdx.x == 0) P.trace[nph++] = gtimer();
    };
    for (int it = 1; it <= P.maxit; ++it) {
        if (P.trace && it == 2 && blockIdx.x == 0 && threadIdx.x == 0) P.trace[nph++] = gtimer();
        // ---------------- q = A p (H2, k = 1)
        for (int l = 0; l < P.nup; ++l) {
            if (l == 0 && P.nid)
                for (int64_t e = i0; e < P.id_tot; e += stride) {
                    int lv = 0;
                    while (e >= P.id_beg[lv + 1]) ++lv;
                    P.id_xh[lv][e - P.id_beg[lv]] = ldv(P.p + P.idb[e]);
                }
            for (int w = P.up_off[l] + blockIdx.x; w < P.up_off[l + 1]; w += gridDim.x) basis_up_item(P.up[w], sm);
            sync(it);
        }
        {
            constexpr int NG = PH_T / (SY_NW * 32);
            const int grp = threadIdx.x / (SY_NW * 32);
            for (int w = blockIdx.x * NG + grp; w < P.npieces; w += gridDim.x * NG)
                sym_piece<KID, EVAL>(P.pieces[w], P.xin, P.vals, P.scratch, P.kp, P.shift, P.d, grp,
                               sm + grp * SY_NW * P.nbmax);
            sync(it);
        }
        for (int w = blockIdx.x; w < P.nbig; w += gridDim.x) gather_item_cta(P.gnodes[w], P.gcon, P.yout, P.scratch, sm);
        for (int w = P.nbig + blockIdx.x * PH_W + (threadIdx.x >> 5); w < P.ngnodes; w += gridDim.x * PH_W)
            gather_item_warp(P.gnodes[w], P.gcon, P.yout, P.scratch);
        sync(it);
        for (int l = 0; l < P.ndn; ++l) {
            for (int w = P.dn_off[l] + blockIdx.x; w < P.dn_off[l + 1]; w += gridDim.x) basis_down_item(P.dn[w], sm);
            sync(it);
        }
        // ---------------- identity-level scatters (fused) and alpha = rz / p^T q
        {
            double s = 0.0;
            for (int64_t o = i0; o < N; o += stride) {
                double qo = ldv(P.q + o);
                if (P.nid) {
                    double acc = 0.0;
                    bool has = false;
                    for (int lv = P.nid - 1; lv >= 0; --lv) {
                        const int a = P.ida[(size_t)lv * N + o];
                        if (a < 0) continue;
                        const double v = ldv(P.id_yh[lv] + a);
                        acc = has ? v + acc : v;
                        has = true;
                    }
                    if (has) { qo = qo + acc; P.q[o] = qo; }
                }
                s += ldv(P.p + o) * qo;
            }
            s = cta_sum(s, red);
            if (threadIdx.x == 0) part_pq[blockIdx.x] = s;
        }
        sync(it);
        const double pq = grid_total(part_pq, &bc);
        if (!(pq > 0.0)) { err = 1; iters = it; break; }
        const double alpha = rz / pq;
        {
            double s = 0.0;
            for (int64_t i = i0; i < N; i += stride) {
                P.x[i] = ldv(P.x + i) + alpha * ldv(P.p + i);
                const double ri = ldv(P.r + i) - alpha * ldv(P.q + i);
                P.r[i] = ri;
                s += ri * ri;
            }
            s = cta_sum(s, red);
            if (threadIdx.x == 0) part_rr[blockIdx.x] = s;
        }
        sync(it);
        rr = grid_total(part_rr, &bc);
        iters = it;
        if (sqrt(rr) / P.nb <= P.tol) { conv = 1; break; }
        // ---------------- z = M r (HSS solve, k = 1)
        for (int l = 0; l < P.nhs; ++l) {
            if (P.hs_cta[l]) {
                for (int w = P.hs_off[l] + blockIdx.x; w < P.hs_off[l + 1]; w += gridDim.x) hss_item(P.hs, P.hsi[w], sm);
            } else {
                for (int w = P.hs_off[l] + blockIdx.x * PH_W + (threadIdx.x >> 5); w < P.hs_off[l + 1];
                     w += gridDim.x * PH_W)
                    hss_item_warp(P.hs, P.hsi[w]);
            }
            sync(it);
        }
        // ---------------- beta = r^T z / rz ; p = z + beta p
        {
            double s = 0.0;
            for (int64_t i = i0; i < N; i += stride) s += ldv(P.r + i) * ldv(P.z + i);
            s = cta_sum(s, red);
            if (threadIdx.x == 0) part_rz[blockIdx.x] = s;
        }
        sync(it);
        const double rzn = grid_total(part_rz, &bc);
        if (!(rzn > 0.0)) { err = 2; break; }
        const double beta = rzn / rz;
        rz = rzn;
        for (int64_t i = i0; i < N; i += stride) P.p[i] = ldv(P.z + i) + beta * ldv(P.p + i);
        sync(it);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.scal[1] = rr;
        P.scal[2] = iters;
        P.scal[3] = conv;
        P.scal[4] = err;
    }
}

// ---------------------------------------------------------------- host
struct PcgPersistent::Impl {
    PcgPlan plan{};
    DBuf<char> arena;
    DBuf<double> part, scal;
    size_t smem = 0;
    int grid = 0;
    double bytes_per_iter = 0.0;
    bool eval = false;
    DBuf<unsigned long long> trace;
};

PcgPersistent::~PcgPersistent() { delete impl; }

template <class T>
static const T* put(std::vector<char>& buf, const std::vector<T>& v, std::vector<size_t>& fix) {
    size_t off = (buf.size() + 255) & ~(size_t)255;
    buf.resize(off + v.size() * sizeof(T));
    if (!v.empty()) memcpy(buf.data() + off, v.data(), v.size() * sizeof(T));
    fix.push_back(off);
    return (const T*)(uintptr_t)off;     // relocated after upload
}

static void* kernel_ptr(int kid, bool eval) {
    switch (kid) {
    case SPD_K_GAUSSIAN: return eval ? (void*)pcg_persistent_kernel<SPD_K_GAUSSIAN, true> : (void*)pcg_persistent_kernel<SPD_K_GAUSSIAN, false>;
    case SPD_K_MATERN32: return eval ? (void*)pcg_persistent_kernel<SPD_K_MATERN32, true> : (void*)pcg_persistent_kernel<SPD_K_MATERN32, false>;
    case SPD_K_EXPONENTIAL: return eval ? (void*)pcg_persistent_kernel<SPD_K_EXPONENTIAL, true> : (void*)pcg_persistent_kernel<SPD_K_EXPONENTIAL, false>;
    case SPD_K_RPY: return eval ? (void*)pcg_persistent_kernel<SPD_K_RPY, true> : (void*)pcg_persistent_kernel<SPD_K_RPY, false>;
    default: return eval ? (void*)pcg_persistent_kernel<SPD_K_IMQ, true> : (void*)pcg_persistent_kernel<SPD_K_IMQ, false>;
    }
}

bool pcg_persistent_prepare(PcgPersistent& pk, spd_h2_s* A, spd_hss_s* M, double* x, double* r, double* p, double* q,
                            double* z, cudaStream_t s, int precond) {
    const TreeH& t = A->tree;
    const int L = t.L;
    if (L < 2 || !M || A->stored_mode != 1) return false;
    h2sym_build(A, A->sym_budget, s);
    // blocks evaluated on the fly: the stand-alone kernels (CUDA-graph path) run them at
    // full occupancy, the persistent kernel would with 8 warps per SM
    if (A->sym.stored_frac < 1.0 && !getenv("SPD_PCG_PERSISTENT_EVAL")) return false;
    stage_mark(s, "pcg h2sym_build");
    auto* im = new PcgPersistent::Impl();
    pk.impl = im;
    PcgPlan& P = im->plan;
    P.N = A->N;
    P.x = x; P.r = r; P.p = p; P.q = q; P.z = z;
    // H2 product: xh/yh workspaces of the handle (k = 1)
    std::vector<double*> xh(L, nullptr), yh(L, nullptr);
    for (int lk = 1; lk < L; ++lk) { xh[lk] = A->xh[lk].p; yh[lk] = A->yh[lk].p; }
    int ncmax = 1, smax = 1;
    auto up = basis_up_plan(A, p, xh, L - 1, &ncmax, nullptr);
    auto dn = basis_down_plan(A, yh, L - 1, q, &smax, nullptr);
    // HSS solve plan on the handle's k = 1 workspaces
    std::vector<double*> zl(L + 1, nullptr), zs(L + 1, nullptr), ub(L + 1, nullptr);
    for (int l = 1; l < L; ++l) { zl[l] = M->z[l].p; zs[l] = M->zs[l].p; }
    for (int l = 2; l <= L; ++l) ub[l] = M->ub[l].p;
    auto hs = precond == 1 ? bj_solve_plan(M, r, z, M->bt.p) : hss_solve_plan(M, r, z, M->bt.p, zl, zs, ub);
    if ((int)hs.size() > PK_MAXPH || L - 1 > PK_MAXPH) return false;
    std::vector<char> buf;
    std::vector<size_t> fix;
    std::vector<BasisItem> upf, dnf;
    // ---- identity levels (bitwise-equal fusion of their gathers / scatters; see PcgPlan)
    int nid = 0;
    for (int lk = 1; lk < L - 1 && !getenv("SPD_PCG_NOFUSE"); ++lk) {
        const H2Level& lv = A->lv[lk];
        bool idl = true;
        for (int a = 0; a < lv.count && idl; ++a) idl = lv.rank[a] == lv.ncand[a];
        if (!idl) break;
        nid = lk;
    }
    if (nid > PK_MAXID) nid = PK_MAXID;
    std::vector<int> idb_h, ida_h, comp_h;
    std::vector<int64_t> comp_off;
    if (nid) {
        std::vector<std::vector<int>> bmap(nid + 1);
        P.id_beg[0] = 0;
        for (int lk = 1; lk <= nid + 1; ++lk) {
            const H2Level& lv = A->lv[lk];
            const std::vector<int> piv = lv.piv.download(s);
            if (lk <= nid) bmap[lk].assign(std::max<int64_t>(0, lv.S), -1);
            if (lk == nid + 1) comp_off.assign(lv.count + 1, 0);
            for (int a = 0; a < lv.count; ++a) {
                const int i = lv.first + a, sr = lv.rank[a], nc = lv.ncand[a];
                auto cand_row = [&](int e) -> int {      // row of x behind candidate e of node a
                    if (lk == 1) return (int)(t.begin[i] + e);
                    const H2Level& pv = A->lv[lk - 1];
                    return bmap[lk - 1][pv.off[2 * i + 1 - pv.first] + e];
                };
                if (lk <= nid) {
                    for (int k = 0; k < sr; ++k) bmap[lk][lv.off[a] + k] = cand_row(piv[lv.piv_off[a] + k]);
                } else {
                    comp_off[a + 1] = comp_off[a] + (sr ? nc : 0);
                    if (sr)
                        for (int k = 0; k < nc; ++k) comp_h.push_back(cand_row(piv[lv.piv_off[a] + k]));
                }
            }
            if (lk <= nid) {
                idb_h.insert(idb_h.end(), bmap[lk].begin(), bmap[lk].end());
                P.id_beg[lk] = (int)idb_h.size();
                P.id_xh[lk - 1] = xh[lk];
                P.id_yh[lk - 1] = yh[lk];
            }
        }
        ida_h.assign((size_t)nid * A->N, -1);
        for (int lk = 1; lk <= nid; ++lk)
            for (size_t e = 0; e < bmap[lk].size(); ++e)
                if (bmap[lk][e] >= 0) ida_h[(size_t)(lk - 1) * A->N + bmap[lk][e]] = (int)e;
    }
    P.nid = nid;
    P.id_tot = (int)idb_h.size();
    P.nup = 0;
    P.up_off[0] = 0;
    for (int lk = nid + 1; lk < L; ++lk) {
        if (up[lk].empty()) continue;
        upf.insert(upf.end(), up[lk].begin(), up[lk].end());
        P.up_off[++P.nup] = (int)upf.size();
    }
    if (nid && P.nup == 0) { P.nup = 1; P.up_off[1] = 0; }   // a phase for the gathers alone
    P.ndn = 0;
    P.dn_off[0] = 0;
    for (int lk = L - 1; lk >= nid + 1; --lk) {
        if (dn[lk].empty()) continue;
        dnf.insert(dnf.end(), dn[lk].begin(), dn[lk].end());
        P.dn_off[++P.ndn] = (int)dnf.size();
    }
    std::vector<HsNode> hsf;
    std::vector<HsItem> hsi;
    int nsm_dev = 148;
    {
        int dv = 0;
        SPD_CUDA(cudaGetDevice(&dv));
        SPD_CUDA(cudaDeviceGetAttribute(&nsm_dev, cudaDevAttrMultiProcessorCount, dv));
    }
    P.nhs = 0;
    P.hs_off[0] = 0;
    int mmax = 1, rmax = 1;
    for (const auto& ph : hs) {
        if (ph.items.empty()) continue;
        const int base = (int)hsf.size();
        for (const auto& nd : ph.nodes) {
            mmax = std::max(mmax, nd.m);
            rmax = std::max(rmax, nd.r);
            if (ph.mode != 3 && nd.m > 32 * HS_MT) return false;
        }
        hsf.insert(hsf.end(), ph.nodes.begin(), ph.nodes.end());
        for (auto itm : ph.items) { itm.node += base; hsi.push_back(itm); }
        P.hs_cta[P.nhs] = (!hss_phase_uses_warps(ph.mode, ph.items.size(), nsm_dev) || getenv("SPD_HSS_CTA")) ? 1 : 0;
        P.hs_off[++P.nhs] = (int)hsi.size();
    }
    const int* idb_rel = put(buf, idb_h, fix);
    const int* ida_rel = put(buf, ida_h, fix);
    const int* comp_rel = put(buf, comp_h, fix);
    const BasisItem* up_rel = put(buf, upf, fix);
    const BasisItem* dn_rel = put(buf, dnf, fix);
    const HsNode* hs_rel = put(buf, hsf, fix);
    const HsItem* hsi_rel = put(buf, hsi, fix);
    im->arena.alloc(std::max<size_t>(1, buf.size()));
    if (nid && !up[nid + 1].empty()) {
        // level nid + 1 reads p directly: its pivots composed with the identity levels' maps
        const H2Level& lv = A->lv[nid + 1];
        std::unordered_map<int64_t, int> node_of;
        for (int a = 0; a < lv.count; ++a) node_of[lv.piv_off[a]] = a;
        BasisItem* items = (BasisItem*)(buf.data() + (uintptr_t)up_rel);
        for (int w = 0; w < P.up_off[1]; ++w) {
            const int a = node_of.at((int64_t)(items[w].piv - lv.piv.p));
            items[w].in = p;
            items[w].piv = (const int*)(im->arena.p + (uintptr_t)comp_rel) + comp_off[a];
        }
    }
    SPD_CUDA(cudaMemcpyAsync(im->arena.p, buf.data(), buf.size(), cudaMemcpyHostToDevice, s));
    P.up = (const BasisItem*)(im->arena.p + (uintptr_t)up_rel);
    P.idb = (const int*)(im->arena.p + (uintptr_t)idb_rel);
    P.ida = (const int*)(im->arena.p + (uintptr_t)ida_rel);
    P.dn = (const BasisItem*)(im->arena.p + (uintptr_t)dn_rel);
    P.hs = (const HsNode*)(im->arena.p + (uintptr_t)hs_rel);
    P.hsi = (const HsItem*)(im->arena.p + (uintptr_t)hsi_rel);
    const H2SymStore& st = A->sym;
    P.pieces = st.pieces.p; P.npieces = st.npieces;
    P.vals = st.vals.p; P.scratch = st.scratch.p;
    P.gnodes = st.gnodes.p; P.ngnodes = st.ngnodes; P.nbig = st.nbig; P.gcon = st.gcon.p; P.nbmax = st.nbmax;
    P.xin.p[0] = p; P.yout.p[0] = q;
    for (int lk = 1; lk < L; ++lk) { P.xin.p[lk] = xh[lk]; P.yout.p[lk] = yh[lk]; }
    P.kp = A->kp; P.shift = A->kern.shift; P.d = A->d;
    // shared memory: the largest body
    const size_t sm_d = std::max<size_t>({(size_t)hss_item_smem_doubles(mmax, rmax), (size_t)ncmax + PH_W * 32,
                                          (size_t)smax + PH_W * 32, (size_t)PH_W * 32,
                                          (size_t)(PH_T / 32) * st.nbmax});
    im->smem = sizeof(double) * sm_d;
    if (im->smem > 200 * 1024) return false;
    im->eval = st.stored_frac < 1.0;
    void* kfn = kernel_ptr(A->kp.id, im->eval);
    SPD_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)im->smem));
    int dev = 0, nsm = 0, per = 0;
    SPD_CUDA(cudaGetDevice(&dev));
    SPD_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    SPD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, PH_T, im->smem));
    if (per < 1) return false;
    im->grid = nsm * std::min(per, im->eval ? 1 : PCG_CTAS);    // all CTAs co-resident (cooperative launch)
    im->part.alloc((size_t)3 * im->grid);
    im->scal.alloc(8);
    P.part = im->part.p;
    P.scal = im->scal.p;
    P.trace = nullptr;
    if (getenv("SPD_PCG_TRACE")) {
        im->trace.alloc(4 * PK_MAXPH);
        im->trace.zero(s);
        P.trace = im->trace.p;
    }
    // algorithmic bytes of one iteration: stored blocks + basis T (up and down) + HSS factors + vectors
    double by = st.bytes;
    for (int lk = 1; lk < L; ++lk) {
        const H2Level& lv = A->lv[lk];
        for (int a = 0; a < lv.count; ++a) by += 2.0 * 8.0 * (double)lv.rank[a] * (lv.ncand[a] - lv.rank[a]);
    }
    for (const auto& nd : hsf) by += nd.P ? 8.0 * (0.5 * nd.m * (nd.m + 1) + (double)nd.m * nd.r) : 8.0 * (double)nd.m * nd.m;
    by += 8.0 * 14.0 * A->N;
    im->bytes_per_iter = by;
    return true;
}

// iterations 1..maxit from the state (x, r, p, z, rz = scal[0]) already on the device
void pcg_persistent_run(PcgPersistent& pk, double rz, double nb, double tol, int maxit, double out[4], cudaStream_t s) {
    auto* im = pk.impl;
    PcgPlan P = im->plan;
    P.maxit = maxit;
    P.nb = nb;
    P.tol = tol;
    SPD_CUDA(cudaMemcpyAsync(im->scal.p, &rz, sizeof(double), cudaMemcpyHostToDevice, s));
    void* args[] = {(void*)&P};
    {
        ProfScope prof(s, "pcg_persistent", 0, 0);
        SPD_CUDA(cudaLaunchCooperativeKernel(kernel_ptr(P.kp.id, im->eval), dim3(im->grid), dim3(PH_T), args, im->smem, s));
        count_launch();
    }
    double h[8];
    SPD_CUDA(cudaMemcpyAsync(h, im->scal.p, sizeof(double) * 8, cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    out[0] = h[1]; out[1] = h[2]; out[2] = h[3]; out[3] = h[4];
    if (P.trace) {
        std::vector<unsigned long long> tr = im->trace.download(s);
        fprintf(stderr, "[pcg trace] phases of iteration 2 (us):");
        for (size_t i = 1; i < tr.size() && tr[i]; ++i) fprintf(stderr, " %.1f", (tr[i] - tr[i - 1]) * 1e-3);
        fprintf(stderr, "\n[pcg trace] up %d, down %d, hss %d levels; pieces %d, gather nodes %d\n", P.nup, P.ndn,
                P.nhs, P.npieces, P.ngnodes);
    }
    prof_update_last("pcg_persistent", 0.0, im->bytes_per_iter * h[2]);
}

}  // namespace spd
