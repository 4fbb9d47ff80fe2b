// capi.cpp -- the extern "C" boundary of libspdhss (include/spdhss.h).
// Argument validation, error translation, layout handling.  No numerics here.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include "h2.hpp"
#include "hss.hpp"
#include "comm.hpp"
#include "../../include/spdhss_testing.h"

namespace spd {
static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }
}  // namespace spd


using namespace spd;

#define SPD_TRY(...)                                                      \
    try { __VA_ARGS__; return SPD_OK; }                                   \
    catch (const spd::Error& e) { set_last_error(e.what()); return e.code; } \
    catch (const std::bad_alloc&) { set_last_error("host allocation failed"); return SPD_ENOMEM; } \
    catch (const std::exception& e) { set_last_error(e.what()); return SPD_ECUDA; }

extern "C" {

const char* spd_last_error(void) { return g_last_error.c_str(); }

spd_status spd_comm_unique_id(void* out128) {
    SPD_TRY({
        SPD_REQUIRE(out128 != nullptr, "spd_comm_unique_id: out is NULL");
        comm_unique_id(out128);
    })
}

spd_status spd_comm_init(const void* id, int nranks, int rank, spd_comm_t* out) {
    SPD_TRY({
        SPD_REQUIRE(out != nullptr, "spd_comm_init: out is NULL");
        *out = comm_create(id, nranks, rank);
    })
}
spd_status spd_comm_init_host(const spd_host_coll* ops, int nranks, int rank, spd_comm_t* out) {
    SPD_TRY({
        SPD_REQUIRE(out != nullptr, "spd_comm_init_host: out is NULL");
        *out = comm_create_host(ops, nranks, rank);
    })
}
void spd_comm_free(spd_comm_t c) { comm_destroy(c); }

int spd_test_shard_owner(int nranks, int count, int a) {
    spd_comm_s c;
    c.nranks = nranks;
    return shard_owner(&c, count, a);
}

spd_status h2_build(const double* pts, int64_t n, int d, spd_kernel k, int leaf, double tol,
                    const spd_h2_opts* opts, spd_comm_t c, void* stream, spd_h2_t* out) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        SPD_REQUIRE(out != nullptr, "h2_build: out is NULL");
        *out = nullptr;
        SPD_REQUIRE(pts != nullptr && n >= 1, "h2_build: need n >= 1 points");
        SPD_REQUIRE(d == 2 || d == 3, "h2_build: d must be 2 or 3");
        SPD_REQUIRE(leaf >= 1, "h2_build: leaf >= 1");
        SPD_REQUIRE(tol >= 0.0 && tol < 1.0, "h2_build: tol in [0, 1)");
        SPD_REQUIRE(k.id >= 0 && k.id <= 4, "h2_build: unknown kernel id");
        SPD_REQUIRE(k.id != SPD_K_RPY || d == 3, "h2_build: the RPY kernel needs 3D points");
        SPD_REQUIRE(k.l > 0.0 && std::isfinite(k.l), "h2_build: kernel length l must be > 0");
        SPD_REQUIRE(k.shift >= 0.0 && std::isfinite(k.shift), "h2_build: shift must be >= 0");
        SPD_REQUIRE(n <= (int64_t)1 << 30, "h2_build: n too large");
        auto* h = new spd_h2_s();
        h->m = k.id == SPD_K_RPY ? 3 : 1;
        h->dim = d;
        h->N = n * h->m;                              // rows of the operator (dofs)
        h->d = d + (h->m > 1 ? 1 : 0);               // coordinate rows of X (RPY: + component)
        h->kern = k; h->kp = make_kernel(k); h->tol = tol; h->leaf = leaf;
        h->n_proxy = (opts && opts->n_proxy > 0) ? opts->n_proxy : (d == 2 ? 4096 : 6144);
        h->comm = c;
        h->inject = opts ? opts->inject_skeletons : nullptr;
        try { h2_build_impl(h, pts, (cudaStream_t)stream); }
        catch (...) { delete h; throw; }
        *out = h;
    })
}

void h2_free(spd_h2_t h) { if (h) { cudaDeviceSynchronize(); delete h; } }

spd_status h2_release_store(spd_h2_t h) {
    SPD_TRY({
        SPD_REQUIRE(h != nullptr, "h2_release_store: null handle");
        SPD_CUDA(cudaDeviceSynchronize());
        h->sym = spd::H2SymStore();
        h->kbc.valid = false;                      // its plan may point into the store
        h->kbc.plan = spd::KbPlan();
        h->stored_mode = -1;
        h->sym_budget = 0.0;
    })
}

spd_status h2_matvec(spd_h2_t h, int layout, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t k,
                     void* stream) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        SPD_REQUIRE(h != nullptr, "h2_matvec: null handle");
        SPD_REQUIRE(layout == SPD_LAYOUT_ORIGINAL || layout == SPD_LAYOUT_TREE, "h2_matvec: bad layout");
        SPD_REQUIRE(k >= 0 && ldx >= h->N && ldy >= h->N, "h2_matvec: ld must be >= n");
        SPD_REQUIRE(k <= (1 << 20), "h2_matvec: k too large");
        if (k == 0) return SPD_OK;
        SPD_REQUIRE(X != nullptr && Y != nullptr, "h2_matvec: null X or Y");
        cudaStream_t s = (cudaStream_t)stream;
        const bool shard = true;                   // products are subtree-sharded under a real communicator
        if (layout == SPD_LAYOUT_TREE) {
            h2_apply_tree(h, X, ldx, Y, ldy, (int)k, s, shard);
        } else {
            double *xt = nullptr, *yt = nullptr;
            h2_perm_ws(h, (int)k, &xt, &yt);
            permute_rows(s, h->perm.p, h->N, (int)k, X, ldx, xt, h->N, true);
            h2_apply_tree(h, xt, h->N, yt, h->N, (int)k, s, shard);
            permute_rows(s, h->perm.p, h->N, (int)k, yt, h->N, Y, ldy, false);
        }
    })
}

spd_status spdhss_build(spd_h2_t h, int rank_cap, double rel_tol, int oversample, uint64_t seed,
                        const double* omega, void* stream, spd_hss_t* out) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        SPD_REQUIRE(out != nullptr, "spdhss_build: out is NULL");
        *out = nullptr;
        SPD_REQUIRE(h != nullptr, "spdhss_build: null H2 handle");
        SPD_REQUIRE(rank_cap >= 0 && oversample >= 0 && rank_cap + oversample >= 1,
                    "spdhss_build: need rank_cap >= 0, oversample >= 0, rank_cap + oversample >= 1");
        SPD_REQUIRE(rel_tol >= 0.0 && rel_tol < 1.0, "spdhss_build: rel_tol in [0, 1)");
        auto* H = new spd_hss_s();
        H->h2 = h; H->cap = rank_cap; H->p = oversample; H->w = rank_cap + oversample; H->tol = rel_tol;
        try { hss_build_impl(H, omega, seed, (cudaStream_t)stream); }
        catch (...) { delete H; throw; }
        *out = H;
    })
}

spd_status spdhss_build_adaptive(spd_h2_t h, int r0, int r_max, double rel_tol, int oversample, uint64_t seed,
                                 const double* omega, void* stream, spd_hss_t* out, int* cap_out) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        SPD_REQUIRE(out != nullptr, "spdhss_build_adaptive: out is NULL");
        *out = nullptr;
        SPD_REQUIRE(h != nullptr, "spdhss_build_adaptive: null H2 handle");
        SPD_REQUIRE(r0 >= 1 && r_max >= r0 && oversample >= 0, "spdhss_build_adaptive: need 1 <= r0 <= r_max");
        SPD_REQUIRE(rel_tol >= 0.0 && rel_tol < 1.0, "spdhss_build_adaptive: rel_tol in [0, 1)");
        // grow Omega until every sketch Lambda_{ii^c} Omega is compressed to the
        // threshold (its rank stops on |R_tt| <= tol |R_00| below the cap); restart form:
        // cap = r0, 2 r0, ... up to r_max, Omega = the leading cap + p columns of one
        // sketch (Philox counters / the injected N x (r_max + p) matrix), reading R27
        int cap = r0;
        for (;;) {
            auto* H = new spd_hss_s();
            H->h2 = h; H->cap = cap; H->p = oversample; H->w = cap + oversample; H->tol = rel_tol;
            try { hss_build_impl(H, omega, seed, (cudaStream_t)stream); }
            catch (...) { delete H; throw; }
            int maxr = 0;
            for (size_t l = 1; l + 1 < H->lv.size(); ++l)
                for (int r : H->lv[l].rank) maxr = std::max(maxr, r);
            if (maxr < cap || cap >= r_max) {
                *out = H;
                if (cap_out) *cap_out = cap;
                break;
            }
            cudaStreamSynchronize((cudaStream_t)stream);
            delete H;
            cap = std::min(2 * cap, r_max);
        }
    })
}

void hss_free(spd_hss_t H) { if (H) { cudaDeviceSynchronize(); delete H; } }

spd_status hss_solve(spd_hss_t H, int layout, const double* B, int64_t ldb, double* X, int64_t ldx, int64_t nrhs,
                     void* stream) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        SPD_REQUIRE(H != nullptr, "hss_solve: null handle");
        SPD_REQUIRE(layout == SPD_LAYOUT_ORIGINAL || layout == SPD_LAYOUT_TREE, "hss_solve: bad layout");
        const int64_t N = H->h2->N;
        SPD_REQUIRE(nrhs >= 0 && ldb >= N && ldx >= N, "hss_solve: ld must be >= n");
        if (nrhs == 0) return SPD_OK;
        SPD_REQUIRE(B != nullptr && X != nullptr, "hss_solve: null B or X");
        cudaStream_t s = (cudaStream_t)stream;
        if (layout == SPD_LAYOUT_TREE) {
            hss_solve_tree(H, B, ldb, X, ldx, (int)nrhs, s);
        } else {
            DBuf<double> bt((size_t)N * nrhs), xt((size_t)N * nrhs);
            permute_rows(s, H->h2->perm.p, N, (int)nrhs, B, ldb, bt.p, N, true);
            hss_solve_tree(H, bt.p, N, xt.p, N, (int)nrhs, s);
            permute_rows(s, H->h2->perm.p, N, (int)nrhs, xt.p, N, X, ldx, false);
        }
    })
}

spd_status hss_matvec(spd_hss_t H, int layout, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t k,
                      void* stream) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        SPD_REQUIRE(H != nullptr, "hss_matvec: null handle");
        SPD_REQUIRE(layout == SPD_LAYOUT_ORIGINAL || layout == SPD_LAYOUT_TREE, "hss_matvec: bad layout");
        const int64_t N = H->h2->N;
        SPD_REQUIRE(k >= 0 && ldx >= N && ldy >= N, "hss_matvec: ld must be >= n");
        SPD_REQUIRE(k <= (1 << 20), "hss_matvec: k too large");
        if (k == 0) return SPD_OK;
        SPD_REQUIRE(X != nullptr && Y != nullptr, "hss_matvec: null X or Y");
        cudaStream_t s = (cudaStream_t)stream;
        if (layout == SPD_LAYOUT_TREE) {
            hss_apply_tree(H, X, ldx, Y, ldy, (int)k, s);
        } else {
            DBuf<double> xt((size_t)N * k), yt((size_t)N * k);
            permute_rows(s, H->h2->perm.p, N, (int)k, X, ldx, xt.p, N, true);
            hss_apply_tree(H, xt.p, N, yt.p, N, (int)k, s);
            permute_rows(s, H->h2->perm.p, N, (int)k, yt.p, N, Y, ldy, false);
        }
    })
}

static spd_status pcg_common(spd_h2_t A, spd_hss_t M, int precond, int layout, const double* b, double* x,
                             double tol, int maxit, spd_pcg_report* rep, void* stream) {
    spd_pcg_report local{};
    if (!rep) rep = &local;
    try {
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        SPD_REQUIRE(A != nullptr && b != nullptr && x != nullptr, "pcg_solve: null argument");
        SPD_REQUIRE(M == nullptr || M->h2 == A, "pcg_solve: preconditioner built from another H2");
        SPD_REQUIRE(layout == SPD_LAYOUT_ORIGINAL || layout == SPD_LAYOUT_TREE, "pcg_solve: bad layout");
        SPD_REQUIRE(tol >= 0.0 && maxit >= 0, "pcg_solve: tol >= 0, maxit >= 0");
        cudaStream_t s = (cudaStream_t)stream;
        const int64_t N = A->N;
        if (layout == SPD_LAYOUT_TREE) {
            pcg_tree(A, M, b, x, tol, maxit, rep, s, precond);
        } else {
            DBuf<double> bt(N), xt(N);
            permute_rows(s, A->perm.p, N, 1, b, N, bt.p, N, true);
            pcg_tree(A, M, bt.p, xt.p, tol, maxit, rep, s, precond);
            stage_mark(s, "pcg teardown");
            permute_rows(s, A->perm.p, N, 1, xt.p, N, x, N, false);
        }
        stage_mark(s, "pcg permute back");
        if (!rep->converged) {
            set_last_error("pcg_solve: not converged in maxit iterations");
            return SPD_ENOCONV;
        }
        return SPD_OK;
    } catch (const spd::Error& e) { set_last_error(e.what()); return e.code; }
    catch (const std::exception& e) { set_last_error(e.what()); return SPD_ECUDA; }
}

spd_status pcg_solve(spd_h2_t A, spd_hss_t M, int layout, const double* b, double* x, double tol, int maxit,
                     spd_pcg_report* rep, void* stream) {
    return pcg_common(A, M, PC_HSS, layout, b, x, tol, maxit, rep, stream);
}

spd_status pcg_solve_bj(spd_h2_t A, spd_hss_t M, int layout, const double* b, double* x, double tol, int maxit,
                        spd_pcg_report* rep, void* stream) {
    if (!M) { set_last_error("pcg_solve_bj: needs the SPD-HSS handle (its leaf factors)"); return SPD_EINVAL; }
    return pcg_common(A, M, PC_BJ, layout, b, x, tol, maxit, rep, stream);
}

static size_t need(size_t have, size_t want) {
    if (have < want) throw Error(SPD_EINVAL, "spd_query: buffer too small (" + std::to_string(want) + " bytes needed)");
    return want;
}

spd_status spd_query(const void* handle, int what, void* buf, size_t bytes) {
    SPD_TRY({
        SPD_REQUIRE(handle != nullptr && buf != nullptr, "spd_query: null argument");
        if (what >= SPD_Q_HSS_RANKS && what < SPD_Q_TIMINGS) {
            SPD_REQUIRE(hss_if_hss(handle) != nullptr, "spd_query: HSS query on a non-HSS handle");
            hss_query((const spd_hss_s*)handle, what, buf, bytes);
            return SPD_OK;
        }
        if (what == SPD_Q_SYM_STORE) {
            SPD_REQUIRE(!hss_if_hss(handle), "spd_query: SPD_Q_SYM_STORE needs an H2 handle");
            const spd_h2_s* h2 = (const spd_h2_s*)handle;
            const int64_t v[2] = {(int64_t)h2->sym.bytes, (int64_t)h2->sym.npieces};
            need(bytes, sizeof(v));
            std::memcpy(buf, v, sizeof(v));
            return SPD_OK;
        }
        if (what == SPD_Q_COMM_BYTES) {
            SPD_REQUIRE(!hss_if_hss(handle), "spd_query: SPD_Q_COMM_BYTES needs an H2 handle");
            const spd_comm_s* c = ((const spd_h2_s*)handle)->comm;
            const int64_t v[2] = {c ? c->bytes_in : 0, c ? c->ncoll : 0};
            need(bytes, sizeof(v));
            std::memcpy(buf, v, sizeof(v));
            return SPD_OK;
        }
        if (what == SPD_Q_SHARD_WORK) {
            const spd_hss_s* H = hss_if_hss(handle);
            const int64_t* sw = H ? hss_shard_work(H) : ((const spd_h2_s*)handle)->shard_work;
            need(bytes, 2 * sizeof(int64_t));
            std::memcpy(buf, sw, 2 * sizeof(int64_t));
            return SPD_OK;
        }
        if (what == SPD_Q_TIMINGS) {
            // handle may be either kind: the first field tells (magic)
            const spd_hss_s* H = hss_if_hss(handle);
            const double* tm = H ? hss_timings(H) : ((const spd_h2_s*)handle)->timings;
            need(bytes, 16 * sizeof(double));
            std::memcpy(buf, tm, 16 * sizeof(double));
            return SPD_OK;
        }
        SPD_REQUIRE(hss_if_hss(handle) == nullptr, "spd_query: H2 query on an HSS handle");
        const spd_h2_s* h = (const spd_h2_s*)handle;
        SPD_REQUIRE(h->magic == 0x48324832u, "spd_query: not an H2 handle");
        const TreeH& t = h->tree;
        switch (what) {
        case SPD_Q_N: { int64_t v = h->N; std::memcpy(buf, &v, need(bytes, 8)); break; }
        case SPD_Q_LEVELS: { int32_t v = t.L; std::memcpy(buf, &v, need(bytes, 4)); break; }
        case SPD_Q_NNODES: { int32_t v = t.nnodes; std::memcpy(buf, &v, need(bytes, 4)); break; }
        case SPD_Q_PERM: std::memcpy(buf, t.perm.data(), need(bytes, 8 * t.perm.size())); break;
        case SPD_Q_NODES: {
            std::vector<int64_t> v;
            for (int i = 0; i < t.nnodes; ++i) { v.push_back(t.begin[i]); v.push_back(t.end[i]); }
            std::memcpy(buf, v.data(), need(bytes, 8 * v.size()));
            break;
        }
        case SPD_Q_BOXES: {
            std::vector<double> v;
            for (int i = 0; i < t.nnodes; ++i) {
                for (int a = 0; a < t.d; ++a) v.push_back(t.lo[(size_t)i * t.d + a]);
                for (int a = 0; a < t.d; ++a) v.push_back(t.hi[(size_t)i * t.d + a]);
            }
            std::memcpy(buf, v.data(), need(bytes, 8 * v.size()));
            break;
        }
        case SPD_Q_H2_RANKS: {
            std::vector<int32_t> v(t.nnodes, 0);
            for (int k = 1; k < t.L; ++k)
                for (int a = 0; a < h->lv[k].count; ++a) v[h->lv[k].first + a] = h->lv[k].rank[a];
            std::memcpy(buf, v.data(), need(bytes, 4 * v.size()));
            break;
        }
        case SPD_Q_SKELETONS: {
            std::vector<int64_t> v;
            for (int i = 0; i < t.nnodes; ++i) {
                int k = t.level(i);
                if (k >= t.L) continue;
                const H2Level& lv = h->lv[k];
                int a = i - lv.first;
                if (lv.rank[a] == 0) continue;
                std::vector<int> tmp(lv.rank[a]);
                SPD_CUDA(cudaMemcpy(tmp.data(), lv.skel.p + lv.off[a], 4 * tmp.size(), cudaMemcpyDeviceToHost));
                for (int x : tmp) v.push_back(x);
            }
            std::memcpy(buf, v.data(), need(bytes, 8 * v.size()));
            break;
        }
        case SPD_Q_LIST_COUNTS: {
            std::vector<int64_t> v{(int64_t)h->lists.near.size()};
            for (int k = 1; k <= t.L; ++k) v.push_back((int64_t)h->lists.type1[k].size());
            for (int k = 1; k <= t.L; ++k) v.push_back((int64_t)h->lists.type3[k].size());
            std::memcpy(buf, v.data(), need(bytes, 8 * v.size()));
            break;
        }
        case SPD_Q_NEAR: {
            std::vector<int32_t> v;
            for (auto& p : h->lists.near) { v.push_back(p.first); v.push_back(p.second); }
            std::memcpy(buf, v.data(), need(bytes, 4 * v.size()));
            break;
        }
        case SPD_Q_TYPE3:
        case SPD_Q_TYPE1: {
            std::vector<int32_t> v;
            for (int k = 1; k <= t.L; ++k)
                for (auto& p : (what == SPD_Q_TYPE3 ? h->lists.type3[k] : h->lists.type1[k])) {
                    v.push_back(k); v.push_back(p.first); v.push_back(p.second);
                }
            std::memcpy(buf, v.data(), need(bytes, 4 * v.size()));
            break;
        }
        default: throw Error(SPD_EINVAL, "spd_query: unknown query " + std::to_string(what));
        }
    })
}

// ------------------------------------------------------------------ testing entry points
spd_status spd_test_gemm(int transA, int transB, int m, int n, int k, double alpha, const double* A, int lda,
                         const double* B, int ldb, double beta, double* C, int ldc, void* stream) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        std::vector<GemmDesc> d{{A, B, C, m, n, k, lda, ldb, ldc}};
        gemm_batched((cudaStream_t)stream, d, transA != 0, transB != 0, alpha, beta);
        SPD_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    })
}

spd_status spd_test_potrf(double* A, int n, int lda, int* info_host, void* stream) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        cudaStream_t s = (cudaStream_t)stream;
        DBuf<int> info(1);
        DBuf<double> bad(1);
        info.zero(s);
        potrf_batched(s, {{A, n, n, lda}}, info.p, bad.p);
        *info_host = info.download(s)[0];
    })
}

spd_status spd_test_trsm(char uplo, int trans, const double* T, int n, int ldt, double* X, int nrhs, int ldx,
                         void* stream) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        trsm_batched((cudaStream_t)stream, {{T, X, n, nrhs, ldt, ldx}}, uplo, trans != 0);
        SPD_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    })
}

spd_status spd_test_qrcp(int batch, double* A, int m, int n, int ld, int64_t stride, int max_rank,
                         double rel_tol, int* piv, int* rank, double* Q, int64_t qstride, void* stream) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        cudaStream_t s = (cudaStream_t)stream;
        DBuf<double> beta((size_t)batch * std::max(1, std::min(m, n)));
        DBuf<double> norms((size_t)batch * std::max(1, n));
        std::vector<QrcpDesc> d;
        for (int b = 0; b < batch; ++b)
            d.push_back({A + b * stride, m, n, ld, max_rank, piv + (size_t)b * n,
                         beta.p + (size_t)b * std::max(1, std::min(m, n)), rank + b, norms.p + (size_t)b * std::max(1, n)});
        qrcp_batched(s, d, rel_tol);
        if (Q) {
            std::vector<FormQDesc> f;
            for (int b = 0; b < batch; ++b)
                f.push_back({A + b * stride, d[b].beta, rank + b, Q + b * qstride, m, n, ld, m});
            formq_batched(s, f);
        }
        SPD_CUDA(cudaStreamSynchronize(s));
    })
}

spd_status spd_test_qr_unpivoted(int batch, double* A, int m, int n, int ld, int64_t stride, void* stream) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        std::vector<QrDesc> d;
        for (int b = 0; b < batch; ++b) d.push_back({A + b * stride, m, n, ld});
        qr_unpivoted_batched((cudaStream_t)stream, d);
    })
}

spd_status spd_test_proxies(spd_h2_t h, int node, double* P_host, void* stream) {
    SPD_TRY({
        AllocStreamScope alloc_scope_((cudaStream_t)stream);
        SPD_REQUIRE(h != nullptr && P_host != nullptr, "spd_test_proxies: null argument");
        cudaStream_t s = (cudaStream_t)stream;
        const int64_t np = (int64_t)h->m * h->n_proxy;     // proxy dofs (RPY: 3 per proxy point)
        DBuf<double> P((size_t)np * h->d);
        proxies_for_node(h, node, P.p, s);
        std::vector<double> v = P.download(s);
        for (int p = 0; p < h->n_proxy; ++p)                // the proxy points (first dof of each)
            for (int a = 0; a < h->dim; ++a) P_host[(size_t)p * h->dim + a] = v[(size_t)a * np + (size_t)h->m * p];
    })
}

spd_status spd_test_tree_host(const double* pts, int64_t n, int d, int leaf, int64_t* perm, double* boxes,
                              int64_t* list_counts) {
    SPD_TRY({
        SPD_REQUIRE(pts && perm && boxes && list_counts && n >= 1 && (d == 2 || d == 3) && leaf >= 1,
                    "spd_test_tree_host: bad argument");
        TreeH t;
        ListsH l;
        build_tree(pts, n, d, leaf, t);
        build_lists(t, l);
        std::memcpy(perm, t.perm.data(), sizeof(int64_t) * n);
        for (int i = 0; i < t.nnodes; ++i)
            for (int a = 0; a < d; ++a) {
                boxes[((size_t)i * 2) * d + a] = t.lo[(size_t)i * d + a];
                boxes[((size_t)i * 2 + 1) * d + a] = t.hi[(size_t)i * d + a];
            }
        list_counts[0] = (int64_t)l.near.size();
        for (int k = 1; k <= t.L; ++k) {
            list_counts[k] = (int64_t)l.type1[k].size();
            list_counts[t.L + k] = (int64_t)l.type3[k].size();
        }
    })
}

spd_status spd_test_philox_normal(double* out, int64_t n, int w, uint64_t seed, void* stream) {
    SPD_TRY({
        SPD_REQUIRE(out != nullptr && n >= 0 && w >= 0, "spd_test_philox_normal: bad argument");
        philox_normal((cudaStream_t)stream, out, n, w, seed);
    })
}

}  // extern "C"
