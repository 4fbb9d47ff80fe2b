/* spdhss_testing.h -- internal kernels of libspdhss exported for the GPU unit
 * tests only (single-matrix wrappers around the batched device kernels).
 * All pointers are device pointers, column-major.  Not part of the product API. */
#ifndef SPDHSS_TESTING_H
#define SPDHSS_TESTING_H
#include "spdhss.h"
#ifdef __cplusplus
extern "C" {
#endif
/* C = alpha op(A) op(B) + beta C on FP64 DMMA tiles */
spd_status spd_test_gemm(int transA, int transB, int m, int n, int k, double alpha, const double* A, int lda,
                         const double* B, int ldb, double beta, double* C, int ldc, void* stream);
/* in-place lower Cholesky; *info_host = 0 or failing column + 1 */
spd_status spd_test_potrf(double* A, int n, int lda, int* info_host, void* stream);
/* X := op(T)^{-1} X, uplo 'L'/'U' */
spd_status spd_test_trsm(char uplo, int trans, const double* T, int n, int ldt, double* X, int nrhs, int ldx,
                         void* stream);
/* pivoted QR (R4) of `batch` matrices A_b = A + b*stride (m x n, ld); forms Q (m x r) into Q + b*qstride
 * (ld m) when Q != NULL; piv (n per matrix) and rank (1 per matrix) on the device */
spd_status spd_test_qrcp(int batch, double* A, int m, int n, int ld, int64_t stride, int max_rank,
                         double rel_tol, int* piv, int* rank, double* Q, int64_t qstride, void* stream);
/* unpivoted blocked Householder QR (R only) of `batch` matrices A_b = A + b*stride (m x n, ld);
 * on exit the upper triangle of each A_b[:n, :n] holds R with diag(R) >= 0 */
spd_status spd_test_qr_unpivoted(int batch, double* A, int m, int n, int ld, int64_t stride, void* stream);
/* proxy points of heap node `node` of an H2 handle: P host, n_proxy x d row-major
 * (d = spatial dimension; for RPY the points, not their 3 dofs each) */
spd_status spd_test_proxies(spd_h2_t h, int node, double* P_host, void* stream);
/* the HOST tree / list builder (tree.cpp, kept for leaves beyond the device sort) on host
 * points: perm[n] (tree position -> original index), boxes[nnodes * 2 * d] (lo, hi per
 * node) and list_counts[1 + 2L] (near pairs, then type1[k], type3[k] for k = 1..L), the
 * layouts of SPD_Q_PERM / SPD_Q_BOXES / SPD_Q_LIST_COUNTS -- to check the device builder */
spd_status spd_test_tree_host(const double* pts, int64_t n, int d, int leaf, int64_t* perm, double* boxes,
                              int64_t* list_counts);
/* the device Omega generator of spdhss_build (Philox4x32-10 + Box-Muller, reading R29):
 * out (device) n x w column-major, ld n, tree-order element e = row + col n */
spd_status spd_test_philox_normal(double* out, int64_t n, int w, uint64_t seed, void* stream);
/* subtree-sharding plan (host logic only, no GPU): owner rank of node a of a level
 * with `count` nodes for nranks ranks, -1 when the level is computed redundantly */
int spd_test_shard_owner(int nranks, int count, int a);
#ifdef __cplusplus
}
#endif
#endif
