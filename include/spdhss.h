/* spdhss.h -- C ABI of the B200-native SPD-HSS-from-H2 library (libspdhss.so).
 *
 * Method: arXiv 2011.07632, "quasilinear construction of an SPD HSS
 * approximation driven by an H2 representation".  Every numeric step of the
 * entry points below runs in hand-written fp64 CUDA kernels for sm_100a.
 *
 * Conventions:
 *  - All numerics are fp64.  Array arguments are DEVICE pointers on the
 *    current device unless marked "host".  Multi-vectors are column-major
 *    with a leading dimension (ld >= n).  Points are row-major n x d.
 *  - Vectors at the boundary are in the caller's ORIGINAL point order when
 *    layout == SPD_LAYOUT_ORIGINAL, or in the library's tree order when
 *    layout == SPD_LAYOUT_TREE (see spd_query(SPD_Q_PERM)).
 *  - Ownership: the caller owns every buffer it passes; the library copies
 *    what it keeps.  Handles own their device memory and are released by the
 *    *_free calls.  An spd_hss_t references its spd_h2_t: free it first.
 *  - Streams: all work is enqueued on the given stream (0 = legacy default).
 *    Builds synchronize the stream internally (ranks decide allocations);
 *    h2_matvec and hss_solve do not synchronize the host.
 *  - Errors: every call returns an spd_status; spd_last_error() returns a
 *    thread-local message (for SPD_ENOTPD it names level, node and the failed
 *    pivot).  Rank deficiency is never an error: ranks shrink, down to 0.
 */
#ifndef SPDHSS_H
#define SPDHSS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPD_OK = 0,
    SPD_EINVAL = 1,   /* invalid argument / dimension mismatch */
    SPD_ENOTPD = 2,   /* leaf Cholesky failed or I + B_ii not SPD */
    SPD_ENOMEM = 3,   /* device allocation failed */
    SPD_ECUDA = 4,    /* CUDA runtime error */
    SPD_ENCCL = 5,    /* collective error (multi-GPU) */
    SPD_ENOCONV = 6   /* PCG reached maxit; report filled; not fatal */
} spd_status;

/* Kernel functions K(r), r = |x - y|_2 (BASELINE.json forms, reading R13;
 * PAPER.md §6 P:1073-1077 for the families).  shift sigma is added only on
 * exact diagonal entries. */
typedef enum {
    SPD_K_GAUSSIAN = 0,     /* exp(-r^2 / l^2)                       */
    SPD_K_MATERN32 = 1,     /* (1 + sqrt3 r / l) exp(-sqrt3 r / l)   */
    SPD_K_EXPONENTIAL = 2,  /* exp(-r / l)                           */
    SPD_K_IMQ = 3,          /* 1 / sqrt(r^2 + l^2)                   */
    SPD_K_RPY = 4           /* Rotne-Prager-Yamakawa 3x3 tensor, l = particle radius a
                               (reading R28); points in 3D only.  The
                               operator is over 3n DEGREES OF FREEDOM: dof 3p + c is
                               component c of point p, so every vector / matrix
                               argument of the H2 / HSS / PCG calls has 3n rows  */
} spd_kernel_id;

typedef struct { int id; double l; double shift; } spd_kernel;

typedef enum { SPD_LAYOUT_ORIGINAL = 0, SPD_LAYOUT_TREE = 1 } spd_layout;

typedef struct {
    int n_proxy;        /* proxy points per node; 0 = 4096 (2D) / 6144 (3D) (reading R3) */
    int reserved;
    /* Parity hook of the certified-tie protocol (reading R19):
     * host, nullable.  For every heap node at levels 1..L-1 in heap order: s_i, then the
     * s_i skeleton TREE POSITIONS in pivot order (s_i = 0 for inactive nodes).  The ID
     * QRCP of each node then takes these pivots instead of its own (Alg. 2 step 3,
     * P:827) and stops after s_i steps, so later stages can be compared with another
     * implementation's (the oracle's) skeletons.  Read during h2_build only.
     * SPD_EINVAL if a count or position does not fit the tree and the candidates. */
    const int32_t* inject_skeletons;
} spd_h2_opts;

typedef struct spd_comm_s* spd_comm_t;
typedef struct spd_h2_s* spd_h2_t;
typedef struct spd_hss_s* spd_hss_t;

typedef struct {
    int iters;               /* H2 matvecs performed                      */
    int converged;           /* 1 if ||r_k|| <= tol ||b||                 */
    double relres;           /* recursively updated relative residual     */
    double seconds;          /* wall time of the solve (host clock)       */
    double relres_true;      /* ||b - A x|| / ||b|| with the H2 operator, after the last iteration */
} spd_pcg_report;

/* Communicator for multi-GPU runs (NCCL over NVLink/NVSwitch,
 * loaded at run time from libnccl.so.2).  One process per GPU; every rank calls
 * with identical global arguments and the points replicated.
 *   spd_comm_unique_id: rank 0 creates the 128-byte NCCL id (host buffer) and
 *                       shares it (e.g. torch.distributed.broadcast_object_list).
 *   spd_comm_init:      nranks a power of 2; id NULL with nranks == 1 (single
 *                       GPU) or nranks > 1 (a "virtual" communicator: the sharded
 *                       code path emulated in one process on one GPU -- tests).
 * Sharding (h2_build): rank p computes the nodes of subtree p at every level with
 * >= nranks nodes (p count/P .. (p+1) count/P - 1), levels with fewer nodes are
 * computed redundantly; after each sharded level the owners' contiguous ranges of
 * the level arrays are broadcast (ncclBroadcast group = an all-gather of variable
 * size) and the ranks all-reduced, so every rank ends with the full H2.  The
 * caller owns the communicator; handles keep a reference (free them first).
 * Errors: SPD_EINVAL (bad nranks / rank), SPD_ENCCL (library or NCCL failure). */
spd_status spd_comm_unique_id(void* nccl_unique_id_out);
spd_status spd_comm_init(const void* nccl_unique_id, int nranks, int rank, spd_comm_t* out);

/* Host-staged collectives: the same sharded path with every exchange routed through
 * caller callbacks on host buffers (the library drains the stream, copies the device
 * buffer to pageable host memory, calls, copies back).  For transports without NCCL
 * (e.g. torch.distributed over gloo) and for multi-process tests of the sharded path;
 * slow by construction.  Callbacks return 0 on success (else SPD_ENCCL), operate in
 * place, and are called by every rank in the same order:
 *   allreduce_sum_f64 / _i32: buf[0..n) = sum over ranks
 *   broadcast:                buf[0..bytes) = root's buf
 * ops is copied; ctx is passed back untouched and must outlive the communicator. */
typedef struct {
    void* ctx;
    int (*allreduce_sum_f64)(void* ctx, double* buf, size_t n);
    int (*allreduce_sum_i32)(void* ctx, int* buf, size_t n);
    int (*broadcast)(void* ctx, void* buf, size_t bytes, int root);
} spd_host_coll;
spd_status spd_comm_init_host(const spd_host_coll* ops, int nranks, int rank, spd_comm_t* out);
void spd_comm_free(spd_comm_t c);

/* h2_build: H2 representation of A = K(X, X) + shift I.
 *   pts   device, n x d row-major (original order), d in {2, 3}
 *   leaf  maximum leaf size; tree depth ceil(log2(n / leaf)) (reading R1)
 *   tol   relative tolerance of the proxy-point IDs (reading R4), e.g. 1e-10
 * Builds the KD tree, the Type-1/Type-3 lists (PAPER.md P:657-663, P:891-913,
 * reading R2), the proxy points (R3) and the nested interpolative bases by
 * QRCP (R4).  Near blocks and B^{H2}_ij = K(X_Ji, X_Jj) are never stored: they
 * are evaluated on the fly (north star).  opts may be NULL. */
spd_status h2_build(const double* pts, int64_t n, int d, spd_kernel k, int leaf, double tol,
                    const spd_h2_opts* opts, spd_comm_t c, void* stream, spd_h2_t* out);

/* h2_matvec: Y = A X (A = the H2 matrix incl. shift), X and Y n x k
 * (column-major, ldx, ldy >= n) in the given layout.  Near field on the fly,
 * up pass (U^T), Type-3 coupling on the fly, down pass (U)  (eqn:nested). */
spd_status h2_matvec(spd_h2_t h, int layout, const double* X, int64_t ldx, double* Y,
                     int64_t ldy, int64_t k, void* stream);

/* spdhss_build: Alg. 4 of PAPER.md (alg:spdhss_h2).
 *   rank_cap, rel_tol   HSS rank rule: r_i = min(cap, first t with |R_tt| <= tol |R_00|) (R4, R5)
 *   oversample          p; sketch width w = rank_cap + p
 *   seed                Philox seed for Omega when omega == NULL
 *   omega               optional device N x w column-major (ld = n) Gaussian sketch in TREE
 *                       order (parity hook); one Omega serves every level (reading R8)
 * The nonleaf factorization uses Cholesky of I + B_ii (reading R9, identical R_i, B_ij).
 * Fails with SPD_ENOTPD if a leaf block or some I + B_ii is not SPD (R18). */
spd_status spdhss_build(spd_h2_t h, int rank_cap, double rel_tol, int oversample, uint64_t seed,
                        const double* omega, void* stream, spd_hss_t* out);

/* spdhss_build_adaptive: the threshold-driven variant sketched in PAPER.md P:998-999
 * ("adaptively adding more vectors to Omega and compressing Lambda_{ii^c} Omega_{i^c}
 * with this error threshold"), in restart form (reading R27): builds with rank cap
 * r0, 2 r0, 4 r0, ... (<= r_max) until every node's rank stops on the threshold
 * |R_tt| <= rel_tol |R_00| below the cap.  Omega = the leading cap + oversample
 * columns of one sketch: Philox(seed), or omega (device, N x (r_max + oversample),
 * ld = N, tree order).  *cap_out (host, nullable) = the cap used. */
spd_status spdhss_build_adaptive(spd_h2_t h, int r0, int r_max, double rel_tol, int oversample, uint64_t seed,
                                 const double* omega, void* stream, spd_hss_t* out, int* cap_out);

/* hss_solve: X = H^{-1} B for the SPD HSS H, by the recursive solve of reading
 * R12 (the "ULV-style" solve of PAPER.md P:1119-1123), nrhs columns. */
spd_status hss_solve(spd_hss_t H, int layout, const double* B, int64_t ldb, double* X,
                     int64_t ldx, int64_t nrhs, void* stream);

/* hss_matvec: Y = H X with the SPD-HSS matrix itself (the nested representation of
 * Alg. 4: leaf D_i = A_ii, U_i = S_i V_i, transfers R_i, sibling couplings B),
 * e.g. for the paper's approximation error ||H x - A x|| / ||A x|| (Fig. 5).
 *   X, Y  device, n x k column-major (ld >= n), layout as for hss_solve; Y overwritten.
 * Errors: SPD_EINVAL (bad layout / ld / null), SPD_ECUDA. */
spd_status hss_matvec(spd_hss_t H, int layout, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t k,
                      void* stream);

/* pcg_solve: (K + shift I) x = b by PCG with H2 matvecs, preconditioner
 * M = the SPD HSS (hss_solve) or none (M == NULL).  x holds x0 = 0 on output the
 * solution.  Stops when ||r_k|| <= tol ||b|| (recursive residual, R15) or at maxit
 * (returns SPD_ENOCONV with the report filled).  rep is a host pointer. */
spd_status pcg_solve(spd_h2_t A, spd_hss_t M, int layout, const double* b, double* x,
                     double tol, int maxit, spd_pcg_report* rep, void* stream);

/* pcg_solve_bj: the same PCG with the block-Jacobi preconditioner built from M's leaf
 * Cholesky factors, x_i = A_ii^{-1} b_i (the paper's BJ baseline, P:1216,
 * SPD-HSS "combines a BJ preconditioner with off-diagonal
 * approximations").  M must not be NULL (SPD_EINVAL). */
spd_status pcg_solve_bj(spd_h2_t A, spd_hss_t M, int layout, const double* b, double* x, double tol, int maxit,
                        spd_pcg_report* rep, void* stream);

/* Introspection (host buffers).  `what` selects:                            */
enum {
    SPD_Q_N = 1,            /* int64: n                                       */
    SPD_Q_LEVELS = 2,       /* int32: L                                       */
    SPD_Q_PERM = 3,         /* int64[n]: tree position -> original index     */
    SPD_Q_NODES = 4,        /* int64[nnodes*2]: begin, end per heap node      */
    SPD_Q_BOXES = 5,        /* double[nnodes*2*d]: lo[d], hi[d] per node      */
    SPD_Q_NNODES = 6,       /* int32: number of nodes                         */
    SPD_Q_H2_RANKS = 7,     /* int32[nnodes]: skeleton size s_i (0 inactive)  */
    SPD_Q_SKELETONS = 8,    /* int64[sum s_i]: skeleton tree positions, node order */
    SPD_Q_LIST_COUNTS = 9,  /* int64[1 + 2L]: near pairs, then type1[k], type3[k] k=1..L */
    SPD_Q_NEAR = 10,        /* int32[2 * nnear]: ordered near leaf pairs      */
    SPD_Q_TYPE3 = 11,       /* int32[3 * n3]: (level, i, j) ordered Type-3 pairs */
    SPD_Q_TYPE1 = 12,       /* int32[3 * n1]: (level, i, j) ordered Type-1 pairs */
    SPD_Q_HSS_RANKS = 20,   /* int32[nnodes]: HSS rank r_i (levels 1..L-1)    */
    SPD_Q_HSS_EXPORT_SIZE = 21, /* int64: doubles needed by SPD_Q_HSS_EXPORT */
    SPD_Q_HSS_EXPORT = 22,  /* double[]: leaf D_i (n_i^2), U_i (n_i r_i) per leaf in node
                               order; R_i (m_i r_i) per nonleaf at levels 2..L-1; then the
                               sibling B_{c1 c2} (r_c1 r_c2) for every nonleaf parent
                               in heap order; all column-major                   */
    SPD_Q_HSS_PIVOTS = 23,  /* int32[sum w]: QRCP pivots of every node (w each) */
    SPD_Q_TIMINGS = 30,     /* double[16]: phase seconds of the last build      */
    SPD_Q_SHARD_WORK = 31,  /* int64[2]: nodes whose per-node work (H2: proxy ID; HSS:
                               factorisation, QRCP, bases) this process computed, and
                               the number of such nodes; equal unless sharded (§8(e)) */
    SPD_Q_SYM_STORE = 32,   /* int64[2] (H2 handle): bytes of stored symmetric blocks on this
                               process and their number of pieces (0 before the first k = 1
                               product / PCG, or before the first multi-vector product when
                               the store fits SPD_STORE_FRAC = 0.25 of the free memory, and
                               after h2_release_store); sharded: the blocks touching owned nodes */
    SPD_Q_COMM_BYTES = 33   /* int64[2] (H2 handle): bytes this process has received through the
                               library's collectives on the handle's communicator so far (broadcast
                               ranges of the other ranks, all-reduced buffers) and the number of
                               collective calls; 0 without a real communicator (§8(e) evidence) */
};
spd_status spd_query(const void* handle, int what, void* host_buf, size_t bytes);

/* Instrumentation (bench.py): number of library kernel launches so far, and an
 * optional per-kernel-class timer (CUDA events recorded on the launching stream
 * around every launch; flops/bytes are the ALGORITHMIC counts of each launch). */
long long spd_launch_count(void);
void spd_prof_enable(int on);
void spd_prof_reset(void);
int spd_prof_count(void);
/* out4 = {launches, total ms, total flops, total bytes}; returns 0 if idx valid */
int spd_prof_get(int idx, char* name, int name_len, double* out4);

/* h2_release_store: free the stored symmetric kernel blocks of h (built by the first
 * k = 1 product / PCG within 40 % of the free memory, or on demand for multi-vector
 * products within SPD_STORE_FRAC = 0.25 of it); products evaluate the blocks on the fly
 * again until a later k = 1 product rebuilds it.  Synchronizes the device.
 * SPD_EINVAL on a null handle. */
spd_status h2_release_store(spd_h2_t h);
void h2_free(spd_h2_t h);
void hss_free(spd_hss_t H);
const char* spd_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SPDHSS_H */
