// h2.hpp -- H2 handle (internal).  PAPER.md §5.1.
#pragma once
#include "common.cuh"
#include <unordered_map>
#include "kblock.cuh"
#include "tree.hpp"

namespace spd {

struct H2Level {
    int k = 0, first = 0, count = 0;
    std::vector<int> rank;        // s_i per node of the level (0 when inactive)
    std::vector<int> ncand;       // candidates n_c per node
    std::vector<int64_t> off;     // row offset of node i in the level's coefficient space
    int64_t S = 0;                // sum of ranks
    int64_t Sw = 0;               // leading dimension of the multi-column x^ / y^ workspaces: S rounded
                                  // up to a multiple of 8 (16-byte aligned columns for TMA, kblock.cu)
    DBuf<int> skel;               // S skeleton tree positions
    DBuf<double> skelX;           // d x S skeleton coordinates (SoA, stride S)
    std::vector<int64_t> E_off;   // offset of E_i (n_c x s_i, col-major) in E
    DBuf<double> E;               // leaf U_i / nonleaf R_i (interpolation matrices)
    // the same interpolation matrices in ID form: E_i[piv[k], k] = 1 (k < s_i),
    // E_i[piv[s_i + c], k] = T_i[k, c]; T_i is s_i x (n_c - s_i), col-major
    std::vector<int64_t> T_off, piv_off;
    DBuf<double> T;
    DBuf<int> piv;                // n_c pivots per node (QRCP column order of the candidates)
};

struct Timer;

// symmetric stored blocks for k = 1 products (h2sym.cu)
constexpr int SYM_MAX_SLOTS = 32;
struct SymBuild { const double* tx; const double* sx; int64_t tds, sds, tid0, sid0; int nr, nb; int64_t vbase; };
struct SymPiece {            // a band of up to 4 row tiles of a block (rows nr <= 128)
    int64_t vbase, xa_off, xb_off, fwd, trn;   // vbase < 0: evaluated on the fly
    int slot, nr, nb;
    const double* tx; const double* sx; int64_t tds, sds, tid0, sid0;   // row / column points, ids (shift)
};
struct SymGNode { int slot, n; int64_t off; int c0, c1; };   // lists >= SYM_BIG: one CTA
constexpr int SYM_BIG = 48;
struct SymContrib { int64_t soff; int ro, len; };
struct SymVecs { const double* p[SYM_MAX_SLOTS]; };
struct SymVecsOut { double* p[SYM_MAX_SLOTS]; };
struct H2SymStore {
    DBuf<double> vals, scratch;
    DBuf<SymPiece> pieces;
    DBuf<SymGNode> gnodes;
    DBuf<SymContrib> gcon;
    int npieces = 0, ngnodes = 0, nbig = 0;      // gnodes[0, nbig): long lists
    int nbmax = 1;
    std::vector<int> piece_off;                  // pieces of slot l: [piece_off[l], piece_off[l+1])
    std::vector<SymGNode> gnodes_h;              // host copy (per-slot schedules of the persistent PCG)
    double flops = 0, bytes = 0, stored_frac = 1.0;
    bool built = false;
    // fully stored blocks (a <= b) of slot s: sym_key(s, a, b) -> offset in vals of band 0
    // (bands of a block are consecutive), for the multi-vector products (kblock kmode)
    std::unordered_map<uint64_t, int64_t> base;
};
inline uint64_t sym_key(int slot, int a, int b) {
    return ((uint64_t)slot << 56) | ((uint64_t)(uint32_t)a << 28) | (uint64_t)(uint32_t)b;
}

}  // namespace spd

struct spd_h2_s {
    uint32_t magic = 0x48324832u;   // 'H2H2'
    spd::TreeH tree;
    spd::ListsH lists;
    std::vector<char> active;
    spd_kernel kern{};
    spd::KernelParams kp{};
    double tol = 0.0;
    int n_proxy = 0;
    int leaf = 0;
    int d = 0;
    int64_t N = 0;
    spd::DBuf<double> X;          // d x N tree-order points (SoA)
    spd::DBuf<int64_t> perm;      // tree position -> original index
    std::vector<spd::H2Level> lv; // [0..L-1], level k at lv[k] (lv[0] unused)
    double sym_need = -1.0;          // bytes of the full symmetric store (cached plan size)
    int m = 1, dim = 3;              // dofs per point (RPY: 3), spatial dimension; N = m * points,
                                     // d = coordinate rows of X (RPY: dim + 1, the component)
    double timings[16] = {0};
    int64_t shard_work[2] = {0, 0};  // nodes ID'd by this process / nodes with an ID (sharding evidence)
    // matvec workspace
    int64_t ws_k = 0;
    spd::DBuf<double> xt, yt;
    std::vector<spd::DBuf<double>> xh, yh;
    spd_comm_t comm = nullptr;
    const int32_t* inject = nullptr;   // spd_h2_opts.inject_skeletons during h2_build only (host)
    // symmetric k = 1 product (near field + Type-3 couplings, h2sym.cu): blocks stored
    // up to sym_budget bytes, the rest evaluated on the fly
    int stored_mode = -1;          // -1 undecided, 0 old per-level path (tests), 1 symmetric
    double sym_budget = 0.0;
    double sym_frac = 1.0;         // fraction of the blocks to store (rest: evaluated, overlapping HBM and FP64)
    spd::H2SymStore sym;
    // plan of the last multi-column product (kblock.cuh KbPlan), replayed while the width,
    // the buffers, the sharding and the block store are unchanged
    struct KbCache {
        bool valid = false;
        int k = 0;
        const double* x = nullptr; double* y = nullptr;
        int64_t ldx = 0, ldy = 0;
        bool stored = false, shard = false;
        const double* store = nullptr;
        const double* xh1 = nullptr;   // the coefficient workspace the plan points into
        spd::KbPlan plan;
    } kbc;
};

namespace spd {
// y = A x in tree order (x, y: N x k, ld >= N); y is overwritten.  shard (real
// communicator): near and coupling work only for the owned subtrees, then the owners'
// rows of y are broadcast (x replicated; up/down passes redundant)
void h2_apply_tree(spd_h2_s* h, const double* x, int64_t ldx, double* y, int64_t ldy, int k,
                   cudaStream_t s, bool shard = false);
// gather/scatter between original and tree order
void permute_rows(cudaStream_t s, const int64_t* perm, int64_t N, int k, const double* src, int64_t lds,
                  double* dst, int64_t ldd, bool to_tree);
void h2_build_impl(spd_h2_s* h, const double* pts_dev, cudaStream_t s);
void h2_prepare(spd_h2_s* h, int k, cudaStream_t s);   // allocate matvec workspace for width k
void h2_perm_ws(spd_h2_s* h, int k, double** xt, double** yt);   // N x k permutation buffers (handle-owned)
// which nodes a basis pass covers: levels [lo, hi], and at levels with >= P nodes only
// those of subtree `rank` (the sharded product; P = 1: every node)
struct BasisFilter {
    int lo = 1, hi = 1 << 30, P = 1, rank = 0;
    bool keep(int level, int count, int a) const {
        if (level < lo || level > hi) return false;
        return P <= 1 || count < P || a / (count / P) == rank;
    }
};
void h2_up(const spd_h2_s* h, const double* x, int64_t ldx, int k, const std::vector<double*>& xh, int top,
           cudaStream_t s, const BasisFilter* f = nullptr);
void h2_down(const spd_h2_s* h, const std::vector<double*>& yh, int top, double* y, int64_t ldy, int k,
             cudaStream_t s, const BasisFilter* f = nullptr);
// k = 1 basis passes in interpolative form (h2basis.cu)
void h2_up_vec(const spd_h2_s* h, const double* x, const std::vector<double*>& xh, int top, cudaStream_t s,
               const BasisFilter* f = nullptr);
void h2_down_vec(const spd_h2_s* h, const std::vector<double*>& yh, int top, double* y, cudaStream_t s,
                 const BasisFilter* f = nullptr);
size_t h2sym_bytes(const spd_h2_s* h);
void h2sym_build(spd_h2_s* h, double budget_bytes, cudaStream_t s);
// kernel blocks of multi-vector products from the symmetric store (built on demand when
// the k = 1 policy stores blocks); h2_use_store marks entry e of block (a, b) of slot
// `slot` (0: leaves, l: level-l skeletons; na, nb their sizes) if the store holds it
bool h2_store_for_products(spd_h2_s* h, cudaStream_t s, bool build = true);
void h2_use_store(const spd_h2_s* h, int slot, int a, int b, int na, int nb, KbEntry& e);
void h2sym_apply(spd_h2_s* h, const double* x, double* y, const std::vector<double*>& xh,
                 const std::vector<double*>& yh, cudaStream_t s);
// proxy points of heap node `node` into P_dev (d x n_proxy SoA)
void proxies_for_node(spd_h2_s* h, int node, double* P_dev, cudaStream_t s);
}  // namespace spd
