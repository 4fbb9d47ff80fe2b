// kblock.cuh -- on-the-fly kernel block x multi-vector interface.
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace spd {

struct KbBlock {            // a point set: coordinate a of point p at x[a * ds + p]
    const double* x;
    int64_t ds;
    int n;
    int64_t id0;            // global id of point 0 (ids contiguous); -1: no ids (no shift)
};
struct KbEntry {            // Y[:, :ncols] += K(target, blocks[src]) X[:, :ncols]
    int src;
    const double* X; int ldx;
    double* Y; int ldy;
    int ncols;
    // optional: the block is read from the symmetric k = 1 store (h2sym.cu) instead of
    // being evaluated: kmode 1 -- stored as (target, src), entry (r, c) at
    // kst[(r / 32) 32 kld + 32 c + r % 32], kld = n_src; kmode 2 -- stored as (src, target),
    // entry (r, c) at kst[(c / 32) 32 kld + 32 r + c % 32], kld = n_target.  Stored
    // values include the diagonal shift.
    const double* kst = nullptr;
    int kmode = 0, kld = 0;
    // set by kblock_plan: X staged by TMA through tensor map tmi of the plan (row coordinate
    // tr of X's first row); -1: X read by plain loads
    int tmi = -1, tr = 0;
};
// TMA tensor maps of one planned product: one 2-D map (rows x columns, 16 x NC boxes,
// 128-byte swizzle) per X buffer the entries read
constexpr int KB_NTMA = 16;
struct KbTma { CUtensorMap map[KB_NTMA]; unsigned box_bytes[KB_NTMA]; };
struct KbTarget { int blk; int e_begin, e_end; };

// entries of a target must be contiguous; consecutive entries with the same Y
// accumulate in registers before one read-modify-write of Y.
void kblock_apply(cudaStream_t s, const KernelParams& kp, double shift, int d,
                  const std::vector<KbBlock>& blocks, const std::vector<KbTarget>& targets,
                  const std::vector<KbEntry>& entries);

// the device-side plan of one multi-column (ncols > 4) kblock product: descriptor arrays,
// the balanced work list and the split-target partial slots; built once and replayed
// (h2_matvec keeps the plan of its last product in the handle: repeated products of the
// same width on the same buffers skip the host-side planning and the uploads)
struct KbWork;
struct KbRed;
struct KbPlan {
    bool ok = false;
    int NC = 0, nwork = 0, nred = 0;
    int ntma = 0;             // tensor maps in use (0: the register-prefetch kernel)
    bool tma_mix = false;     // some entries without a map (their X slices prefetched through registers)
    KbTma tma;
    double fl = 0, by = 0;
    DBuf<KbBlock> b;
    DBuf<KbTarget> t;
    DBuf<KbEntry> e;
    DBuf<char> w, r;          // KbWork / KbRed arrays (types private to kblock.cu)
    DBuf<double> partial;
};
// false: the product is empty or narrow (ncols <= 4: the vector kernel, not planned)
bool kblock_plan(cudaStream_t s, const std::vector<KbBlock>& blocks, const std::vector<KbTarget>& targets,
                 const std::vector<KbEntry>& entries, KbPlan& plan);
void kblock_run(cudaStream_t s, const KernelParams& kp, double shift, int d, const KbPlan& plan);

}  // namespace spd
