// kblock.cuh -- on-the-fly kernel block x multi-vector interface.
#pragma once
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
};
struct KbTarget { int blk; int e_begin, e_end; };

// entries of a target must be contiguous; consecutive entries with the same Y
// accumulate in registers before one read-modify-write of Y.
void kblock_apply(cudaStream_t s, const KernelParams& kp, double shift, int d,
                  const std::vector<KbBlock>& blocks, const std::vector<KbTarget>& targets,
                  const std::vector<KbEntry>& entries);

}  // namespace spd
