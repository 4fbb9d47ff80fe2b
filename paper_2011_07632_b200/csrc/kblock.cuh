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
};
struct KbTarget { int blk; int e_begin, e_end; };

// Stored kernel blocks for repeated single-vector products (PCG):
// the first k=1 apply through a store evaluates K once into a 32-row-tile layout,
// later k=1 applies stream it (HBM-bound GEMV instead of evaluation-bound).
struct KbStore {
    DBuf<double> vals;
    bool built = false;
};
// bytes a store would need for this list structure
size_t kblock_store_bytes(const std::vector<KbBlock>& blocks, const std::vector<KbTarget>& targets,
                          const std::vector<KbEntry>& entries);

// entries of a target must be contiguous; consecutive entries with the same Y
// accumulate in registers before one read-modify-write of Y.
void kblock_apply(cudaStream_t s, const KernelParams& kp, double shift, int d,
                  const std::vector<KbBlock>& blocks, const std::vector<KbTarget>& targets,
                  const std::vector<KbEntry>& entries, KbStore* store = nullptr);

}  // namespace spd
