// comm.hpp -- communicator of libspdhss (NCCL, loaded at run time; comm.cpp).
#pragma once
#include <vector>
#include "common.cuh"

struct spd_comm_s {
    int nranks = 1, rank = 0;
    bool virt = false;          // single-process emulation of nranks ranks (tests)
    void* nccl = nullptr;       // ncclComm_t
    bool hosted = false;        // host-staged collectives through caller callbacks
    spd_host_coll host{};
    // bytes this process received through the library's collectives (broadcast ranges of
    // the other ranks, all-reduced buffers): exchange-volume evidence (SPD_Q_COMM_BYTES)
    mutable int64_t bytes_in = 0;
    mutable int64_t ncoll = 0;
};

namespace spd {

struct Nccl128 { char b[128]; };   // ncclUniqueId

void comm_unique_id(void* out128);
spd_comm_s* comm_create(const void* id, int nranks, int rank);
spd_comm_s* comm_create_host(const spd_host_coll* ops, int nranks, int rank);
// true when collectives really move data (NCCL or host-staged), i.e. the sharded path runs
inline bool comm_real(const spd_comm_s* c) { return c && c->nranks > 1 && !c->virt; }
void comm_destroy(spd_comm_s* c);
// owner rank of node a (0 <= a < count) of a level, -1 when the level is redundant
int shard_owner(const spd_comm_s* c, int count, int a);
// every rank q broadcasts elements [begin[q], end[q]) of buf (elem bytes each), in one group
void comm_bcast_ranges(const spd_comm_s* c, void* buf, size_t elem, const std::vector<int64_t>& begin,
                       const std::vector<int64_t>& end, cudaStream_t s);
// column-major rows: every rank q broadcasts rows [begin[q], end[q]) of all ncols columns
void comm_bcast_rows(const spd_comm_s* c, double* buf, int64_t ld, int ncols, const std::vector<int64_t>& begin,
                     const std::vector<int64_t>& end, cudaStream_t s);
void comm_allreduce_sum(const spd_comm_s* c, double* buf, size_t n, cudaStream_t s);
void comm_allreduce_sum(const spd_comm_s* c, int* buf, size_t n, cudaStream_t s);

}  // namespace spd
