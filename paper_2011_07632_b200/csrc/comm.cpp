// comm.cpp -- the library's communicator: NCCL over NVLink /
// NVSwitch, loaded at run time (dlopen "libnccl.so.2", the copy PyTorch ships is
// already in the process), so single-GPU use has no NCCL dependency.
//
// Subtree sharding plan (shard_owner): at a level with count >= P nodes, rank p owns
// the contiguous node range [p count / P, (p + 1) count / P) -- the nodes of subtree p
// below level L - log2 P, so a rank's nodes are contiguous in every level array and an
// exchange is one broadcast per owner (an all-gather of variable-size ranges).
// Levels with fewer nodes than ranks are computed redundantly by every rank.
//
// A "virtual" communicator (nranks > 1, no NCCL id) runs the sharded code path in a
// single process on one GPU: every virtual rank's share is computed in turn and the
// exchange is the identity.  It exercises the ownership / ordering logic of the
// sharded build against the unsharded one (tests), not the transport.
//
// A "host-staged" communicator (spd_comm_init_host) runs every collective through
// caller-supplied host callbacks (e.g. torch.distributed over gloo): the stream is
// drained, the buffer goes through host memory.  Several processes can then run the
// real sharded path -- separate address spaces, real exchanges -- on one GPU or on
// CPU-only transports; tests use it, production uses NCCL.
#include <dlfcn.h>
#include <cstring>
#include "comm.hpp"

namespace spd {

namespace {
typedef int (*fn_get_id)(void*);
typedef int (*fn_init_rank)(void**, int, Nccl128, int);
typedef int (*fn_bcast)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*fn_allreduce)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*fn_group)();
typedef int (*fn_destroy)(void*);
typedef const char* (*fn_errstr)(int);
struct NcclApi {
    void* h = nullptr;
    fn_get_id get_id = nullptr;
    fn_init_rank init_rank = nullptr;
    fn_bcast bcast = nullptr;
    fn_allreduce allreduce = nullptr;
    fn_group group_start = nullptr, group_end = nullptr;
    fn_destroy destroy = nullptr;
    fn_errstr errstr = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    if (api.h) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error(SPD_ENCCL, std::string("libnccl.so.2 not loadable: ") + dlerror());
    api.get_id = (fn_get_id)dlsym(h, "ncclGetUniqueId");
    api.init_rank = (fn_init_rank)dlsym(h, "ncclCommInitRank");
    api.bcast = (fn_bcast)dlsym(h, "ncclBroadcast");
    api.allreduce = (fn_allreduce)dlsym(h, "ncclAllReduce");
    api.group_start = (fn_group)dlsym(h, "ncclGroupStart");
    api.group_end = (fn_group)dlsym(h, "ncclGroupEnd");
    api.destroy = (fn_destroy)dlsym(h, "ncclCommDestroy");
    api.errstr = (fn_errstr)dlsym(h, "ncclGetErrorString");
    if (!api.get_id || !api.init_rank || !api.bcast || !api.allreduce || !api.group_start || !api.group_end ||
        !api.destroy)
        throw Error(SPD_ENCCL, "libnccl.so.2: missing symbols");
    api.h = h;
    return api;
}
void check(int r, const char* what) {
    if (r != 0) {
        const char* m = nccl().errstr ? nccl().errstr(r) : "?";
        throw Error(SPD_ENCCL, std::string(what) + ": " + m);
    }
}
// ncclDataType_t / ncclRedOp_t values (nccl.h)
constexpr int NCCL_INT8 = 0, NCCL_INT32 = 2, NCCL_FLOAT64 = 8, NCCL_SUM = 0;
}  // namespace

void comm_unique_id(void* out128) { check(nccl().get_id(out128), "ncclGetUniqueId"); }

spd_comm_s* comm_create(const void* id, int nranks, int rank) {
    SPD_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "spd_comm_init: bad nranks / rank");
    SPD_REQUIRE((nranks & (nranks - 1)) == 0, "spd_comm_init: nranks must be a power of 2 (binary subtrees)");
    auto* c = new spd_comm_s();
    c->nranks = nranks;
    c->rank = rank;
    if (nranks > 1 && id) {
        Nccl128 uid;
        memcpy(uid.b, id, sizeof(uid.b));
        try { check(nccl().init_rank(&c->nccl, nranks, uid, rank), "ncclCommInitRank"); }
        catch (...) { delete c; throw; }
    } else if (nranks > 1) {
        c->virt = true;                            // single-process emulation (tests)
    }
    return c;
}

spd_comm_s* comm_create_host(const spd_host_coll* ops, int nranks, int rank) {
    SPD_REQUIRE(ops && ops->allreduce_sum_f64 && ops->allreduce_sum_i32 && ops->broadcast,
                "spd_comm_init_host: missing callback");
    SPD_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "spd_comm_init_host: bad nranks / rank");
    SPD_REQUIRE((nranks & (nranks - 1)) == 0, "spd_comm_init_host: nranks must be a power of 2 (binary subtrees)");
    auto* c = new spd_comm_s();
    c->nranks = nranks;
    c->rank = rank;
    c->hosted = true;
    c->host = *ops;
    return c;
}

namespace {
// host-staged collective: stream drained, buffer through pageable host memory
void host_check(int r, const char* what) {
    if (r != 0) throw Error(SPD_ENCCL, std::string("host collective ") + what + " failed");
}
template <class T>
void host_allreduce(const spd_comm_s* c, T* buf, size_t n, cudaStream_t s,
                    int (*fn)(void*, T*, size_t)) {
    if (!n) return;
    std::vector<T> h(n);
    SPD_CUDA(cudaMemcpyAsync(h.data(), buf, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    SPD_CUDA(cudaStreamSynchronize(s));
    host_check(fn(c->host.ctx, h.data(), n), "allreduce");
    SPD_CUDA(cudaMemcpyAsync(buf, h.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
    SPD_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

void comm_destroy(spd_comm_s* c) {
    if (!c) return;
    if (c->nccl) nccl().destroy(c->nccl);
    delete c;
}

int shard_owner(const spd_comm_s* c, int count, int a) {
    const int P = c ? c->nranks : 1;
    if (P <= 1 || count < P) return -1;            // redundant level
    const int per = count / P;
    return a / per;
}

void comm_bcast_ranges(const spd_comm_s* c, void* buf, size_t elem, const std::vector<int64_t>& begin,
                       const std::vector<int64_t>& end, cudaStream_t s) {
    if (!c || c->nranks <= 1 || c->virt) return;   // one copy of everything already
    for (int q = 0; q < c->nranks; ++q)
        if (q != c->rank && end[q] > begin[q]) c->bytes_in += (end[q] - begin[q]) * (int64_t)elem;
    c->ncoll += 1;
    if (c->hosted) {
        SPD_CUDA(cudaStreamSynchronize(s));
        for (int q = 0; q < c->nranks; ++q) {
            const int64_t n = end[q] - begin[q];
            if (n <= 0) continue;
            std::vector<char> h((size_t)n * elem);
            char* p = (char*)buf + (size_t)begin[q] * elem;
            if (q == c->rank) SPD_CUDA(cudaMemcpy(h.data(), p, h.size(), cudaMemcpyDeviceToHost));
            host_check(c->host.broadcast(c->host.ctx, h.data(), h.size(), q), "broadcast");
            if (q != c->rank) SPD_CUDA(cudaMemcpy(p, h.data(), h.size(), cudaMemcpyHostToDevice));
        }
        return;
    }
    NcclApi& api = nccl();
    check(api.group_start(), "ncclGroupStart");
    for (int q = 0; q < c->nranks; ++q) {
        const int64_t n = end[q] - begin[q];
        if (n <= 0) continue;
        char* p = (char*)buf + (size_t)begin[q] * elem;
        check(api.bcast(p, p, (size_t)n * elem, NCCL_INT8, q, c->nccl, s), "ncclBroadcast");
    }
    check(api.group_end(), "ncclGroupEnd");
}

void comm_bcast_rows(const spd_comm_s* c, double* buf, int64_t ld, int ncols, const std::vector<int64_t>& begin,
                     const std::vector<int64_t>& end, cudaStream_t s) {
    if (!c || c->nranks <= 1 || c->virt) return;
    if (c->hosted) {                               // (counted per column by comm_bcast_ranges)
        for (int j = 0; j < ncols; ++j) comm_bcast_ranges(c, buf + (size_t)j * ld, sizeof(double), begin, end, s);
        return;
    }
    for (int q = 0; q < c->nranks; ++q)
        if (q != c->rank && end[q] > begin[q]) c->bytes_in += (end[q] - begin[q]) * (int64_t)sizeof(double) * ncols;
    c->ncoll += 1;
    NcclApi& api = nccl();
    constexpr int kGroupOps = 512;                 // bounded group size
    int ops = 0;
    check(api.group_start(), "ncclGroupStart");
    for (int j = 0; j < ncols; ++j)
        for (int q = 0; q < c->nranks; ++q) {
            const int64_t n = end[q] - begin[q];
            if (n <= 0) continue;
            double* p = buf + (size_t)j * ld + begin[q];
            check(api.bcast(p, p, (size_t)n, NCCL_FLOAT64, q, c->nccl, s), "ncclBroadcast");
            if (++ops % kGroupOps == 0) {
                check(api.group_end(), "ncclGroupEnd");
                check(api.group_start(), "ncclGroupStart");
            }
        }
    check(api.group_end(), "ncclGroupEnd");
}

void comm_allreduce_sum(const spd_comm_s* c, double* buf, size_t n, cudaStream_t s) {
    if (!c || c->nranks <= 1 || c->virt) return;
    c->bytes_in += (int64_t)(n * sizeof(double));  // the summed buffer (the ring moves ~2x (P-1)/P of it)
    c->ncoll += 1;
    if (c->hosted) return host_allreduce<double>(c, buf, n, s, c->host.allreduce_sum_f64);
    check(nccl().allreduce(buf, buf, n, NCCL_FLOAT64, NCCL_SUM, c->nccl, s), "ncclAllReduce");
}
void comm_allreduce_sum(const spd_comm_s* c, int* buf, size_t n, cudaStream_t s) {
    if (!c || c->nranks <= 1 || c->virt) return;
    c->bytes_in += (int64_t)(n * sizeof(int));
    c->ncoll += 1;
    if (c->hosted) return host_allreduce<int>(c, buf, n, s, c->host.allreduce_sum_i32);
    check(nccl().allreduce(buf, buf, n, NCCL_INT32, NCCL_SUM, c->nccl, s), "ncclAllReduce");
}

}  // namespace spd
