// prof.cpp -- launch counter and per-kernel-class event timing (instrumentation).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include "common.cuh"

namespace spd {

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
struct Rec { std::string name; double flops, bytes; cudaEvent_t a, b; };
}  // namespace
struct ProfCaptured { std::vector<Rec> recs; };
namespace {
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
cudaEvent_t get_ev() {
    if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
struct Agg { long long n = 0; double ms = 0, flops = 0, bytes = 0; };
std::map<std::string, Agg> g_agg;
void drain() {       // caller holds the mutex
    for (auto& r : g_recs) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        Agg& a = g_agg[r.name];
        a.n += 1; a.ms += ms; a.flops += r.flops; a.bytes += r.bytes;
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
}
}  // namespace

// stage marks (env SPD_STAGES=1): synchronize and print the wall time since the last mark
void stage_mark(cudaStream_t s, const char* name, int level) {
    static const bool on = getenv("SPD_STAGES") != nullptr;
    static double last = 0.0;
    if (!on) return;
    cudaStreamSynchronize(s);
    const double t = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    if (name) fprintf(stderr, "[stage] %-24s L%-2d %9.3f ms\n", name, level, last > 0.0 ? (t - last) * 1e3 : 0.0);
    last = t;
}

cudaStream_t& alloc_stream() {
    static thread_local cudaStream_t st = nullptr;
    return st;
}
void init_mem_pool() {
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return; }
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) { cudaGetLastError(); return; }
        // The pool keeps up to half the device memory mapped across synchronizations and is
        // pre-grown once: growing it mid-build (mapping new physical memory when no free
        // block fits) stalled single allocations for 50 ms - 1.3 s on B200 (measured in
        // tools/phase_probe.py: spdhss_build 72 ms -> up to 1391 ms), a pre-grown pool of
        // min(30 % of the free memory, 48 GB) removed the outliers.  SPD_POOL_RESERVE_GB
        // overrides the reservation (0: none).
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); fr = tot = (size_t)48 << 30; }
        uint64_t thr = getenv("SPD_POOL_KEEP_ALL") ? ~0ull : (uint64_t)(tot / 2);   // >= the reserve
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        size_t reserve = std::min<size_t>((size_t)(0.3 * (double)fr), (size_t)48 << 30);
        if (const char* r = getenv("SPD_POOL_RESERVE_GB")) reserve = (size_t)(atof(r) * (double)(1ull << 30));
        if (reserve > 0) {
            void* p = nullptr;
            if (cudaMallocAsync(&p, reserve, 0) == cudaSuccess) { cudaFreeAsync(p, 0); cudaStreamSynchronize(0); }
            cudaGetLastError();
        }
    });
}

// device memory available to the library: free device memory plus the memory the pool
// has mapped but not handed out (the pre-grown reserve)
size_t device_free_bytes() {
    size_t fr = 0, tot = 0;
    SPD_CUDA(cudaMemGetInfo(&fr, &tot));
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t res = 0, used = 0;
        if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && res > used)
            fr += (size_t)(res - used);
    }
    cudaGetLastError();
    return fr;
}

DescArena*& desc_arena() {
    static thread_local DescArena* a = nullptr;
    return a;
}

static bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    return st == cudaStreamCaptureStatusActive;
}

ProfScope::ProfScope(cudaStream_t st, const char* name, double flops, double bytes) : s(st) {
    if (!g_on) return;
    std::lock_guard<std::mutex> lk(g_mu);
    Rec r{name, flops, bytes, get_ev(), get_ev()};
    ext = capturing(s);
    if (ext) cudaEventRecordWithFlags(r.a, s, cudaEventRecordExternal);
    else cudaEventRecord(r.a, s);
    g_recs.push_back(r);
    slot = (int)g_recs.size() - 1;
}
ProfScope::~ProfScope() {
    if (slot < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    if (ext) cudaEventRecordWithFlags(g_recs[slot].b, s, cudaEventRecordExternal);
    else cudaEventRecord(g_recs[slot].b, s);
    if (!ext && g_recs.size() > 20000) drain();
}

bool prof_on() { return g_on; }

void prof_update_last(const char* name, double flops, double bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = g_recs.size(); i-- > 0;)
        if (g_recs[i].name == name) { g_recs[i].flops = flops; g_recs[i].bytes = bytes; return; }
}

size_t prof_mark() {
    std::lock_guard<std::mutex> lk(g_mu);
    return g_recs.size();
}
ProfCaptured* prof_capture_take(size_t first) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto* c = new ProfCaptured();
    if (first < g_recs.size()) {
        c->recs.assign(g_recs.begin() + first, g_recs.end());
        g_recs.resize(first);
    }
    return c;
}
void prof_accumulate(ProfCaptured* c) {
    if (!c) return;
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& r : c->recs) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) { cudaGetLastError(); continue; }
        Agg& a = g_agg[r.name];
        a.n += 1; a.ms += ms; a.flops += r.flops; a.bytes += r.bytes;
    }
}
void prof_release(ProfCaptured* c) {
    if (!c) return;
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& r : c->recs) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
    delete c;
}

}  // namespace spd

extern "C" {
void spd_prof_enable(int on) { spd::g_on = on != 0; }
void spd_prof_reset(void) {
    std::lock_guard<std::mutex> lk(spd::g_mu);
    spd::drain();
    spd::g_agg.clear();
}
int spd_prof_count(void) {
    std::lock_guard<std::mutex> lk(spd::g_mu);
    spd::drain();
    return (int)spd::g_agg.size();
}
int spd_prof_get(int idx, char* name, int name_len, double* out4) {
    std::lock_guard<std::mutex> lk(spd::g_mu);
    spd::drain();
    int i = 0;
    for (auto& kv : spd::g_agg) {
        if (i++ != idx) continue;
        std::strncpy(name, kv.first.c_str(), name_len - 1);
        name[name_len - 1] = 0;
        out4[0] = (double)kv.second.n; out4[1] = kv.second.ms; out4[2] = kv.second.flops; out4[3] = kv.second.bytes;
        return 0;
    }
    return 1;
}
long long spd_launch_count(void) { return spd::g_launches.load(); }
}
