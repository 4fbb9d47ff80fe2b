// tree_dev.cu -- the cluster tree (reading R1) and the dual-tree interaction lists
// (reading R2) built on the device (§2 P:176-198 for the
// tree, §5.1 P:657-663 and P:891-913 for the near / Type-1 / Type-3 pairs).
//
// Tree, level by level from the root (all nodes of a level at once):
//   * node ranges are data-independent (a node of n points splits into ceil(n/2),
//     floor(n/2)), so they are computed on the host;
//   * tight boxes: segmented min / max over each node's points (exact, order free);
//   * split dimension: argmax of the extent, lowest dimension on ties;
//   * the left child is the SET of the ceil(n/2) smallest points by the 96-bit key
//     (order-preserving bits of the coordinate, original index) -- unique keys, so an
//     MSD radix select (12 passes of 8 bits) finds the ceil(n/2)-th key exactly and a
//     partition moves the points (their order inside a child does not matter: the
//     child is selected again by its own key);
//   * the last split level sorts every node's points by that key (bitonic sort in
//     shared memory): this fixes the order inside each leaf.
// Every comparison is exact (integer keys; -0.0 is canonicalized to +0.0 so the key
// order is the order of double comparison), hence the permutation, node ranges and
// boxes are bit-identical to the oracle's (R1) and to the host builder (tree.cpp).
//
// Lists: breadth-first dual-tree traversal from (root, root), one launch per level:
// a pair (i, j) of level k is Type-3 if i != j and far (R2, exact single-rounded ops),
// else Type-1 if i != j, a near block if k = 1, else its four child pairs go to the
// next level.  Output positions come from atomics; the lists are sorted afterwards
// (the same sorted lists as the host traversal).
#include "tree.hpp"
#include "common.cuh"
#include <algorithm>
#include <cstring>

namespace spd {

namespace {

constexpr int TCH = 4096;          // points per work item
constexpr int SORT_MAX = 4096;     // largest node sorted in shared memory (2 leaves)

struct SegItem { int seg; int64_t b, e; };

__device__ __forceinline__ unsigned long long coord_key(double x) {
    if (x == 0.0) x = 0.0;                                   // -0.0 -> +0.0 (equal as doubles)
    const unsigned long long u = (unsigned long long)__double_as_longlong(x);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// 8-bit digit p (0 = most significant) of the 96-bit key (coord key, index)
__device__ __forceinline__ unsigned digit(unsigned long long ck, unsigned idx, int p) {
    return p < 8 ? (unsigned)(ck >> (56 - 8 * p)) & 255u : (idx >> (24 - 8 * (p - 8))) & 255u;
}

__global__ void bbox_partial_kernel(const SegItem* __restrict__ items, const int* __restrict__ idx,
                                    const double* __restrict__ pts, int d, double* __restrict__ part) {
    const SegItem it = items[blockIdx.x];
    __shared__ double slo[8][3], shi[8][3];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t p = it.b + threadIdx.x; p < it.e; p += blockDim.x) {
        const int64_t o = (int64_t)idx[p] * d;
        for (int a = 0; a < d; ++a) { const double x = pts[o + a]; lo[a] = fmin(lo[a], x); hi[a] = fmax(hi[a], x); }
    }
    for (int a = 0; a < d; ++a)
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
        for (int a = 0; a < d; ++a) { slo[w][a] = lo[a]; shi[w][a] = hi[a]; }
    __syncthreads();
    if (threadIdx.x < d) {
        double l = INFINITY, h = -INFINITY;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { l = fmin(l, slo[q][threadIdx.x]); h = fmax(h, shi[q][threadIdx.x]); }
        part[(size_t)blockIdx.x * 6 + threadIdx.x] = l;
        part[(size_t)blockIdx.x * 6 + 3 + threadIdx.x] = h;
    }
}

// one thread per segment: reduce its items' partials into the node box, pick the split
// dimension (argmax extent, lowest on ties), reset the selection state
__global__ void bbox_reduce_kernel(const int2* __restrict__ seg_items, const double* __restrict__ part, int nseg,
                                   int first_node, int d, double* __restrict__ lo, double* __restrict__ hi,
                                   int* __restrict__ sdim) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    const int2 r = seg_items[s];
    double l[3] = {INFINITY, INFINITY, INFINITY}, h[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int q = r.x; q < r.y; ++q)
        for (int a = 0; a < d; ++a) { l[a] = fmin(l[a], part[(size_t)q * 6 + a]); h[a] = fmax(h[a], part[(size_t)q * 6 + 3 + a]); }
    const int node = first_node + s;
    int best = 0;
    double bext = __dsub_rn(h[0], l[0]);
    for (int a = 0; a < d; ++a) {
        lo[(size_t)node * d + a] = l[a];
        hi[(size_t)node * d + a] = h[a];
        const double ext = __dsub_rn(h[a], l[a]);
        if (a > 0 && ext > bext) { bext = ext; best = a; }
    }
    sdim[s] = best;
}

struct SelState { unsigned long long ck; unsigned ix; int k; };   // prefix key (digits so far) and rank left

__global__ void select_hist_kernel(const SegItem* __restrict__ items, const int* __restrict__ idx,
                                   const double* __restrict__ pts, int d, const int* __restrict__ sdim,
                                   const SelState* __restrict__ st, int pass, unsigned* __restrict__ hist) {
    __shared__ unsigned h[256];
    const SegItem it = items[blockIdx.x];
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const int sd = sdim[it.seg];
    const SelState s = st[it.seg];
    for (int64_t p = it.b + threadIdx.x; p < it.e; p += blockDim.x) {
        const unsigned ix = (unsigned)idx[p];
        const unsigned long long ck = coord_key(pts[(int64_t)ix * d + sd]);
        bool match = true;                               // the first `pass` digits equal the prefix
        for (int q = 0; q < pass && match; ++q) match = digit(ck, ix, q) == digit(s.ck, s.ix, q);
        if (match) atomicAdd(&h[digit(ck, ix, pass)], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd(&hist[(size_t)it.seg * 256 + b], h[b]);
}

__global__ void select_step_kernel(SelState* __restrict__ st, unsigned* __restrict__ hist, int nseg, int pass) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    SelState x = st[s];
    unsigned* hs = hist + (size_t)s * 256;
    int b = 0;
    for (; b < 256; ++b) {
        const int c = (int)hs[b];
        if (x.k < c) break;
        x.k -= c;
    }
    for (int q = 0; q < 256; ++q) hs[q] = 0;
    if (pass < 8) x.ck |= (unsigned long long)b << (56 - 8 * pass);
    else x.ix |= (unsigned)b << (24 - 8 * (pass - 8));
    st[s] = x;
}

__global__ void partition_kernel(const SegItem* __restrict__ items, const int* __restrict__ idx_in,
                                 int* __restrict__ idx_out, const double* __restrict__ pts, int d,
                                 const int* __restrict__ sdim, const SelState* __restrict__ st,
                                 const int64_t* __restrict__ seg_b, const int64_t* __restrict__ seg_mid,
                                 unsigned long long* __restrict__ cnt) {
    const SegItem it = items[blockIdx.x];
    const int sd = sdim[it.seg];
    const SelState s = st[it.seg];
    for (int64_t p = it.b + threadIdx.x; p < it.e; p += blockDim.x) {
        const unsigned ix = (unsigned)idx_in[p];
        const unsigned long long ck = coord_key(pts[(int64_t)ix * d + sd]);
        const bool left = ck < s.ck || (ck == s.ck && ix <= s.ix);
        const unsigned long long o = atomicAdd(&cnt[2 * it.seg + (left ? 0 : 1)], 1ull);
        idx_out[(left ? seg_b[it.seg] : seg_mid[it.seg]) + (int64_t)o] = (int)ix;
    }
}

// last split level: sort every node's points by (coord key, index), bitonic in smem
__global__ void __launch_bounds__(512) segment_sort_kernel(const int64_t* __restrict__ seg_b,
                                                           const int64_t* __restrict__ seg_e, int* __restrict__ idx,
                                                           const double* __restrict__ pts, int d,
                                                           const int* __restrict__ sdim) {
    extern __shared__ unsigned long long sk[];                // ck[P2], then ix[P2] as unsigned
    const int s = blockIdx.x;
    const int64_t b = seg_b[s];
    const int n = (int)(seg_e[s] - b);
    int P2 = 1;
    while (P2 < n) P2 <<= 1;
    unsigned* sx = (unsigned*)(sk + P2);
    const int sd = sdim[s];
    for (int q = threadIdx.x; q < P2; q += blockDim.x) {
        if (q < n) { const unsigned ix = (unsigned)idx[b + q]; sx[q] = ix; sk[q] = coord_key(pts[(int64_t)ix * d + sd]); }
        else { sx[q] = 0xffffffffu; sk[q] = ~0ull; }
    }
    __syncthreads();
    for (int kk = 2; kk <= P2; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int q = threadIdx.x; q < P2; q += blockDim.x) {
                const int l = q ^ j;
                if (l > q) {
                    const bool up = (q & kk) == 0;
                    const bool gt = sk[q] > sk[l] || (sk[q] == sk[l] && sx[q] > sx[l]);
                    if (gt == up) {
                        const unsigned long long tk = sk[q]; sk[q] = sk[l]; sk[l] = tk;
                        const unsigned tx = sx[q]; sx[q] = sx[l]; sx[l] = tx;
                    }
                }
            }
            __syncthreads();
        }
    for (int q = threadIdx.x; q < n; q += blockDim.x) idx[b + q] = (int)sx[q];
}

// ---------------------------------------------------------------- lists
__device__ bool is_far_dev(const double* __restrict__ lo, const double* __restrict__ hi, int d, int i, int j) {
    if (i == j) return false;
    double ei[3], ej[3], mi = 0.0, mj = 0.0;
    for (int a = 0; a < d; ++a) {
        ei[a] = __dmul_rn(0.5, __dsub_rn(hi[(size_t)i * d + a], lo[(size_t)i * d + a]));
        ej[a] = __dmul_rn(0.5, __dsub_rn(hi[(size_t)j * d + a], lo[(size_t)j * d + a]));
        mi = fmax(mi, ei[a]);
        mj = fmax(mj, ej[a]);
    }
    for (int a = 0; a < d; ++a) {
        const double hi_ = fmax(ei[a], __dmul_rn(0.25, mi)), hj_ = fmax(ej[a], __dmul_rn(0.25, mj));
        const double gap = fmax(__dsub_rn(lo[(size_t)j * d + a], hi[(size_t)i * d + a]),
                                __dsub_rn(lo[(size_t)i * d + a], hi[(size_t)j * d + a]));
        if (gap > 0.0 && gap >= fmax(hi_, hj_)) return true;
    }
    return false;
}

// counters: 0 type3, 1 type1, 2 near, 3 next
__global__ void list_level_kernel(const int2* __restrict__ in, int n_in, int leaf_level, const double* __restrict__ lo,
                                  const double* __restrict__ hi, int d, int2* __restrict__ t3, int2* __restrict__ t1,
                                  int2* __restrict__ nr, int2* __restrict__ next, int* __restrict__ cnt) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_in) return;
    const int2 pr = in[q];
    if (pr.x != pr.y && is_far_dev(lo, hi, d, pr.x, pr.y)) { t3[atomicAdd(&cnt[0], 1)] = pr; return; }
    if (pr.x != pr.y) t1[atomicAdd(&cnt[1], 1)] = pr;
    if (leaf_level) { nr[atomicAdd(&cnt[2], 1)] = pr; return; }
    const int o = atomicAdd(&cnt[3], 4);
    int c = 0;
    for (int ci = 2 * pr.x + 1; ci <= 2 * pr.x + 2; ++ci)
        for (int cj = 2 * pr.y + 1; cj <= 2 * pr.y + 2; ++cj) next[o + c++] = make_int2(ci, cj);
}

}  // namespace

bool build_tree_device(const double* pts, int64_t N, int d, int leaf, TreeH& t, cudaStream_t s) {
    int depth = 0;
    while ((int64_t)leaf << depth < N) ++depth;
    // host ranges (data-independent)
    t.N = N; t.d = d; t.depth = depth; t.L = depth + 1; t.nnodes = (1 << (depth + 1)) - 1;
    t.begin.assign(t.nnodes, 0); t.end.assign(t.nnodes, 0);
    t.end[0] = N;
    for (int i = 0; 2 * i + 2 < t.nnodes; ++i) {
        const int64_t b = t.begin[i], e = t.end[i], mid = b + (e - b + 1) / 2;
        t.begin[2 * i + 1] = b; t.end[2 * i + 1] = mid;
        t.begin[2 * i + 2] = mid; t.end[2 * i + 2] = e;
    }
    if (depth > 0) {
        const int last = (1 << (depth - 1)) - 1;                  // nodes sorted at the last split level
        for (int i = last; i < last + (1 << (depth - 1)); ++i)
            if (t.size(i) > SORT_MAX) return false;                // very large leaves: host builder
    }
    if (N > (int64_t)0x7fffffff) return false;
    DBuf<int> idx(N), idx2(N);
    {
        std::vector<int> io(N);
        for (int64_t p = 0; p < N; ++p) io[p] = (int)p;
        idx.upload(io, s);
    }
    DBuf<double> lo_d((size_t)t.nnodes * d), hi_d((size_t)t.nnodes * d);
    for (int dl = 0; dl <= depth; ++dl) {
        const int first = (1 << dl) - 1, nseg = 1 << dl;
        std::vector<SegItem> items;
        std::vector<int2> seg_items(nseg);
        std::vector<int64_t> sb(nseg), se(nseg), smid(nseg);
        for (int a = 0; a < nseg; ++a) {
            const int i = first + a;
            sb[a] = t.begin[i]; se[a] = t.end[i]; smid[a] = sb[a] + (se[a] - sb[a] + 1) / 2;
            seg_items[a].x = (int)items.size();
            for (int64_t b = sb[a]; b < se[a] || b == sb[a]; b += TCH) items.push_back({a, b, std::min(se[a], b + TCH)});
            seg_items[a].y = (int)items.size();
        }
        DevArray<SegItem> di(s, items);
        DevArray<int2> dsi(s, seg_items);
        DBuf<double> part(items.size() * 6);
        DBuf<int> sdim(nseg);
        bbox_partial_kernel<<<(unsigned)items.size(), 256, 0, s>>>(di.p, idx.p, pts, d, part.p);
        SPD_LAUNCH();
        bbox_reduce_kernel<<<ceil_div(nseg, 128), 128, 0, s>>>(dsi.p, part.p, nseg, first, d, lo_d.p, hi_d.p, sdim.p);
        SPD_LAUNCH();
        if (dl == depth) break;
        DBuf<int64_t> sb_d, se_d;
        sb_d.upload(sb, s);
        se_d.upload(se, s);
        if (dl == depth - 1) {                     // children are leaves: full sort fixes their order
            int p2max = 1;
            for (int a = 0; a < nseg; ++a) { int p2 = 1; while (p2 < se[a] - sb[a]) p2 <<= 1; p2max = std::max(p2max, p2); }
            const size_t sh = (size_t)p2max * 12;
            static bool attr = false;
            if (!attr) {
                SPD_CUDA(cudaFuncSetAttribute(segment_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
                attr = true;
            }
            segment_sort_kernel<<<nseg, 512, sh, s>>>(sb_d.p, se_d.p, idx.p, pts, d, sdim.p);
            SPD_LAUNCH();
            continue;
        }
        // radix select of the ceil(n/2)-th key per node, then partition
        std::vector<SelState> st0(nseg);
        for (int a = 0; a < nseg; ++a) st0[a] = {0ull, 0u, (int)(smid[a] - sb[a]) - 1};
        DevArray<SelState> st(s, st0);
        DBuf<unsigned> hist((size_t)nseg * 256);
        hist.zero(s);
        for (int pass = 0; pass < 12; ++pass) {
            select_hist_kernel<<<(unsigned)items.size(), 256, 0, s>>>(di.p, idx.p, pts, d, sdim.p, st.p, pass, hist.p);
            SPD_LAUNCH();
            select_step_kernel<<<ceil_div(nseg, 128), 128, 0, s>>>(st.p, hist.p, nseg, pass);
            SPD_LAUNCH();
        }
        DBuf<int64_t> smid_d;
        smid_d.upload(smid, s);
        DBuf<unsigned long long> cnt((size_t)2 * nseg);
        cnt.zero(s);
        partition_kernel<<<(unsigned)items.size(), 256, 0, s>>>(di.p, idx.p, idx2.p, pts, d, sdim.p, st.p, sb_d.p,
                                                                smid_d.p, cnt.p);
        SPD_LAUNCH();
        std::swap(idx, idx2);
    }
    std::vector<int> io = idx.download(s);
    t.perm.resize(N);
    for (int64_t p = 0; p < N; ++p) t.perm[p] = io[p];
    t.lo = lo_d.download(s);
    t.hi = hi_d.download(s);
    return true;
}

void build_lists_device(const TreeH& t, ListsH& l, cudaStream_t s) {
    l.near.clear();
    l.type1.assign(t.L + 1, {});
    l.type3.assign(t.L + 1, {});
    DBuf<double> lo_d, hi_d;
    lo_d.upload(t.lo, s);
    hi_d.upload(t.hi, s);
    DBuf<int> cnt(4);
    std::vector<int2> init{make_int2(0, 0)};
    DBuf<int2> cur;
    {
        cur.alloc(1);
        SPD_CUDA(cudaMemcpyAsync(cur.p, init.data(), sizeof(int2), cudaMemcpyHostToDevice, s));
    }
    int n_in = 1;
    auto to_pairs = [&](const DBuf<int2>& b, int n, std::vector<Pair>& out) {
        std::vector<int2> h(n);
        if (n) {
            SPD_CUDA(cudaMemcpyAsync(h.data(), b.p, sizeof(int2) * n, cudaMemcpyDeviceToHost, s));
            SPD_CUDA(cudaStreamSynchronize(s));
        }
        out.reserve(out.size() + n);
        for (auto& p : h) out.push_back({p.x, p.y});
    };
    for (int k = t.L; k >= 1 && n_in > 0; --k) {
        DBuf<int2> t3(n_in), t1(n_in), nr(k == 1 ? n_in : 1), next(k > 1 ? 4 * (size_t)n_in : 1);
        cnt.zero(s);
        list_level_kernel<<<ceil_div(n_in, 256), 256, 0, s>>>(cur.p, n_in, k == 1 ? 1 : 0, lo_d.p, hi_d.p, t.d,
                                                             t3.p, t1.p, nr.p, next.p, cnt.p);
        SPD_LAUNCH();
        std::vector<int> c = cnt.download(s);
        to_pairs(t3, c[0], l.type3[k]);
        to_pairs(t1, c[1], l.type1[k]);
        if (k == 1) to_pairs(nr, c[2], l.near);
        cur = std::move(next);
        n_in = c[3];
    }
    std::sort(l.near.begin(), l.near.end());
    for (int k = 0; k <= t.L; ++k) {
        std::sort(l.type1[k].begin(), l.type1[k].end());
        std::sort(l.type3[k].begin(), l.type3[k].end());
    }
}

}  // namespace spd
