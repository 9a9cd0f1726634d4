// ks_exact.cu -- exact-mode K-sort: reproduces the reference's partition
// permutation (sort_core.py:81-105) and op counts (sort_core.py:108-143,
// 199-217) on the device.
//
// Used for ksort_partition (golden-trace API), k_sort(a, counts), and inputs
// that hold both -0.0 and +0.0 (the only finite keys that compare equal while
// differing in bits, so the only case where the arrangement of equal keys is
// observable in the output bytes).
//
// Level-synchronous driver: partitions of disjoint segments commute, so the
// reference's LIFO recursion tree (sort_core.py:182-198) is processed one
// tree level at a time ("processing order does not
// matter").  Large segments: one CTA per segment applies the data-parallel
// closed form of the partition (block-wide ballot/popc + scan ranks).
// Small segments: one lane per segment runs the reference's sequential
// partition loop itself.
#include <cstdio>
#include <unordered_map>
#include <vector>

#include "ks_host.h"
#include "ks_internal.cuh"

namespace ks {

constexpr int kExactThreads = 512;
constexpr int kExactSmall = 512;   // segments <= this run the sequential loop on one lane

struct XSeg {
    long long L, R;
};

struct XLog {                // one node of the recursion tree (counts mode)
    long long L, R;
    long long v;             // pivot index, or local max pending for a collapsed subtree
    long long collapsed;
};

struct XStatus {
    int nbig[2];
    int nsmall;
    int nlog;
    int overflow;
    int levels;   // levels that had work (counted on the device: the host launches them in batches)
    unsigned long long comparisons, moves;
};

// ---- block helpers -----------------------------------------------------------

// exclusive prefix of a 0/1 flag across the block (ballot + popc per warp)
__device__ __forceinline__ int block_flag_scan(int flag, int *sw, int *total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned b = __ballot_sync(0xffffffffu, flag);
    int in_warp = __popc(b & ((1u << lane) - 1u));
    if (lane == 0) sw[wid] = __popc(b);
    __syncthreads();
    if (wid == 0) {
        int x = lane < nw ? sw[lane] : 0, inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane < nw) sw[lane] = inc - x;
        if (lane == 31) sw[32] = inc;
    }
    __syncthreads();
    int r = sw[wid] + in_warp;
    *total = sw[32];
    __syncthreads();
    return r;
}

__device__ __forceinline__ long long block_sum_ll(long long x, long long *sh)
{
    long long t;
    block_exclusive_scan(x, sh, &t);
    return t;
}

// ---- one exact partition of a[L..R] by one CTA ----------------------------------
//
// Closed form (checked against sort_core._partition):
//   nl = #{p in (L,R] : a[p] < key},  piv = L + nl,  A = [L+1, piv], Z = [piv+1, R]
//   B_1..B_c = ge positions in A (increasing), G_1..G_c = lt positions in Z (decreasing)
//   out[p-1] = a[p] for lt p in A;  out[B_k - 1] = a[G_k]
//   out[piv] = key
//   Z: out[G_k] = a[B_{k+1}] (k < c); out[G_c] = a[e*] if a[e*] >= key; out[e*] = a[B_1]
//   with e* = piv+1; Z unchanged when c == 0.
struct XPart {
    long long piv;
    long long c;
    int flag;
    unsigned long long moves;
};

__device__ XPart exact_partition_cta(const double *a, double *out, long long L, long long R,
                                     long long *Bl, long long *Gl, int *sw, long long *sh)
{
    const double key = a[L];
    long long nl_local = 0;
    for (long long p = L + 1 + threadIdx.x; p <= R; p += blockDim.x) nl_local += (a[p] < key) ? 1 : 0;
    const long long nl = block_sum_ll(nl_local, sh);
    const long long piv = L + nl;
    const long long e = piv + 1;

    // G list: lt positions in Z scanned from R downwards
    long long c = 0;
    for (long long base = R; base > piv; base -= blockDim.x) {
        long long q = base - threadIdx.x;
        int f = (q > piv && a[q] < key) ? 1 : 0;
        int tot;
        int r = block_flag_scan(f, sw, &tot);
        if (f) Gl[L + c + r] = q;
        c += tot;
    }
    __syncthreads();
    // A: shift left by one, ge slots take G values; record B list
    long long cb = 0;
    for (long long base = L + 1; base <= piv; base += blockDim.x) {
        long long p = base + threadIdx.x;
        int inA = p <= piv;
        double v = inA ? a[p] : 0.0;
        int f = (inA && !(v < key)) ? 1 : 0;
        int tot;
        int r = block_flag_scan(f, sw, &tot);
        if (inA) {
            if (f) {
                Bl[L + cb + r] = p;
                out[p - 1] = a[Gl[L + cb + r]];
            } else {
                out[p - 1] = v;
            }
        }
        cb += tot;
    }
    __syncthreads();
    if (threadIdx.x == 0) out[piv] = key;
    // Z
    const bool estar_ge = (c >= 1) && !(a[e] < key);
    long long cg = 0;
    for (long long base = R; base > piv; base -= blockDim.x) {
        long long q = base - threadIdx.x;
        int inZ = q > piv;
        double v = inZ ? a[q] : 0.0;
        int f = (inZ && v < key) ? 1 : 0;
        int tot;
        int r = block_flag_scan(f, sw, &tot);
        if (inZ) {
            if (c == 0) {
                out[q] = v;
            } else if (f) {
                long long kk = cg + r;                       // 0-based index into G
                if (kk < c - 1) out[q] = a[Bl[L + kk + 1]];
                else out[q] = estar_ge ? a[e] : a[Bl[L]];    // G_c (== e* when a[e*] < key)
            } else if (q == e) {
                out[q] = a[Bl[L]];                           // stashed temp lands at e*
            } else {
                out[q] = v;
            }
        }
        cg += tot;
    }
    __syncthreads();
    XPart res;
    res.piv = piv;
    res.c = c;
    res.flag = piv < R ? 1 : 0;
    // moves = nl + nb + 1 + flag, nb = c + [Z non-empty and a[e*] >= key]
    const long long nb = c + ((piv < R && !(a[e] < key)) ? 1 : 0);
    res.moves = (unsigned long long)(nl + nb + 1 + res.flag);
    return res;
}

// ---- sequential reference loop on one lane (sort_core.py:81-105) -------------------
__device__ long long seq_partition(double *a, long long left, long long right,
                                   unsigned long long &cmp, unsigned long long &mv)
{
    const double key = a[left];
    long long i = left, j = right + 1, p = left + 1;
    bool flag = false;
    double temp = 0.0;
    while (j - i >= 2) {
        double v = a[p];
        ++cmp;
        if (key <= v) {
            if (j == right + 1) { temp = v; flag = true; ++mv; }
            else if (p != j) { a[j] = v; ++mv; }
            --j;
            p = j;
        } else {
            a[i] = v;
            ++mv;
            ++i;
            p = i + 1;
        }
    }
    a[i] = key;
    ++mv;
    if (flag) { a[i + 1] = temp; ++mv; }
    return i;
}

// sort_core.py:182-198 driver on one lane; returns the local max pending size
__device__ long long seq_k_sort(double *a, long long L, long long R, unsigned long long &cmp,
                                unsigned long long &mv)
{
    long long sl[64], sr[64];
    int top = 0;
    sl[0] = L;
    sr[0] = R;
    top = 1;
    long long hmax = 0;
    while (top > 0) {
        --top;
        long long left = sl[top], right = sr[top];
        long long piv = seq_partition(a, left, right, cmp, mv);
        long long lo_len = piv - left, hi_len = right - piv;
        if (lo_len <= hi_len) {
            if (hi_len >= 2) { sl[top] = piv + 1; sr[top] = right; ++top; }
            if (lo_len >= 2) { sl[top] = left; sr[top] = piv - 1; ++top; }
        } else {
            if (lo_len >= 2) { sl[top] = left; sr[top] = piv - 1; ++top; }
            if (hi_len >= 2) { sl[top] = piv + 1; sr[top] = right; ++top; }
        }
        if (top > hmax) hmax = top;
    }
    return hmax;
}

// ---- kernels -------------------------------------------------------------------

__device__ __forceinline__ void push_child(long long L, long long R, const double *src, double *keys,
                                           bool dst_is_keys, XSeg *big, XSeg *small, XStatus *xs,
                                           int big_cap, int small_cap)
{
    const long long len = R - L + 1;
    if (len <= 0) return;
    if (len == 1) {
        if (!dst_is_keys) keys[L] = src[L];   // final (never pushed, sort_core.py:190-198)
        return;
    }
    if (len <= kExactSmall) {
        int i = atomicAdd(&xs->nsmall, 1);
        if (i >= small_cap) { xs->overflow = 1; return; }
        small[i] = XSeg{L, R};
    } else {
        int i = atomicAdd(&xs->nbig[1], 1);   // caller swaps tables
        if (i >= big_cap) { xs->overflow = 2; return; }
        big[i] = XSeg{L, R};
    }
}

__global__ void __launch_bounds__(kExactThreads) k_exact_level(const XSeg *segs, const int *nseg,
                                                               const double *src, double *dst, double *keys,
                                                               int dst_is_keys, long long *Bl, long long *Gl,
                                                               XSeg *next_big, XSeg *small, XStatus *xs,
                                                               XLog *log, int log_cap, int big_cap,
                                                               int small_cap)
{
    __shared__ int sw[33];
    __shared__ long long sh[33];
    const int ns = *nseg;
    for (int s = blockIdx.x; s < ns; s += gridDim.x) {
        const XSeg g = segs[s];
        XPart pr = exact_partition_cta(src, dst, g.L, g.R, Bl, Gl, sw, sh);
        if (threadIdx.x == 0) {
            const long long m = g.R - g.L + 1;
            atomicAdd(&xs->comparisons, (unsigned long long)(m - 1));
            atomicAdd(&xs->moves, pr.moves);
            if (!dst_is_keys) keys[pr.piv] = dst[pr.piv];
            if (log) {
                int i = atomicAdd(&xs->nlog, 1);
                if (i < log_cap) log[i] = XLog{g.L, g.R, pr.piv, 0};
                else xs->overflow = 3;
            }
            // children (sort_core.py:187-198 pushes only lengths >= 2)
            push_child(g.L, pr.piv - 1, dst, keys, dst_is_keys, next_big, small, xs, big_cap, small_cap);
            push_child(pr.piv + 1, g.R, dst, keys, dst_is_keys, next_big, small, xs, big_cap, small_cap);
        }
        __syncthreads();
    }
}

// one lane per small segment: copy into the user buffer, then the reference's
// own sequential partition + LIFO driver
__global__ void k_exact_small(const XSeg *small, const int *nsmall, const double *src, double *keys,
                              int src_is_keys, XStatus *xs, XLog *log, int log_cap)
{
    const int ns = *nsmall;
    unsigned long long cmp = 0, mv = 0;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
        const XSeg g = small[s];
        if (!src_is_keys)
            for (long long i = g.L; i <= g.R; ++i) keys[i] = src[i];
        long long h = seq_k_sort(keys, g.L, g.R, cmp, mv);
        if (log) {
            int i = atomicAdd(&xs->nlog, 1);
            if (i < log_cap) log[i] = XLog{g.L, g.R, h, 1};
            else xs->overflow = 3;
        }
    }
    if (cmp) atomicAdd(&xs->comparisons, cmp);
    if (mv) atomicAdd(&xs->moves, mv);
}

// level bookkeeping on the device (the host launches kExactBatch levels per
// status read): phase 0, after the small-segment kernel: count the level,
// empty the small list and the next big table; phase 1, after the level
// kernel: the next table becomes the current one.
__global__ void k_exact_advance(XStatus *xs, int phase)
{
    if (threadIdx.x || blockIdx.x) return;
    if (phase == 0) {
        if (xs->nsmall > 0 || xs->nbig[0] > 0) ++xs->levels;
        xs->nsmall = 0;
        xs->nbig[1] = 0;
    } else {
        xs->nbig[0] = xs->nbig[1];
    }
}

__global__ void k_exact_init(long long n, XSeg *big, XSeg *small, XStatus *xs)
{
    if (threadIdx.x || blockIdx.x) return;
    if (n > kExactSmall) {
        big[0] = XSeg{0, n - 1};
        xs->nbig[0] = 1;
    } else if (n >= 2) {
        small[0] = XSeg{0, n - 1};
        xs->nsmall = 1;
    }
}

__global__ void k_exact_gate(const double *keys, long long n, unsigned long long *bad)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        if (!isfinite(keys[i])) atomicMin(bad, (unsigned long long)i);
}

// single partition (ksort_partition) by one CTA, then copy back in place
__global__ void __launch_bounds__(kExactThreads) k_exact_partition_one(double *keys, double *tmp, long long L,
                                                                       long long R, long long *Bl, long long *Gl,
                                                                       long long *out)
{
    __shared__ int sw[33];
    __shared__ long long sh[33];
    XPart pr = exact_partition_cta(keys, tmp, L, R, Bl, Gl, sw, sh);
    __syncthreads();
    for (long long p = L + threadIdx.x; p <= R; p += blockDim.x) keys[p] = tmp[p];
    if (threadIdx.x == 0) {
        out[0] = pr.piv;
        out[1] = pr.flag;
        out[2] = R - L;           // comparisons = m - 1
        out[3] = (long long)pr.moves;
    }
}

// ---- host ------------------------------------------------------------------------
static size_t al(size_t x) { return (x + 255) & ~size_t(255); }

ExactLayout exact_layout(long long n, bool with_log)
{
    ExactLayout L{};
    L.big_cap = (int)(n / kExactSmall + 4);
    L.small_cap = (int)(2 * (n / kExactSmall) + 8);
    L.log_cap = with_log ? (int)(n + 8) : 0;
    size_t off = 0;
    L.o_status = off; off = al(off + sizeof(XStatus));
    L.o_bad = off; off = al(off + 8);
    L.o_big[0] = off; off = al(off + sizeof(XSeg) * L.big_cap);
    L.o_big[1] = off; off = al(off + sizeof(XSeg) * L.big_cap);
    L.o_small = off; off = al(off + sizeof(XSeg) * L.small_cap);
    L.o_log = off; off = al(off + sizeof(XLog) * (size_t)L.log_cap);
    L.o_bl = off; off = al(off + sizeof(long long) * (size_t)n);
    L.o_gl = off; off = al(off + sizeof(long long) * (size_t)n);
    L.o_out = off; off = al(off + 64);
    L.o_tmp = off; off = al(off + sizeof(double) * (size_t)n);
    L.total = off;
    return L;
}

#define XK_CK(x)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            fprintf(stderr, "ksort(exact): %s failed: %s\n", #x, cudaGetErrorString(e_)); \
            return KS_CUDA_ERROR;                                                     \
        }                                                                             \
    } while (0)

// max_pending_ranges of sort_core.py:199-217, replayed on the logged tree
static unsigned long long replay_max_pending(long long n, const std::vector<XLog> &log)
{
    if (n < 2) return 0;
    std::unordered_map<unsigned long long, const XLog *> map;
    map.reserve(log.size() * 2 + 1);
    auto keyf = [](long long L, long long R) {
        return (unsigned long long)L * 0x9E3779B97F4A7C15ull ^ (unsigned long long)R;
    };
    for (const XLog &e : log) map[keyf(e.L, e.R)] = &e;
    std::vector<std::pair<long long, long long>> stack;
    stack.push_back({0, n - 1});
    unsigned long long maxp = 1;
    while (!stack.empty()) {
        auto [L, R] = stack.back();
        stack.pop_back();
        auto it = map.find(keyf(L, R));
        if (it == map.end() || it->second->L != L || it->second->R != R) return ~0ull;  // bug guard
        const XLog &e = *it->second;
        if (e.collapsed) {
            unsigned long long v = stack.size() + (unsigned long long)e.v;
            if (v > maxp) maxp = v;
            continue;
        }
        long long piv = e.v, lo_len = piv - L, hi_len = R - piv;
        if (lo_len <= hi_len) {
            if (hi_len >= 2) stack.push_back({piv + 1, R});
            if (lo_len >= 2) stack.push_back({L, piv - 1});
        } else {
            if (lo_len >= 2) stack.push_back({L, piv - 1});
            if (hi_len >= 2) stack.push_back({piv + 1, R});
        }
        if (stack.size() > maxp) maxp = stack.size();
    }
    return maxp;
}

int exact_sort(double *keys, long long n, void *ws, size_t ws_bytes, cudaStream_t stream, bool counts,
               ExactResult *res)
{
    ExactLayout L = exact_layout(n, counts);
    if (ws_bytes < L.total) return KS_WORKSPACE_SMALL;
    char *w = static_cast<char *>(ws);
    XStatus *xs = reinterpret_cast<XStatus *>(w + L.o_status);
    unsigned long long *bad = reinterpret_cast<unsigned long long *>(w + L.o_bad);
    XSeg *big[2] = {reinterpret_cast<XSeg *>(w + L.o_big[0]), reinterpret_cast<XSeg *>(w + L.o_big[1])};
    XSeg *small = reinterpret_cast<XSeg *>(w + L.o_small);
    XLog *log = counts ? reinterpret_cast<XLog *>(w + L.o_log) : nullptr;
    long long *Bl = reinterpret_cast<long long *>(w + L.o_bl);
    long long *Gl = reinterpret_cast<long long *>(w + L.o_gl);
    double *tmp = reinterpret_cast<double *>(w + L.o_tmp);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);

    XK_CK(cudaMemsetAsync(xs, 0, sizeof(XStatus), stream));
    XK_CK(cudaMemsetAsync(bad, 0xff, 8, stream));
    k_exact_gate<<<sms * 4, 256, 0, stream>>>(keys, n, bad);
    k_exact_init<<<1, 32, 0, stream>>>(n, big[0], small, xs);
    unsigned long long hbad = ~0ull;
    XStatus h{};
    XK_CK(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, stream));
    XK_CK(cudaMemcpyAsync(&h, xs, sizeof(XStatus), cudaMemcpyDeviceToHost, stream));
    XK_CK(cudaStreamSynchronize(stream));
    res->bad_index = hbad == ~0ull ? -1 : (long long)hbad;
    if (res->bad_index >= 0) return KS_OK;   // caller raises NonFiniteKeyError; nothing written

    // xs->nbig[0] counts the current level's big segments (table big[cur]);
    // k_exact_level appends the next level's to big[cur ^ 1] through nbig[1].
    // Levels are launched in batches with fixed grids (the kernels read their
    // segment counts on the device and exit at once when a level is empty):
    // one status read per kExactBatch levels instead of one per level.
    constexpr int kExactBatch = 16;
    int level = 0;
    int cur = 0;
    int syncs = 1;
    while (h.nbig[0] > 0 || h.nsmall > 0) {
        for (int b = 0; b < kExactBatch; ++b) {
            const double *src = (level & 1) ? tmp : keys;
            double *dst = (level & 1) ? keys : tmp;
            // small segments of this level live in `src` (they were produced by the previous level)
            k_exact_small<<<sms * 4, 128, 0, stream>>>(small, &xs->nsmall, src, keys, (level & 1) ? 0 : 1, xs, log,
                                                       L.log_cap);
            k_exact_advance<<<1, 32, 0, stream>>>(xs, 0);
            k_exact_level<<<sms * 2, kExactThreads, 0, stream>>>(big[cur], &xs->nbig[0], src, dst, keys,
                                                                 (level & 1) ? 1 : 0, Bl, Gl, big[cur ^ 1], small, xs,
                                                                 log, L.log_cap, L.big_cap, L.small_cap);
            k_exact_advance<<<1, 32, 0, stream>>>(xs, 1);
            cur ^= 1;
            ++level;
        }
        XK_CK(cudaGetLastError());
        XK_CK(cudaMemcpyAsync(&h, xs, sizeof(XStatus), cudaMemcpyDeviceToHost, stream));
        XK_CK(cudaStreamSynchronize(stream));
        ++syncs;
        if (h.overflow) return KS_CUDA_ERROR;
    }
    (void)syncs;
    level = h.levels;
    res->levels = level;
    res->comparisons = h.comparisons;
    res->moves = h.moves;
    res->max_pending = 0;
    if (counts && n >= 2) {
        std::vector<XLog> hl(h.nlog);
        if (h.nlog > 0) {
            XK_CK(cudaMemcpyAsync(hl.data(), log, sizeof(XLog) * h.nlog, cudaMemcpyDeviceToHost, stream));
            XK_CK(cudaStreamSynchronize(stream));
        }
        res->max_pending = replay_max_pending(n, hl);
        if (res->max_pending == ~0ull) return KS_CUDA_ERROR;
    }
    return KS_OK;
}

int exact_partition(double *keys, long long n, long long left, long long right, void *ws, size_t ws_bytes,
                    cudaStream_t stream, long long out[4], long long *bad_index)
{
    ExactLayout L = exact_layout(n, false);
    if (ws_bytes < L.total) return KS_WORKSPACE_SMALL;
    char *w = static_cast<char *>(ws);
    unsigned long long *bad = reinterpret_cast<unsigned long long *>(w + L.o_bad);
    long long *Bl = reinterpret_cast<long long *>(w + L.o_bl);
    long long *Gl = reinterpret_cast<long long *>(w + L.o_gl);
    long long *dout = reinterpret_cast<long long *>(w + L.o_out);
    double *tmp = reinterpret_cast<double *>(w + L.o_tmp);
    XK_CK(cudaMemsetAsync(bad, 0xff, 8, stream));
    // finiteness of the segment only (sort_core.py:161)
    k_exact_gate<<<64, 256, 0, stream>>>(keys + left, right - left + 1, bad);
    unsigned long long hbad = ~0ull;
    XK_CK(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, stream));
    XK_CK(cudaStreamSynchronize(stream));
    if (hbad != ~0ull) {
        *bad_index = left + (long long)hbad;
        return KS_OK;
    }
    *bad_index = -1;
    k_exact_partition_one<<<1, kExactThreads, 0, stream>>>(keys, tmp, left, right, Bl, Gl, dout);
    XK_CK(cudaGetLastError());
    XK_CK(cudaMemcpyAsync(out, dout, 4 * sizeof(long long), cudaMemcpyDeviceToHost, stream));
    XK_CK(cudaStreamSynchronize(stream));
    return KS_OK;
}

}  // namespace ks
