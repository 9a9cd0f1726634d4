// ks_internal.cuh -- device-side data structures and helpers shared by the
// K-sort engine's kernels (fast mode, exact mode, heap sort, utilities).
//
// Vocabulary follows the reference (sort_core.py): a *segment* is a subrange
// a[left..right] awaiting partition (the reference's worklist entry,
// sort_core.py:182-198); its *key* is its first element (sort_core.py:82);
// values with key <= v route right (sort_core.py:90).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <climits>

#include "../../include/ksort.h"

namespace ks {

// ---------------------------------------------------------------------------
// Fast-mode tunables.
// ---------------------------------------------------------------------------
#ifndef KS_PMAX
#define KS_PMAX 2047
#endif
constexpr int kPMax = KS_PMAX;        // max pivot candidates (first P keys) per global pass
constexpr int kPMaxPow2 = KS_PMAX + 1;
constexpr int kRowsMax = 2 * kPMax + 1;  // classes: gaps + equality runs (4095)
// KS_STAGED: the global pass's count and scatter kernels with 128-bit loads,
// branch-free classification and a shared-memory staged scatter (k_count2,
// k_scatter2); 0 selects the round-1 kernels (k_count, k_scatter).
#ifndef KS_STAGED
#define KS_STAGED 1
#endif
#ifndef KS_STAGE_MAX
#define KS_STAGE_MAX 16896   // keys per staged scatter tile: 10M keys = 592 chunks = 4 per SM
#endif
#ifndef KS_CLS
#define KS_CLS 1             // staged pass: the count kernel stores every key's class (2 B) for the scatter
#endif
#ifndef KS_CHECK
#define KS_CHECK 0           // self-check build: every fast sort verifies its output (sorted per segment,
                             // same multiset by bit-pattern sum and xor) and the staged tiles' bounds
#endif
#ifndef KS_STALL_GUARD
#define KS_STALL_GUARD 1     // stalled segments take pivots sampled across them (see Seg::stall)
#endif
#ifndef KS_SEG_TMA
#define KS_SEG_TMA 0         // segment sorters: the sorted segment leaves shared memory by one TMA bulk copy (measured: C0 +2.3%, C3 +5%; off)
#endif
#ifndef KS_SCAT_TMA
#define KS_SCAT_TMA 1        // staged scatter: each gap run leaves the tile by one TMA bulk copy
#endif
#ifndef KS_STAGED_PF
#define KS_STAGED_PF 0       // staged scatter: L2 prefetch of each chunk's destination runs
#endif
#ifndef KS_STAGE_ITEMS_PER_SM
#define KS_STAGE_ITEMS_PER_SM 4
#endif
#ifndef KS_LUTMAX
#if KS_STAGED
#define KS_LUTMAX 4096       // (the staged scatter's tile needs the shared memory)
#else
#define KS_LUTMAX 8192
#endif
#endif
constexpr int kLutMax = KS_LUTMAX;    // LUT buckets (pow2 >= 4*P)
constexpr int kPMaxLocal = 255;       // ... per local partition (P = len / kKeysPerPivot <= 64)
constexpr int kRowsMaxLocal = 2 * kPMaxLocal + 1;
constexpr int kLutMaxLocal = 2048;
#ifndef KS_KPP
#define KS_KPP 1024
#endif
constexpr int kKeysPerPivot = KS_KPP;   // P = len / 1024 (capped): gaps land in the segment sorters' range (C2 1M keys: 0.153 -> 0.131 ms)
#ifndef KS_LOCAL_KPP
#define KS_LOCAL_KPP 2048
#endif
constexpr int kKeysPerPivotLocal = KS_LOCAL_KPP;   // local partitions (children mostly for the small sorts)
// keys per count-matrix column (one count / scatter CTA work item): chosen per
// pass so that a one-segment pass gives every CTA of the pass grid one chunk;
// passes over several segments keep chunks <= kChunk (a segment's last chunk
// is short, so long chunks would unbalance them)
#ifndef KS_CHUNK
#define KS_CHUNK 16384
#endif
constexpr int kChunk = KS_CHUNK;
#ifndef KS_CHUNK_MIN
#define KS_CHUNK_MIN 2048
#endif
constexpr int kChunkMin = KS_CHUNK_MIN;
constexpr int kChunkAlign = 512;
constexpr int kChunkItemsMax = 2048;  // bound on the pass grid used for the chunk size
constexpr int kCountThreads = 512;
constexpr int kTile = 4096;           // keys staged in shared memory per scatter step
constexpr int kPassThreads = 512;     // threads of scatter CTAs (8 keys each per tile)
constexpr int kLocalMax = 131072;     // segments <= this are partitioned by one CTA (L2-resident)
constexpr int kInitLocalMax = 24576;  // ... for input arrays / batch segments (few items: use all SMs)
constexpr int kLocalBig = 32768;      // local segments above this are scheduled first (LPT)
constexpr int kUnitMax = 512;         // largest run one warp sorts in registers (16 per lane)
constexpr int kFillDirect = 16;       // equality runs up to this are written by the emitting thread
constexpr int kTinyGap = 16;          // gaps up to this are sorted by the emitting thread
// segment sorter: one CTA sorts a whole segment on chip (shared-memory copy ->
// interpolation buckets -> per-thread / per-warp bucket sorts).  Three size
// classes, each with its own CTA shape so that every thread holds 12..16 keys:
//   class 0: <= 2048 keys, 128 threads;  class 1: <= 6144, 512;  class 2: <= kSortMax, 1024 (in k_leaf)
constexpr int kSortClasses = 3;
#ifndef KS_SORTMAX
#define KS_SORTMAX 20480   // class 2 (the leaf kernel's own sorter, single buffer): measured 12K -> 20K: C0 -8.6%, C3 -4%
#endif
constexpr int kSortMax = KS_SORTMAX;
#ifndef KS_T0
#define KS_T0 128
#endif
#ifndef KS_LAM0
#define KS_LAM0 2
#endif
#ifndef KS_LAM1
#define KS_LAM1 2
#endif
#ifndef KS_CAP1
#define KS_CAP1 6144
#endif
#ifndef KS_CAP0
#define KS_CAP0 2048
#endif
// Size classes of the on-chip segment sorter: 0 (<= KS_CAP0 keys), 1 (<= KS_CAP1),
// 2 (<= kSortMax, inside the leaf kernel).  Class 3 is class 1's keys sorted by a
// single-buffer 256-thread sorter, class 4 class 0's keys by a single-buffer
// sorter (more sorters per SM; both chosen for large inputs).
__host__ __device__ constexpr int sort_cap(int c) { return (c == 0 || c == 4) ? KS_CAP0 : ((c == 1 || c == 3) ? KS_CAP1 : kSortMax); }
#ifndef KS_T1
#define KS_T1 512
#endif
#ifndef KS_T3
#define KS_T3 256
#endif
__host__ __device__ constexpr int sort_threads(int c) { return (c == 0 || c == 4) ? KS_T0 : (c == 1 ? KS_T1 : (c == 3 ? KS_T3 : 1024)); }
#ifndef KS_LAM2
#define KS_LAM2 2
#endif
__host__ __device__ constexpr int sort_lambda(int c) { return (c == 0 || c == 4) ? KS_LAM0 : ((c == 1 || c == 3) ? KS_LAM1 : KS_LAM2); }   // keys per bucket
__host__ __device__ __forceinline__ int sort_class(long long len) { return len <= sort_cap(0) ? 0 : (len <= sort_cap(1) ? 1 : 2); }
constexpr int kThreadSortMax = 16;                    // buckets up to this size: one thread, insertion sort
#ifndef KS_LOCAL_THREADS
#define KS_LOCAL_THREADS 1024
#endif
constexpr int kLocalThreads = KS_LOCAL_THREADS;   // CTA of the local partitioner
constexpr int kUnitWarps = 8;         // warps per CTA of the unit sorter

constexpr unsigned long long kNoIndex = ~0ull;

// phase ids (ks_status_t.phase_*)
enum Phase : int { kPhGate = 0, kPhPivots = 1, kPhCount = 2, kPhScan = 3, kPhScatter = 4, kPhPlan = 5,
                   kPhLeaf = 6, kPhOther = 7 };

__device__ __forceinline__ void add_bytes(struct DevStatus *st, int phase, unsigned long long b);

// Device-resident status / counters of one sort call (lives in the workspace).
struct DevStatus {
    unsigned long long bad_index;     // min non-finite index (atomicMin), kNoIndex if none
    unsigned int pos_zero;            // saw +0.0
    unsigned int neg_zero;            // saw -0.0
    int nseg[2];                      // segment counts of the two level tables
    int nunits;                       // warp work items (unit sorts, fills) of the current pass
    int unit_next;                    // ... their work counter (warps of the last sorter kernel claim them)
    int pad_units_;
    // on-chip work queues of the leaf kernel (local partitions, segment sorts)
    int lq_claim, lq_head;            // local queue: slots claimed by producers / taken by consumers
    int lqb_claim;                    // ... big local items (> kLocalBig), stored from the front (LPT)
    int sq_claim, sq_head;            // sort queue
    int pending;                      // local partitions queued or running (the only producers of leaf
                                      // items during a leaf launch; its CTAs may leave once it is zero)
    int nhb;                          // sorter hand-backs (skewed buckets), partitioned by the next leaf launch
    int npasses, nleaves;             // global passes and leaf launches run (device-side count)
    int published;                    // the final status went to the host (device loop: once per call)
    int done;                         // no level left (set by the last leaf launch's reset)
    int nsmall[2];                    // small-segment lists (size classes 0, 1), sorted after the leaf launch
    int small_next[2];                // their work counters
    int nchunks;                      // chunks of the current level
    long long mat_total;              // count-matrix entries of the current level
    int overflow;                     // a capacity bound was exceeded (bug guard)
    int no_item_pf;                   // small call: the sorters' per-item L2 prefetches are skipped
    int bad_arg;                      // segmented call: an offset pair outside [0, n_total] or decreasing
    int scan_next;                    // tile counter of the single-pass count-matrix scan
    int chunk;                        // keys per chunk of the current level
    unsigned long long bytes_moved;   // algorithmic bytes, all passes
    unsigned long long phase_bytes[8];  // per phase (ksort.h KS_FLAG_PROFILE numbering)
    unsigned long long keys_partitioned;
    unsigned long long keys_leaf;
    unsigned long long leaves;
    unsigned long long comparisons;   // exact mode op counts
    unsigned long long moves;
};

// One active segment of a global partition pass.
struct Seg {
    long long start;   // absolute index of the segment's first key (its K-sort key)
    long long len;
    long long mat_off; // first count-matrix entry (class-major rows x nch columns)
    int P;             // pivot candidates: the first P keys of the segment
    int k;             // distinct pivots among them
    int rows;          // 2P+1 matrix rows
    int nch;           // chunks (columns)
    int ch_off;        // first global chunk id
    int piv_off;       // offset into the pivot pool (P+1 slots: +inf sentinel)
    int lut_off;       // offset into the LUT pool (T int2 slots)
    int T;             // LUT buckets (1 = plain binary search)
    int src;           // local rounds: 0 keys / 1 tmp hold the segment
    int bnd;           // leaf items: all keys lie in [lo, scale] (bounds from the parent's pivots)
    double lo, scale;  // LUT transform t = clamp((v - lo) * scale, 0, T-1)
    int stall;         // the parent partition kept > 3/4 of its keys in this one gap (presorted,
                       // reversed, organ-pipe ...): pivots are sampled across the segment
    int spare_[3];
};

// Work item of the on-chip finishing pass.
//  unit: <= kUnitMax keys (a gap plus its pivot's equality run) sorted by one warp
//  fill: an equality run written with the pivot value, no read
enum ItemKind : int { kItemUnit = 0, kItemFill = 1 };
struct Item {
    long long start;
    double value;      // fill value (the pivot of an equality run)
    int len;
    short kind;        // ItemKind
    short src;         // 0: keys hold the data, 1: tmp holds the data
};

__device__ __forceinline__ void add_bytes(DevStatus *st, int phase, unsigned long long b)
{
    if (b == 0) return;
    atomicAdd(&st->phase_bytes[phase], b);
    atomicAdd(&st->bytes_moved, b);
}

__device__ __forceinline__ bool abort_requested(const DevStatus *st)
{
    // Non-finite key (sort_core.py:178), both signed zeros present (the fast
    // engine's output is bit-exact only when equal keys are bitwise equal), or
    // invalid batch offsets (nothing may be written through them).
    return st->bad_index != kNoIndex || (st->pos_zero && st->neg_zero) || st->bad_arg;
}

// Monotone LUT bucket of v: t(v) non-decreasing in v.  (v - lo) and the product
// round monotonically, the float->int conversion saturates (and maps NaN to 0),
// and scale is finite and > 0 whenever T > 1 (guarded where the table is
// built), so the bucket map is monotone on every finite key.
// Order-preserving unsigned image of a double (sign-magnitude -> two's order).
__device__ __forceinline__ unsigned long long ord_bits(double v)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// scale < 0 selects the bit-image map: t = (ord(v) - ord(lo)) * |scale|, used
// when the pivots are spread far more evenly in their bit image than in value
// (log-like data: a linear map would crowd them into a few buckets).  Both
// maps are monotone; keys below lo map to bucket 0.
__device__ __forceinline__ int lut_bucket(double v, double lo, double scale, int T)
{
    if (T <= 1) return 0;
    double t;
    if (scale >= 0.0) {
        t = (v - lo) * scale;
    } else {
        const unsigned long long ov = ord_bits(v), ol = ord_bits(lo);
        t = ov >= ol ? (double)(ov - ol) * -scale : -1.0;
    }
    const int x = __double2int_rz(t);
    return min(max(x, 0), T - 1);
}

// LUT transform for sorted distinct pivots piv[0..k): T buckets, linear or
// bit-image (negative scale), whichever places the pivots' quartiles closer
// to the buckets' quartiles; T = 1 (plain binary search) when no map works.
__device__ __forceinline__ void lut_transform(const double *piv, int k, int &T, double &scale)
{
    scale = 0.0;
    const double lo = piv[0], hi = piv[k > 0 ? k - 1 : 0];
    if (!(T > 1 && k >= 2 && hi > lo)) {
        T = 1;
        return;
    }
    const double sl = (double)T / (hi - lo);
    const double sb = (double)T / (double)(ord_bits(hi) - ord_bits(lo));
    const bool lin_ok = sl > 0.0 && !isinf(sl), bit_ok = sb > 0.0 && !isinf(sb);
    double err_l = 0.0, err_b = 0.0;
    const double span_b = (double)(ord_bits(hi) - ord_bits(lo));
    for (int q = 1; q <= 3; ++q) {
        const double x = piv[(k - 1) * q / 4];
        const double want = 0.25 * q;
        err_l += fabs((x - lo) / (hi - lo) - want);
        err_b += fabs((double)(ord_bits(x) - ord_bits(lo)) / span_b - want);
    }
    if (lin_ok && (!bit_ok || err_l <= err_b + 0.05)) scale = sl;   // (ties favour the linear map)
    else if (bit_ok) scale = -sb;
    else T = 1;
}

constexpr int kPivPad = 4;   // NaN slots after the k pivots (branch-free probes read up to piv[a+3])

// LUT entry: a | (b << 16) with a = #pivots in buckets < t, b = #pivots in
// buckets <= t (k <= kPMax < 65536).
__device__ __forceinline__ unsigned lut_pack(int a, int b) { return (unsigned)a | ((unsigned)b << 16); }

// Class of v against sorted distinct pivots piv[0..k) (piv[k..k+3] = NaN):
//   r = #pivots < v;  class = 2*r + (v == piv[r]).
// Even classes are gaps (open value intervals between pivots, i.e. the
// unfinished subtrees of the K-sort tree), odd classes are equality runs
// (the pivot and its copies: K-sort routes them right of the key, where they
// are already final).  The bucket's LUT entry gives a <= r <= b, and pivots
// past b are > v.  Most buckets hold no pivot (T >= 8P), so most keys are
// classified by one 4-byte shared load; buckets with <= 3 pivots are settled
// by four independent compares; crowded buckets fall back to binary search.
// The NaN sentinel compares false both ways, so +/-inf or NaN keys (rejected
// later by the finiteness gate) still classify in range.
__device__ __forceinline__ int classify(double v, const double *piv, const unsigned *lut, double lo,
                                        double scale, int T)
{
    const unsigned e = lut[lut_bucket(v, lo, scale, T)];
    int a = (int)(e & 0xffffu);
    const int b = (int)(e >> 16);
    if (a == b) return 2 * a;   // no pivot in the bucket: one shared-memory load in all
    const double p0 = piv[a];
    if (b - a == 1) return 2 * (a + (p0 < v ? 1 : 0)) + (p0 == v ? 1 : 0);
    if (b - a <= 3) {
        const double p1 = piv[a + 1], p2 = piv[a + 2], p3 = piv[a + 3];
        const int r = a + (p0 < v) + (p1 < v) + (p2 < v);
        const int eq = (p0 == v) | (p1 == v) | (p2 == v) | (p3 == v);
        return 2 * r + eq;
    }
    int hi = b;
    while (a < hi) {
        const int mid = (a + hi) >> 1;
        if (piv[mid] < v) a = mid + 1; else hi = mid;
    }
    return 2 * a + (piv[a] == v ? 1 : 0);
}

// Batched classify of U independent keys, written so that the U lookup
// chains overlap: all LUT loads, then the first two pivots of every bucket,
// then branch-free class arithmetic.  Buckets with more than two pivots
// (rare when T >= 4P) are finished by the general classify.
template <int U>
__device__ __forceinline__ void classify_batch(const double *v, int *c, const double *piv,
                                               const unsigned *lut, double lo, double scale, int T)
{
    unsigned e[U];
#pragma unroll
    for (int u = 0; u < U; ++u) e[u] = lut[lut_bucket(v[u], lo, scale, T)];
    double p0[U], p1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int a = (int)(e[u] & 0xffffu);
        p0[u] = piv[a];       // piv[k..k+3] are NaN sentinels: always in range
        p1[u] = piv[a + 1];
    }
    unsigned slow = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int a = (int)(e[u] & 0xffffu), d = (int)(e[u] >> 16) - a;
        const bool h0 = d > 0, h1 = d > 1;
        const int r = a + ((h0 && p0[u] < v[u]) ? 1 : 0) + ((h1 && p1[u] < v[u]) ? 1 : 0);
        const int eq = ((h0 && p0[u] == v[u]) || (h1 && p1[u] == v[u])) ? 1 : 0;
        c[u] = 2 * r + eq;
        slow |= (d > 2 ? 1u : 0u) << u;
    }
    if (slow) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if ((slow >> u) & 1u) c[u] = classify(v[u], piv, lut, lo, scale, T);
    }
}

// Asynchronous L2 prefetch of a byte range (TMA bulk prefetch; the range is
// widened to 16-byte alignment).  Used ahead of scattered 8-byte stores: a
// partial-sector store that misses L2 would otherwise wait for a DRAM fill.
__device__ __forceinline__ void l2_prefetch(const void *p, unsigned long long bytes)
{
    if (bytes == 0) return;
    const unsigned long long a0 = reinterpret_cast<unsigned long long>(p) & ~15ull;
    const unsigned long long a1 = (reinterpret_cast<unsigned long long>(p) + bytes + 15ull) & ~15ull;
    for (unsigned long long a = a0; a < a1; a += (1ull << 20)) {   // <= 1 MiB per instruction
        const unsigned long long e = a1 - a < (1ull << 20) ? a1 - a : (1ull << 20);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)e) : "memory");
    }
}

// Per-thread L2 prefetch of the 128-byte lines covering [p, p + bytes): a plain
// (non-uniform) instruction per line, for many small ranges at once -- the
// bulk form takes a uniform operand and serialises across the lanes of a warp.
#ifndef KS_PF_EVL
#define KS_PF_EVL 0   // 1: the scatter's destination prefetches are marked evict-last in L2
#endif
__device__ __forceinline__ void l2_prefetch_lines(const void *p, unsigned long long bytes)
{
    if (bytes == 0) return;
    const unsigned long long a0 = reinterpret_cast<unsigned long long>(p) & ~127ull;
    const unsigned long long a1 = reinterpret_cast<unsigned long long>(p) + bytes;
    for (unsigned long long a = a0; a < a1; a += 128) {
#if KS_PF_EVL
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a) : "memory");
#else
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a) : "memory");
#endif
    }
}

__host__ __device__ __forceinline__ long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

__host__ __device__ __forceinline__ int next_pow2(int x)
{
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Block-wide exclusive scan of one long long per thread (blockDim.x <= 1024,
// multiple of 32).  `sh` needs 33 slots.  Returns the exclusive prefix and the
// block total through *total.
__device__ __forceinline__ long long block_exclusive_scan(long long x, long long *sh, long long *total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sh[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        long long w = lane < nw ? sh[lane] : 0;
        long long winc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, winc, o);
            if (lane >= o) winc += y;
        }
        if (lane < nw) sh[lane] = winc - w;   // exclusive warp offsets
        if (lane == 31) sh[32] = winc;        // lanes >= nw add 0: lane 31 holds the total
    }
    __syncthreads();
    long long res = sh[wid] + inc - x;
    if (total) *total = sh[32];
    __syncthreads();
    return res;
}

// 32-bit variant (same contract; `sh` needs 33 slots).
__device__ __forceinline__ unsigned block_exclusive_scan_u32(unsigned x, unsigned *sh, unsigned *total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sh[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const unsigned w = lane < nw ? sh[lane] : 0u;
        unsigned winc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, winc, o);
            if (lane >= o) winc += y;
        }
        if (lane < nw) sh[lane] = winc - w;
        if (lane == 31) sh[32] = winc;
    }
    __syncthreads();
    const unsigned res = sh[wid] + inc - x;
    if (total) *total = sh[32];
    __syncthreads();
    return res;
}

}  // namespace ks
