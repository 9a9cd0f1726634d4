// ks_fast.cu -- fast-mode K-sort engine: segmented multi-level K-sort passes
// over HBM plus an on-chip finishing pass.
//
// What one global pass does:
//   For every active segment, the K-sort recursion tree below the segment's
//   key is the binary search tree obtained by inserting the segment's keys in
//   order (key = first element, sort_core.py:82; key <= v routes right,
//   sort_core.py:90).  The first P keys of the segment are exactly the top
//   nodes of that tree, so classifying every key against them (binary search
//   over the P sorted pivots) performs the tree's top levels for all keys in
//   one read + one write of HBM.  Keys equal to a pivot are retired as a fat
//   pivot (K-sort routes them right of the key, where they are final).
//   Remaining gaps are the unfinished subtrees: gaps <= S go to the on-chip
//   finishing pass, larger gaps become the next pass's segments.
//
// Kernels per pass: seg_prep -> seg_offsets -> pivots -> count -> scan (3) ->
// scatter -> plan; then local partition rounds (one CTA per segment) and one
// warp-per-unit finishing launch.  No key crosses to the host; the host reads
// one small status block per pass to decide whether another pass is needed.
#include <cooperative_groups.h>
#include <algorithm>
#include <atomic>
#include <cfloat>
#include <cstdio>
#include <memory>
#include <mutex>
#include <type_traits>
#include <vector>

#include "ks_host.h"
#include "ks_internal.cuh"
#include "ks_sortnet.cuh"

namespace ks {
namespace cg = cooperative_groups;

#ifdef KS_TRACE
// optional phase-cycle instrumentation (build with KS_TRACE=1), read via ks_trace_read
__device__ unsigned long long g_trace[32];
#define KS_TR_DECL long long tr_t0 = clock64()
#define KS_TR(slot)                                                                  \
    do {                                                                             \
        if (threadIdx.x == 0) {                                                      \
            long long t1_ = clock64();                                               \
            atomicAdd(&g_trace[slot], (unsigned long long)(t1_ - tr_t0));            \
            tr_t0 = t1_;                                                             \
        }                                                                            \
    } while (0)
#else
#define KS_TR_DECL
#define KS_TR(slot)
#endif

#ifdef KS_TIMELINE
// optional per-item timeline (build with -DKS_TIMELINE): one record per leaf item
// {smid | kernel << 8 | kind << 16, len, t0, t1} (globaltimer ns), read via ks_timeline_read
constexpr int kTlCap = 1 << 17;
__device__ unsigned long long g_tl[4 * kTlCap];
__device__ unsigned g_tl_n;
__device__ __forceinline__ unsigned long long tl_now()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void tl_rec(int kernel, int kind, long long len, unsigned long long t0)
{
    const unsigned long long t1 = tl_now();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const unsigned i = atomicAdd(&g_tl_n, 1u);
    if (i < (unsigned)kTlCap) {
        g_tl[4 * i] = smid | ((unsigned long long)kernel << 8) | ((unsigned long long)(kind + 1) << 16);
        g_tl[4 * i + 1] = (unsigned long long)len;
        g_tl[4 * i + 2] = t0;
        g_tl[4 * i + 3] = t1;
    }
}
#define KS_TL_T0 const unsigned long long tl_t0_ = tl_now()
#define KS_TL(kernel, kind, len) \
    do {                         \
        if (threadIdx.x == 0) tl_rec(kernel, kind, len, tl_t0_); \
    } while (0)
#else
#define KS_TL_T0
#define KS_TL(kernel, kind, len)
#endif

// build-time variants (experiments; defaults are the measured best)
#ifndef KS_BATCH
#define KS_BATCH 0        // batched (overlapped) classify in the count / scatter loops: 1 = all U keys at once
#endif                    // (measured: no gain, spills at 40 registers), 2 = groups of KS_BATCH_G keys
#ifndef KS_SRC_CS
#define KS_SRC_CS 1       // 1: the scatter's source loads are evict-first (ld.global.cs): C0 -3..5%
#endif
#ifndef KS_SPREAD
#define KS_SPREAD 1
#endif
#ifndef KS_SRC_PF
#define KS_SRC_PF 0        // 1: staged scatter prefetches the next tile's keys and classes into L2 during the copy-out
#endif
#ifndef KS_PF_MIN_N
#define KS_PF_MIN_N 2500000   // scatter destinations are prefetched into L2 for calls of at least this many keys
#endif                        // (measured: 1M/2M keys -9%/-6% without, 3M..10M +6..11% without)
#ifndef KS_ITEM_PF_MIN_N
#define KS_ITEM_PF_MIN_N 2500000   // the small-segment sorters prefetch their next item into L2 for calls of at
#endif                             // least this many keys (measured without: 1M -9%, 2M -6%; 3M..10M +6..11%)
#ifndef KS_SBATCH
#define KS_SBATCH 0       // scatter: classify in groups of this many keys (LUT loads, pivot loads, atomics, stores)
#endif
#ifndef KS_SCAT_MINB
#define KS_SCAT_MINB KS_PASS_MINB   // resident scatter CTAs per SM asked (2: 64 registers for the grouped classify)
#endif
#ifndef KS_PF_EARLY
#define KS_PF_EARLY 0     // 1: scatter CTAs issue their destination prefetches before copying the pivot tables
#endif
#ifndef KS_BATCH_G
#define KS_BATCH_G 4
#endif
#ifndef KS_SCATTER_EXP
#define KS_SCATTER_EXP 0
#endif
#ifndef KS_PREFETCH
#define KS_PREFETCH 1     // L2 prefetch of each chunk's scatter destinations
#endif
#ifndef KS_SCAN3
#define KS_SCAN3 0        // 1: three-kernel count-matrix scan instead of the look-back scan
#endif
#ifndef KS_PDL
#define KS_PDL 1          // programmatic dependent launch between the engine's kernels
#endif
#ifndef KS_SEGOFF_PF
#define KS_SEGOFF_PF 0    // L2 prefetch of the count matrix and offsets at the start of a pass (measured: off is better, C2 -7%, C5 -5%)
#endif
#ifndef KS_PDL_HEAVY
#define KS_PDL_HEAVY 0    // PDL also into the persistent grids (count, scatter, leaf, segment sorts)
#endif
#ifndef KS_RANK_LEAF
#define KS_RANK_LEAF 0    // 1: in-bucket ranks per key instead of per-bucket networks
#endif
#ifndef KS_GRAPH
#define KS_GRAPH 1        // replay the speculative schedule as a cached CUDA graph
#endif
#ifndef KS_MID_RANK
#define KS_MID_RANK 1     // 5..16-key buckets of the segment sorter: half-warp ranks instead of insertion sorts
#endif
#ifndef KS_FUSED_HIST
#define KS_FUSED_HIST 1   // bounded leaf items: bucket histogram built while loading (no min / max pass)
#endif
#ifndef KS_SEG_FEED
#define KS_SEG_FEED 1     // small-segment sorters: next item claimed / fetched / prefetched without stalls
#endif
#ifndef KS_SINGLE_MIN_N
#define KS_SINGLE_MIN_N 5000000   // class-1 lists of inputs this large go to the single-buffer sorter (class 3), chained, draining class 0 (smaller single arrays: k_small)
#endif
#ifndef KS_MINB4
#define KS_MINB4 8        // class 4 = class 0's keys by a single-buffer sorter (large inputs)
#endif
#ifndef KS_MINB3
#define KS_MINB3 3
#endif
#ifndef KS_SINGLE2
#define KS_SINGLE2 1      // the leaf's class-2 sorter with a single shared buffer (room for 20K-key segments)
#endif
#ifndef KS_PLAN_FORK
#define KS_PLAN_FORK 2    // the global plan runs concurrently with the scatter (data writes deferred to the finish
#endif                    // pass): 1 forked onto a side stream, 2 chained (PDL) into the scatter's tail
#ifndef KS_SORT_FORK
#define KS_SORT_FORK 1    // class-0 and class-1 list sorters run concurrently (side stream)
#endif
#ifndef KS_FORK_ROOM
#define KS_FORK_ROOM 0    // scatter CTAs given up for the forked plan's CTAs (measured 16: C0 -0.2%, C3 +3%)
#endif
#ifndef KS_MINB0
#define KS_MINB0 5        // resident CTAs per SM asked for the class-0 small-segment sorter
#endif
#ifndef KS_MINB1
#define KS_MINB1 2        // resident CTAs per SM asked for the 512-thread small-segment sorter
#endif
#ifndef KS_LEAF_CHAIN
#define KS_LEAF_CHAIN 1   // the list sorters start (PDL) on the SMs the leaf kernel's CTAs leave
#endif
#ifndef KS_MAPPED_STATUS
#define KS_MAPPED_STATUS 1   // the status block reaches the host through mapped memory (polled)
#endif
#ifndef KS_DEVICE_LOOP
#define KS_DEVICE_LOOP 1   // graph path: the remaining levels run in a conditional WHILE node (no host round
#endif                     // trip) -- 1: for keys whose sorts needed it before, 2: always, 0: never
#ifndef KS_DRAIN0
#define KS_DRAIN0 1       // one large array: the class-1 list sorters drain the class-0 list in the same launch
#endif
#ifndef KS_LU1024
#define KS_LU1024 8       // segment sorter loads in flight per thread at 1024 threads (the leaf kernel's class 2; 4: C0 +0.8%)
#endif
#ifndef KS_PASS_MINB
#define KS_PASS_MINB 3    // min resident CTAs per SM requested for count / scatter
#endif

// Every kernel of the fast engine starts here: wait until the preceding grid in
// the stream has completed (its writes visible), then let the next grid's CTAs
// be scheduled while this one runs (they wait at the same point).  This hides
// the launch gap between the pipeline's dependent kernels.
#if KS_PDL
#define KS_PDL_ENTRY()                                            \
    do {                                                          \
        asm volatile("griddepcontrol.wait;" ::: "memory");        \
        asm volatile("griddepcontrol.launch_dependents;" :::);    \
    } while (0)
#else
#define KS_PDL_ENTRY() \
    do {               \
    } while (0)
#endif

constexpr int kStageMax = KS_STAGE_MAX;   // keys per staged scatter tile (= chunk cap when staged)
constexpr int kScat2Threads = 1024;
constexpr int kCount2Threads = 512;
constexpr int kScanBlock = 4096;   // count-matrix entries per scan CTA (512 thr x 8)
constexpr int kScanThreads = 512;

// ---------------------------------------------------------------------------
// work lists
// ---------------------------------------------------------------------------
__device__ __forceinline__ Item make_item(long long start, long long len, int kind, int src)
{
    Item it{};
    it.start = start;
    it.len = (int)len;
    it.kind = (short)kind;
    it.src = (short)src;
    return it;
}

__device__ __forceinline__ Seg make_seg(long long start, long long len, int src)
{
    Seg g{};
    g.start = start;
    g.len = len;
    g.src = src;
    return g;
}

// leaf item with the value range of its keys (blo <= key <= bhi; +-inf: unknown)
__device__ __forceinline__ Seg make_bseg(long long start, long long len, int src, double blo, double bhi)
{
    Seg g = make_seg(start, len, src);
    g.bnd = (isfinite(blo) && isfinite(bhi)) ? 1 : 0;
    g.lo = blo;
    g.scale = bhi;
    return g;
}
// a queued leaf item as published (bounds included)
__device__ __forceinline__ Seg load_item(const Seg *q)
{
    Seg g = make_seg(__ldcg(&q->start), __ldcg(&q->len), __ldcg(&q->src));
    g.bnd = __ldcg(&q->bnd);
    g.lo = __ldcg(&q->lo);
    g.scale = __ldcg(&q->scale);
    g.stall = __ldcg(&q->stall);
    return g;
}

// Work queues of the leaf kernel.  Producers (the global plan, the local
// partitioner, the segment sorter's hand-back) raise `pending`, claim a slot,
// write the item and publish it by storing the tag (epoch << 32 | claim) into
// the slot's ready word; consumers claim in order and wait for that tag.
// The queues are circular: items still queued are disjoint ranges of more
// than kUnitMax keys (a parent leaves the queue before its children enter),
// so cap >= n / (kUnitMax + 1) + (CTAs in flight) never overwrites a slot
// that has not been read.
struct LeafQ {
    Seg *lq;          // local partitions (kSortMax < len <= kLocalMax)
    unsigned long long *lq_ready;
    int lcap;
    Seg *sq;          // segment sorts (kUnitMax < len <= kSortMax)
    unsigned long long *sq_ready;
    int scap;
    int epoch;        // leaf launch these items belong to
    Seg *small[2];    // segments of size classes 0 / 1: sorted by their own CTA shapes after the leaf launch
    int small_cap[2];
    Seg *hb;          // sorter hand-backs: partitioned by the next leaf launch (its local queue)
    int hb_cap;
    unsigned *seq;    // call sequence word (CallSeq.seq): part of every ready tag
};

// Ready tags are (call sequence, leaf launch, claim index): a slot's word from an
// earlier call or launch never matches, so the words need no clearing per call
// (the init kernel clears them only for a fresh or re-laid-out workspace and
// when the 27-bit sequence wraps).
struct CallSeq {
    unsigned seq;
    unsigned pad_;
    unsigned long long magic;   // workspace layout the ready words belong to
};
constexpr int kTagIdxBits = 25, kTagEpBits = 12;
constexpr unsigned kSeqMask = (1u << (64 - kTagIdxBits - kTagEpBits)) - 1u;
__device__ __forceinline__ unsigned long long q_epoch(const LeafQ &Q)
{
    const unsigned s = *reinterpret_cast<const volatile unsigned *>(Q.seq);
    return ((unsigned long long)s << kTagEpBits) | (unsigned)(Q.epoch & ((1 << kTagEpBits) - 1));
}

// A skewed bucket the on-chip sorter cannot finish goes back to the first-key
// partitioner in the NEXT leaf launch: no queue item appears during a launch
// except from a local partition, so CTAs may leave once none is queued or running.
__device__ __forceinline__ void hb_push(const LeafQ &Q, const Seg &g, DevStatus *st)
{
    const int i = atomicAdd(&st->nhb, 1);
    if (i < Q.hb_cap) Q.hb[i] = g; else st->overflow = 6;
}

// small segments (<= sort_cap(1) keys) go to the size-class lists
__device__ __forceinline__ void small_push(const LeafQ &Q, const Seg &g, DevStatus *st)
{
    const int c = g.len <= sort_cap(0) ? 0 : 1;
    const int i = atomicAdd(&st->nsmall[c], 1);
    if (i < Q.small_cap[c]) (c ? Q.small[1] : Q.small[0])[i] = g; else st->overflow = 5;
}

__device__ __forceinline__ unsigned long long q_tag(unsigned long long ep, int idx)
{
    return (ep << kTagIdxBits) | (unsigned)idx;
}

__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire_s32(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// write the item, then release its tag (the item is visible before the tag)
__device__ __forceinline__ void q_publish(Seg *q, unsigned long long *ready, int cap, int idx, const Seg &g,
                                          unsigned long long epoch)
{
    const int slot = idx % cap;
    q[slot] = g;
    st_release_u64(&ready[slot], q_tag(epoch, idx));
}

// The local queue holds only the global plan's items (all published before
// the leaf launch starts).  Items made during the launch -- segments to sort,
// local children still too large to sort on chip, the sorter's hand-backs --
// go to the sort queue, each tagged with its kind.
constexpr int kItemLocal = 0, kItemSort = 1;
__device__ __forceinline__ Seg with_kind(Seg g, int kind)
{
    g.k = kind;
    return g;
}

// single-item push to the sort queue (pending is raised before the slot can be claimed)
__device__ __forceinline__ void q_push1(bool local, const LeafQ &Q, const Seg &g, DevStatus *st)
{
    if (!local && g.len <= sort_cap(1)) {
        small_push(Q, g, st);
        return;
    }
    if (local) atomicAdd(&st->pending, 1);
    q_publish(Q.sq, Q.sq_ready, Q.scap, atomicAdd(&st->sq_claim, 1), with_kind(g, local ? kItemLocal : kItemSort),
              q_epoch(Q));
}

// Initial routing of one array (or one segment of a batch).
struct InitLists {
    Seg *gsegs;
    LeafQ Q;
    Item *units;
    int seg_cap, unit_cap;
};

// > kInitLocalMax keys -> global pass list, kSortMax < len <= kInitLocalMax ->
// local queue, kUnitMax < len <= kSortMax -> sort queue, 2..kUnitMax -> unit.
__device__ __forceinline__ void route_initial(long long a, long long len, const InitLists &Lst, DevStatus *st)
{
    if (len > kInitLocalMax) {   // (a lone large array is partitioned by all SMs, not by one CTA)
        int i = atomicAdd(&st->nseg[0], 1);
        if (i < Lst.seg_cap) Lst.gsegs[i] = make_seg(a, len, 0); else st->overflow = 1;
    } else if (len > kUnitMax) {
        q_push1(len > kSortMax, Lst.Q, make_seg(a, len, 0), st);
    } else if (len >= 2) {
        int i = atomicAdd(&st->nunits, 1);
        if (i < Lst.unit_cap) Lst.units[i] = make_item(a, len, kItemUnit, 0); else st->overflow = 1;
        atomicAdd(&st->keys_leaf, (unsigned long long)len);
        atomicAdd(&st->leaves, 1ull);
        add_bytes(st, kPhLeaf, 16ull * (unsigned long long)len);
    }
}

// Single array: reset the status block and route the whole array (one launch).
// One CTA, before any queue item of the call is published: next call sequence
// number; ready words cleared when the workspace is fresh / re-laid-out or the
// sequence wraps.
__device__ void seq_advance(const LeafQ &Q, unsigned long long magic)
{
    __shared__ int s_clear;
    if (threadIdx.x == 0) {
        CallSeq *c = reinterpret_cast<CallSeq *>(Q.seq);
        unsigned sq = (c->seq + 1u) & kSeqMask;
        s_clear = (c->magic != magic || sq == 0u) ? 1 : 0;
        if (sq == 0u) sq = 1u;
        c->seq = sq;
        c->magic = magic;
    }
    __syncthreads();
    if (s_clear)
        for (int i = threadIdx.x; i < Q.scap; i += blockDim.x) Q.sq_ready[i] = 0ull;
    __syncthreads();
}

__global__ void k_init_single(long long n, InitLists Lst, DevStatus *st, unsigned long long magic)
{
    KS_PDL_ENTRY();
    seq_advance(Lst.Q, magic);
    static_assert(sizeof(DevStatus) % 8 == 0, "status is cleared in 8-byte words");
    unsigned long long *w = reinterpret_cast<unsigned long long *>(st);
    for (int i = threadIdx.x; i < (int)(sizeof(DevStatus) / 8); i += blockDim.x) w[i] = 0ull;
    __syncthreads();
    if (threadIdx.x != 0) return;
    st->bad_index = kNoIndex;
    st->no_item_pf = n < KS_ITEM_PF_MIN_N ? 1 : 0;
    route_initial(0, n, Lst, st);
}

// Offsets are validated here, before anything is written: a segment with
// off[s] < 0, off[s+1] < off[s] or off[s+1] > n_total raises bad_arg, which
// every writing kernel honours (abort_requested) and the call returns
// KS_BAD_ARG.  Per-pair checks suffice: consecutive pairs share their ends,
// so valid pairs are disjoint ranges inside the buffer.
__device__ __forceinline__ bool seg_ok(long long a, long long b, long long n_total)
{
    return 0 <= a && a <= b && b <= n_total;
}

__global__ void k_init_segmented(const long long *off, long long nseg0, long long n_total, InitLists Lst,
                                 DevStatus *st)
{
    KS_PDL_ENTRY();
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nseg0;
         s += (long long)gridDim.x * blockDim.x) {
        const long long a = off[s], b = off[s + 1];
        if (!seg_ok(a, b, n_total)) {
            atomicOr(reinterpret_cast<unsigned *>(&st->bad_arg), 1u);
            continue;
        }
        route_initial(a, b - a, Lst, st);
    }
}

__device__ __forceinline__ void gate_one(double v, long long idx, long long &bad, unsigned &pz, unsigned &nz)
{
    if (!isfinite(v)) bad = min(bad, idx);
    if (v == 0.0) {
        if (signbit(v)) nz = 1; else pz = 1;
    }
}

__device__ __forceinline__ void gate_flush(long long bad, unsigned pz, unsigned nz, DevStatus *st)
{
    if (bad != LLONG_MAX) atomicMin(&st->bad_index, (unsigned long long)bad);
    if (pz) atomicOr(&st->pos_zero, 1u);
    if (nz) atomicOr(&st->neg_zero, 1u);
}

// Finiteness gate (sort_core.py:50-59) for keys not covered by the level-0
// count pass: segments of <= kInitLocalMax keys (they never see a global pass).
__global__ void k_gate_segments(const double *keys, const long long *off, long long nseg0, long long n_single,
                                long long n_total, DevStatus *st)
{
    KS_PDL_ENTRY();
    long long bad = LLONG_MAX;
    unsigned pz = 0, nz = 0;
    long long checked = 0;
    if (off == nullptr) {
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_single;
             i += (long long)gridDim.x * blockDim.x) {
            gate_one(keys[i], i, bad, pz, nz);
            ++checked;
        }
    } else {
        for (long long s = blockIdx.x; s < nseg0; s += gridDim.x) {
            long long a = off[s], b = off[s + 1];
            if (!seg_ok(a, b, n_total)) continue;  // (flagged by k_init_segmented)
            if (b - a > kInitLocalMax) continue;  // covered by the level-0 count pass
            for (long long i = a + threadIdx.x; i < b; i += blockDim.x) {
                gate_one(keys[i], i, bad, pz, nz);
                ++checked;
            }
        }
    }
    if (checked) add_bytes(st, kPhGate, 8ull * (unsigned long long)checked);
    gate_flush(bad, pz, nz, st);
}

// ---------------------------------------------------------------------------
// pivots: the first P keys of a segment are the top of its K-sort tree.
// Sorted by one warp in registers, de-duplicated (equal keys are one node:
// the fat pivot), NaN sentinels after them, plus the bucket LUT built by a
// histogram of pivot buckets and an exclusive scan (a = #pivots in buckets
// < t, b = #pivots in buckets <= t).
// ---------------------------------------------------------------------------
template <int N>
struct PivotScratch {
    double sp[N];
    double sq[N];
    long long sh[33];
    int sk;
};

// rank of the o-th output of merge(A = s[g0, g0+size), B = s[g0+size, g0+2size)), A first on ties
__device__ __forceinline__ double merge_pick(const double *s, int g0, int size, int d)
{
    const double *A = s + g0, *B = s + g0 + size;
    int lo = d - size > 0 ? d - size : 0, hi = d < size ? d : size;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (!(B[d - 1 - mid] < A[mid])) lo = mid + 1; else hi = mid;
    }
    const int a = lo, b = d - lo;
    if (b >= size) return A[a];
    if (a >= size) return B[b];
    return (B[b] < A[a]) ? B[b] : A[a];
}

// Stride of the pivot sample: 1 (K-sort's first P keys) unless the segment stalled.
__device__ __forceinline__ long long pivot_stride(int stall, long long len, int P)
{
    return (KS_STALL_GUARD && stall && P > 0 && len / P > 1) ? len / P : 1;
}

template <int N>
__device__ void build_pivots(const double *seg, int P, int Treq, double *piv, unsigned *lut, PivotScratch<N> &W,
                             int &k_out, int &T_out, double &lo_out, double &scale_out, long long stride = 1)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int NP = next_pow2(P) < 32 ? 32 : next_pow2(P);
    __syncthreads();
    // each warp sorts a 32-key run in registers (shuffle network), then
    // merge-path passes with one output per thread
    for (int w = wid; w * 32 < NP; w += nw) {
        const int i = w * 32 + lane;
        double x[1] = {i < P ? __ldcg(seg + i * stride) : CUDART_INF};
        warp_bitonic_sort<1>(x);
        W.sp[i] = x[0];
    }
    __syncthreads();
    double *cur = W.sp, *nxt = W.sq;
    for (int size = 32; size < NP; size <<= 1) {
        for (int o = threadIdx.x; o < NP; o += blockDim.x) {
            const int g0 = o & ~(2 * size - 1);
            nxt[o] = merge_pick(cur, g0, size, o - g0);
        }
        __syncthreads();
        double *t = cur;
        cur = nxt;
        nxt = t;
    }
    const double *sp = cur;
    long long carry = 0;
    for (int base = 0; base < P; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int keep = (i < P && (i == 0 || sp[i] != sp[i - 1])) ? 1 : 0;
        long long tot;
        const long long pos = block_exclusive_scan(keep, W.sh, &tot);
        if (keep) piv[carry + pos] = sp[i];
        carry += tot;
    }
    const int k = (int)carry;
    if (threadIdx.x < kPivPad) piv[k + threadIdx.x] = CUDART_NAN;
    __syncthreads();
    int T = Treq;
    const double lo = piv[0];
    double scale;
    lut_transform(piv, k, T, scale);
    for (int t = threadIdx.x; t < T; t += blockDim.x) lut[t] = 0u;
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) atomicAdd(&lut[lut_bucket(piv[j], lo, scale, T)], 1u);
    __syncthreads();
    {   // exclusive scan over T buckets: warp w owns a contiguous slice, scanned 32 at a time
        const int per_w = (T + nw - 1) / nw;
        const int b0 = wid * per_w, b1 = min(T, b0 + per_w);
        int run = 0;
        for (int base = b0; base < b1; base += 32) {
            const int t = base + lane;
            const int c = t < b1 ? (int)lut[t] : 0;
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (t < b1) lut[t] = (unsigned)(run + inc - c);   // exclusive within the warp's slice
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) W.sh[wid] = run;
        __syncthreads();
        int wbase = 0;
        for (int q = 0; q < wid; ++q) wbase += (int)W.sh[q];
        for (int base = b0; base < b1; base += 32) {   // warp-uniform trip count
            const int t = base + lane;
            int a = 0, nxt = 0;
            if (t < b1) {
                a = wbase + (int)lut[t];
                nxt = (t + 1 < b1) ? wbase + (int)lut[t + 1] : wbase + run;
            }
            __syncwarp();   // all reads of this row before any lane overwrites its entry
            if (t < b1) lut[t] = lut_pack(a, nxt);
            __syncwarp();
        }
    }
    __syncthreads();
    k_out = k;
    T_out = T;
    lo_out = lo;
    scale_out = scale;
}

__host__ __device__ __forceinline__ int pivots_for(long long len, int pmax, int keys_per_pivot = kKeysPerPivot)
{
    long long P = cdiv(len, keys_per_pivot);
    if (P > pmax) P = pmax;
    if (P < 1) P = 1;
    return (int)P;
}

__host__ __device__ __forceinline__ int lut_for(int P, int tmax)
{
    int T = P >= 2 ? next_pow2(8 * P) : 1;
    return T > tmax ? tmax : T;
}

// ---------------------------------------------------------------------------
// global pass bookkeeping
// ---------------------------------------------------------------------------
// Count-matrix layout of one segment: one row per gap class j (0..P) holding
// its per-chunk counts, followed by ONE entry with the total of equality run j
// (equality runs are filled, never scattered: only their sizes matter).  A flat
// scan of the rows therefore yields, in class order, each gap chunk's
// destination and each equality run's start.
__host__ __device__ __forceinline__ long long mat_row(const Seg &g) { return (long long)g.nch + 1; }
__host__ __device__ __forceinline__ long long mat_entries(const Seg &g) { return ((long long)g.P + 1) * mat_row(g); }
__host__ __device__ __forceinline__ long long mat_gap(const Seg &g, int j, int chunk)
{
    return g.mat_off + (long long)j * mat_row(g) + chunk;
}
__host__ __device__ __forceinline__ long long mat_eq(const Seg &g, int j) { return g.mat_off + (long long)j * mat_row(g) + g.nch; }

// One CTA: per-segment pass shape (P, rows, chunks, LUT size) and exclusive
// scans over segments for pool offsets and the count-matrix layout; then an
// L2 prefetch of this level's count matrix and offsets (they are written with
// scattered 4- and 8-byte stores).
__device__ void seg_offsets_body(Seg *segs, int ns, DevStatus *st, long long mat_cap, int ch_cap, int piv_cap,
                                 int lut_cap, const unsigned *mat, const long long *moff, unsigned long long *tstat,
                                 int *nseg_next, int items, long long *sh)
{
    // chunk size of this pass (see kChunk)
    long long total = 0;
    for (int base = 0; base < ns; base += blockDim.x) {
        const int s = base + threadIdx.x;
        long long t;
        block_exclusive_scan(s < ns ? segs[s].len : 0ll, sh, &t);
        total += t;
    }
    long long chunk = cdiv(cdiv(total, (long long)min(items, kChunkItemsMax)), (long long)kChunkAlign) * kChunkAlign;
    if (ns > 1 && chunk > kChunk) chunk = kChunk;
    if (KS_STAGED && chunk > kStageMax) chunk = kStageMax;   // one chunk = one staged scatter tile
    if (chunk < kChunkMin) chunk = kChunkMin;
    long long c_piv = 0, c_lut = 0, c_mat = 0, c_ch = 0;
    for (int base = 0; base < ns; base += blockDim.x) {
        int s = base + threadIdx.x;
        Seg g{};
        if (s < ns) {
            g = segs[s];
            g.P = pivots_for(g.len, kPMax);
            g.rows = 2 * g.P + 1;
            g.nch = (int)cdiv(g.len, chunk);
            g.T = lut_for(g.P, kLutMax);
        }
        const bool in = s < ns;
        long long tp, tl, tm, tc;
        long long xp = block_exclusive_scan(in ? g.P + 1 : 0, sh, &tp);
        long long xl = block_exclusive_scan(in ? g.T : 0, sh, &tl);
        long long xm = block_exclusive_scan(in ? mat_entries(g) : 0, sh, &tm);
        long long xc = block_exclusive_scan(in ? g.nch : 0, sh, &tc);
        if (in) {
            g.piv_off = (int)(c_piv + xp);
            g.lut_off = (int)(c_lut + xl);
            g.mat_off = c_mat + xm;
            g.ch_off = (int)(c_ch + xc);
            segs[s] = g;
        }
        c_piv += tp;
        c_lut += tl;
        c_mat += tm;
        c_ch += tc;
    }
    if (threadIdx.x == 0) {
        if (ns > 0) ++st->npasses;
        st->nchunks = (int)c_ch;
        st->chunk = (int)chunk;
        st->mat_total = c_mat;
        add_bytes(st, kPhScan, 16ull * (unsigned long long)c_mat);   // reduce 4B + apply 4B in, 8B out
        add_bytes(st, kPhPivots, 8ull * (unsigned long long)c_piv);  // first P keys of each segment
        if (c_mat > mat_cap || c_ch > ch_cap || c_piv > piv_cap || c_lut > lut_cap) {
            st->overflow = 2;
            st->nchunks = 0;
            st->mat_total = 0;
        } else {
#if KS_PREFETCH && KS_SEGOFF_PF
            l2_prefetch(mat, 4ull * c_mat);
            l2_prefetch(moff, 8ull * c_mat);
#endif
        }
        st->scan_next = 0;
        *nseg_next = 0;   // the plan of this pass appends the next level's segments
    }
    // look-back words of the single-pass scan (c_mat is block-uniform)
    const long long nt = c_mat <= mat_cap ? cdiv(c_mat, kScanBlock) : 0;
    for (long long i = threadIdx.x; i < nt; i += blockDim.x) tstat[i] = 0ull;
}

__global__ void k_seg_offsets(Seg *segs, const int *nseg, DevStatus *st, long long mat_cap, int ch_cap,
                              int piv_cap, int lut_cap, const unsigned *mat, const long long *moff,
                              unsigned long long *tstat, int *nseg_next, int items)
{
    KS_PDL_ENTRY();
    __shared__ long long sh[33];
    seg_offsets_body(segs, *nseg, st, mat_cap, ch_cap, piv_cap, lut_cap, mat, moff, tstat, nseg_next, items, sh);
}

struct PivotsSmem {
    PivotScratch<kPMaxPow2> W;
    double piv[kPMax + kPivPad];
    unsigned lut[kLutMax];
};
constexpr int kPivotThreads = 1024;

__global__ void __launch_bounds__(kPivotThreads) k_pivots(Seg *segs, const int *nseg, const double *src,
                                                          double *piv_pool, unsigned *lut_pool, int *chunk_seg,
                                                          unsigned *mat)
{
    KS_PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PivotsSmem &PS = *reinterpret_cast<PivotsSmem *>(smem_raw);
    auto &W = PS.W;
    double *piv = PS.piv;
    unsigned *lut = PS.lut;
    const int ns = *nseg;
    for (int s = blockIdx.x; s < ns; s += gridDim.x) {
        const Seg g = segs[s];
        int k, T;
        double lo, scale;
        KS_TR_DECL;
        // K-sort's pivots are the segment's first P keys; a stalled segment (its
        // parent kept almost all keys in one gap: first-key pivots are making no
        // progress) takes P keys spread across it instead -- same partition rule
        build_pivots(src + g.start, g.P, g.T, piv, lut, W, k, T, lo, scale, pivot_stride(g.stall, g.len, g.P));
        KS_TR(11);
        for (int i = threadIdx.x; i <= k; i += blockDim.x) piv_pool[g.piv_off + i] = piv[i];
        for (int t = threadIdx.x; t < T; t += blockDim.x) lut_pool[g.lut_off + t] = lut[t];
        for (int c = threadIdx.x; c < g.nch; c += blockDim.x) chunk_seg[g.ch_off + c] = s;
        for (int q = threadIdx.x; q <= g.P; q += blockDim.x) mat[mat_eq(g, q)] = 0u;   // equality-run totals
        KS_TR(12);
        if (threadIdx.x == 0) {
            segs[s].k = k;
            segs[s].T = T;
            segs[s].lo = lo;
            segs[s].scale = scale;
        }
    }
}

// Level 0 of a single array (one segment, P up to 2047): the pivot build is on
// the critical path while all other SMs idle, so it is spread over the GPU.
// k_pivot_rank: each thread ranks one of the first P keys against all of them
// (ties by position) and writes it to its sorted place; k_front_lut: every CTA
// de-duplicates the sorted run and builds its slice of the bucket LUT.
constexpr int kRankThreads = 128;
constexpr int kRankParts = 8;   // threads per ranked key (a power of two dividing 32)

__global__ void __launch_bounds__(kRankThreads) k_pivot_rank(const double *in, int P, double *sorted)
{
    KS_PDL_ENTRY();
    KS_TL_T0;
    __shared__ double x[kPMax + 1];
    constexpr int kU = (kPMax + 1 + kRankThreads - 1) / kRankThreads;   // all loads in flight at once
    double t[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        const int i = u * kRankThreads + threadIdx.x;
        t[u] = i < P ? __ldcg(in + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        const int i = u * kRankThreads + threadIdx.x;
        if (i < P) x[i] = t[u];
    }
    __syncthreads();
    // kRankParts threads per key, each counting over a slice of the P keys
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = gt / kRankParts, part = gt % kRankParts;
    const int per = ((P + kRankParts - 1) / kRankParts) | 1;   // odd stride: the parts read distinct banks
    const int j0 = part * per, j1 = min(P, j0 + per);
    const double v = i < P ? x[i] : 0.0;
    int r = 0;
#pragma unroll 8
    for (int j = j0; j < j1; ++j) {
        const double y = x[j];
        r += (y < v || (y == v && j < i)) ? 1 : 0;
    }
#pragma unroll
    for (int o = kRankParts / 2; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (i < P && part == 0) sorted[r] = v;   // (NaN keys -- rejected by the gate -- may collide; all in range)
    KS_TL(21, 8, 0);
}

constexpr int kLutCtas = 16;


// Front of one large array after the pivot ranking (replaces the init kernel
// that ran beside the ranking and the LUT kernel behind both): the last CTA
// resets the status, advances the call sequence, routes the array, lays out
// the level-0 pass and stores the pivots; the others build one slice each of
// the LUT from the ranked first P keys (the single segment's P, T and table
// offsets follow from n alone).  Both de-duplicate the ranked keys.
__global__ void __launch_bounds__(kPivotThreads) k_front_lut(long long n, InitLists Lst, DevStatus *st, long long mat_cap,
                                                             int ch_cap, int piv_cap, int lut_cap, unsigned *mat,
                                                             const long long *moff, unsigned long long *tstat, int items,
                                                             unsigned long long magic, const double *sorted,
                                                             double *piv_pool, unsigned *lut_pool, int *chunk_seg)
{
    KS_PDL_ENTRY();
    KS_TL_T0;
    __shared__ double piv[kPMax + kPivPad];
    __shared__ long long sh[33];
    const bool init_cta = blockIdx.x == gridDim.x - 1;
    if (init_cta) {
        seq_advance(Lst.Q, magic);
        unsigned long long *w = reinterpret_cast<unsigned long long *>(st);
        for (int i = threadIdx.x; i < (int)(sizeof(DevStatus) / 8); i += blockDim.x) w[i] = 0ull;
        __syncthreads();
        __shared__ long long s_nt;
        if (threadIdx.x == 0) {
            // route_initial + seg_offsets_body for the one segment (no block scans)
            st->bad_index = kNoIndex;
            st->no_item_pf = n < KS_ITEM_PF_MIN_N ? 1 : 0;
            long long chunk = cdiv(cdiv(n, (long long)min(items, kChunkItemsMax)), (long long)kChunkAlign) * kChunkAlign;
            if (KS_STAGED && chunk > kStageMax) chunk = kStageMax;
            if (chunk < kChunkMin) chunk = kChunkMin;
            Seg g = make_seg(0, n, 0);
            g.P = pivots_for(n, kPMax);
            g.rows = 2 * g.P + 1;
            g.nch = (int)cdiv(n, chunk);
            g.T = lut_for(g.P, kLutMax);
            g.piv_off = g.lut_off = g.ch_off = 0;
            g.mat_off = 0;
            Lst.gsegs[0] = g;
            st->nseg[0] = 1;
            st->nseg[1] = 0;
            ++st->npasses;
            const long long c_mat = mat_entries(g);
            st->nchunks = g.nch;
            st->chunk = (int)chunk;
            st->mat_total = c_mat;
            add_bytes(st, kPhScan, 16ull * (unsigned long long)c_mat);
            add_bytes(st, kPhPivots, 8ull * (unsigned long long)(g.P + 1));
            if (c_mat > mat_cap || g.nch > ch_cap || g.P + 1 > piv_cap || g.T > lut_cap || Lst.seg_cap < 1) {
                st->overflow = 2;
                st->nchunks = 0;
                st->mat_total = 0;
            }
            st->scan_next = 0;
            s_nt = c_mat <= mat_cap ? cdiv(c_mat, (long long)kScanBlock) : 0;
        }
        __syncthreads();
        for (long long i = threadIdx.x; i < s_nt; i += blockDim.x) tstat[i] = 0ull;   // look-back words
        __syncthreads();
    }
    const int P = pivots_for(n, kPMax);
    long long carry = 0;
    for (int base = 0; base < P; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const double v = i < P ? __ldcg(sorted + i) : 0.0;
        const int keep = (i < P && (i == 0 || v != __ldcg(sorted + i - 1))) ? 1 : 0;
        long long tot;
        const long long pos = block_exclusive_scan(keep, sh, &tot);
        if (keep) piv[carry + pos] = v;
        carry += tot;
    }
    const int k = (int)carry;
    if (threadIdx.x < kPivPad) piv[k + threadIdx.x] = CUDART_NAN;
    __syncthreads();
    int T = lut_for(P, kLutMax);   // (= the layout's g.T; the single segment's LUT and pivots start at 0)
    const double lo = piv[0];
    double scale;
    lut_transform(piv, k, T, scale);
    const int nlut = gridDim.x - 1;
    const int per_cta = (T + nlut - 1) / nlut;
    const int c0 = blockIdx.x * per_cta, c1 = init_cta ? c0 : min(T, c0 + per_cta);
    const int per = (c1 - c0 + (int)blockDim.x - 1) / (int)blockDim.x;
    const int t0 = c0 + threadIdx.x * per, t1 = min(c1, t0 + per);
    if (t0 < t1) {
        int a = 0, hi_i = k;
        while (a < hi_i) {
            const int mid = (a + hi_i) >> 1;
            if (lut_bucket(piv[mid], lo, scale, T) < t0) a = mid + 1; else hi_i = mid;
        }
        for (int t = t0; t < t1; ++t) {
            int b = a;
            while (b < k && lut_bucket(piv[b], lo, scale, T) <= t) ++b;
            lut_pool[t] = lut_pack(a, b);
            a = b;
        }
    }
    if (init_cta) {
        Seg *segs = Lst.gsegs;
        const Seg g = segs[0];
        for (int i = threadIdx.x; i <= k; i += blockDim.x) piv_pool[g.piv_off + i] = piv[i];
        for (int c = threadIdx.x; c < g.nch; c += blockDim.x) chunk_seg[g.ch_off + c] = 0;
        for (int q = threadIdx.x; q <= g.P; q += blockDim.x) mat[mat_eq(g, q)] = 0u;   // equality-run totals
        __syncthreads();
        if (threadIdx.x == 0) {
            segs[0].k = k;
            segs[0].T = T;
            segs[0].lo = lo;
            segs[0].scale = scale;
        }
    }
    KS_TL(22, 8, 0);
}


// ---------------------------------------------------------------------------
// count: per (segment, chunk) class histogram -> class-major count matrix
// (shared-memory atomics: measured ~0.03 SM-cycles/key on B200, far cheaper
// than ballot- or match-based peer aggregation; scripts/mb_hist.cu)
// ---------------------------------------------------------------------------
struct PassSmem {
    double piv[kPMax + kPivPad];
    unsigned lut[kLutMax];
};

__device__ __forceinline__ void load_seg_tables(const double *piv_pool, const unsigned *lut_pool, const Seg &sg,
                                                PassSmem &P);
__device__ __forceinline__ void load_seg(const Seg *segs, int s, const double *piv_pool, const unsigned *lut_pool,
                                         Seg &sg, PassSmem &P)
{
    if (threadIdx.x == 0) sg = segs[s];
    __syncthreads();
    load_seg_tables(piv_pool, lut_pool, sg, P);
}
// the segment's pivots and LUT into shared memory (descriptor already in sg)
__device__ __forceinline__ void load_seg_tables(const double *piv_pool, const unsigned *lut_pool, const Seg &sg,
                                                PassSmem &P)
{
    // copies unrolled by 8 so that the L2 loads overlap (a rolled copy waits
    // one L2 round trip per element per thread)
    const int np = sg.k + kPivPad, T = sg.T;
    for (int i0 = 0; i0 < np; i0 += 8 * blockDim.x) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x + threadIdx.x;
            x[u] = i < sg.k ? piv_pool[sg.piv_off + i] : CUDART_NAN;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x + threadIdx.x;
            if (i < np) P.piv[i] = x[u];
        }
    }
    for (int i0 = 0; i0 < T; i0 += 8 * blockDim.x) {
        unsigned x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x + threadIdx.x;
            x[u] = i < T ? lut_pool[sg.lut_off + i] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x + threadIdx.x;
            if (i < T) P.lut[i] = x[u];
        }
    }
}

struct CountSmem {
    PassSmem P;
    unsigned hist[kRowsMax];
    Seg sg;
};

template <bool kGate>
__global__ void __launch_bounds__(kCountThreads, KS_PASS_MINB) k_count(const Seg *segs, const int *chunk_seg, const DevStatus *cst,
                                                         const double *src, const double *piv_pool,
                                                         const unsigned *lut_pool, unsigned *mat, DevStatus *st)
{
    KS_PDL_ENTRY();
    constexpr int U = 8;   // keys in flight per lane
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CountSmem &CS = *reinterpret_cast<CountSmem *>(smem_raw);
    PassSmem &P = CS.P;
    unsigned *hist = CS.hist;
    Seg &sg = CS.sg;
    int cached = -1;
    long long bad = LLONG_MAX;
    unsigned pz = 0, nz = 0;
    const int nchunks = cst->nchunks, chunk = cst->chunk;
    for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int s = chunk_seg[ch];
        __syncthreads();
        if (s != cached) {
            load_seg(segs, s, piv_pool, lut_pool, sg, P);
            cached = s;
        }
        for (int c = threadIdx.x; c < sg.rows; c += blockDim.x) hist[c] = 0;
        __syncthreads();
        const int j = ch - sg.ch_off;
        const long long base = sg.start + (long long)j * chunk;
        const int cnt = (int)min((long long)chunk, sg.len - (long long)j * chunk);
        const int T = sg.T;
        const double lo = sg.lo, scale = sg.scale;
        const double *in = src + base + threadIdx.x;
        int i0 = 0;
        for (; i0 + U * kCountThreads <= cnt; i0 += U * kCountThreads) {   // full blocks: no bounds checks
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = in[i0 + u * kCountThreads];
            if (kGate) {   // non-finite or zero keys are rare: check the batch, then look closer
                bool odd = false;
#pragma unroll
                for (int u = 0; u < U; ++u) odd |= !(fabs(v[u]) <= DBL_MAX) || v[u] == 0.0;
                if (odd) {
#pragma unroll
                    for (int u = 0; u < U; ++u) gate_one(v[u], base + threadIdx.x + i0 + u * kCountThreads, bad, pz, nz);
                }
            }
#if KS_BATCH == 2
#pragma unroll
            for (int g0 = 0; g0 < U; g0 += KS_BATCH_G) {
                int c[KS_BATCH_G];
                classify_batch<KS_BATCH_G>(v + g0, c, P.piv, P.lut, lo, scale, T);
#pragma unroll
                for (int u = 0; u < KS_BATCH_G; ++u) atomicAdd(&hist[c[u]], 1u);
            }
#elif KS_BATCH
            int c[U];
            classify_batch<U>(v, c, P.piv, P.lut, lo, scale, T);
#pragma unroll
            for (int u = 0; u < U; ++u) atomicAdd(&hist[c[u]], 1u);
#else
#pragma unroll
            for (int u = 0; u < U; ++u) atomicAdd(&hist[classify(v[u], P.piv, P.lut, lo, scale, T)], 1u);
#endif
        }
        if (i0 < cnt) {   // the last partial block, loads still batched
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kCountThreads + threadIdx.x;
                v[u] = i < cnt ? src[base + i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kCountThreads + threadIdx.x;
                if (i < cnt) {
                    if (kGate) gate_one(v[u], base + i, bad, pz, nz);
                    atomicAdd(&hist[classify(v[u], P.piv, P.lut, lo, scale, T)], 1u);
                }
            }
        }
        __syncthreads();
        for (int c = threadIdx.x; c < sg.rows; c += blockDim.x) {
            if (!(c & 1)) mat[mat_gap(sg, c >> 1, j)] = hist[c];
            else if (hist[c]) atomicAdd(&mat[mat_eq(sg, c >> 1)], hist[c]);   // (zeroed by k_pivots)
        }
    }
    if (kGate) gate_flush(bad, pz, nz, st);
}

// ---------------------------------------------------------------------------
// flat exclusive scan of the count matrix -> absolute-within-level offsets
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const unsigned *mat, const DevStatus *st,
                                                              long long *bsum)
{
    KS_PDL_ENTRY();
    __shared__ long long sh[33];
    const long long total = st->mat_total;
    const long long nb = cdiv(total, kScanBlock);
    for (long long b = blockIdx.x; b < nb; b += gridDim.x) {
        long long s = 0;
        for (int e = threadIdx.x; e < kScanBlock; e += blockDim.x) {
            long long i = b * kScanBlock + e;
            if (i < total) s += mat[i];
        }
        long long tot;
        block_exclusive_scan(s, sh, &tot);
        if (threadIdx.x == 0) bsum[b] = tot;
    }
}

__global__ void __launch_bounds__(1024) k_scan_bsums(long long *bsum, const DevStatus *st)
{
    KS_PDL_ENTRY();
    __shared__ long long sh[33];
    const long long nb = cdiv(st->mat_total, kScanBlock);
    long long carry = 0;
    for (long long base = 0; base < nb; base += blockDim.x) {
        long long i = base + threadIdx.x;
        long long x = i < nb ? bsum[i] : 0;
        long long tot;
        long long ex = block_exclusive_scan(x, sh, &tot);
        if (i < nb) bsum[i] = carry + ex;
        carry += tot;
    }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const unsigned *mat, const DevStatus *st,
                                                             const long long *bsum, long long *moff)
{
    KS_PDL_ENTRY();
    __shared__ long long sh[33];
    constexpr int E = kScanBlock / kScanThreads;
    const long long total = st->mat_total;
    const long long nb = cdiv(total, kScanBlock);
    for (long long b = blockIdx.x; b < nb; b += gridDim.x) {
        const long long i0 = b * kScanBlock + (long long)threadIdx.x * E;
        unsigned v[E];
        long long s = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            v[e] = (i0 + e < total) ? mat[i0 + e] : 0u;
            s += v[e];
        }
        long long ex = block_exclusive_scan(s, sh, nullptr) + bsum[b];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (i0 + e < total) moff[i0 + e] = ex;
            ex += v[e];
        }
    }
}

// Single-pass exclusive scan of the count matrix (decoupled look-back):
// tiles are claimed in order from a counter; each publishes its aggregate,
// then warp 0 walks back over the predecessors' published words (aggregate or
// inclusive prefix) until it meets a prefix.  Word = flag << 62 | value.

__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(const unsigned *mat, DevStatus *st,
                                                                unsigned long long *tstat, long long *moff)
{
    KS_PDL_ENTRY();
    KS_TL_T0;
    constexpr unsigned long long kScanAgg = 1ull << 62, kScanPrefix = 2ull << 62, kScanVal = (1ull << 62) - 1;
    __shared__ long long sh[33];
    __shared__ int s_tile;
    __shared__ long long s_excl;
    constexpr int E = kScanBlock / kScanThreads;
    static_assert(E == 8, "two uint4 per thread");
    const long long total = st->mat_total;
    const int ntiles = (int)cdiv(total, kScanBlock);
    const int lane = threadIdx.x & 31;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&st->scan_next, 1);
        __syncthreads();
        const int t = s_tile;
        if (t >= ntiles) break;
        const long long i0 = (long long)t * kScanBlock + (long long)threadIdx.x * E;
        unsigned v[E];
        if (i0 + E <= total) {
            const uint4 a = *reinterpret_cast<const uint4 *>(mat + i0);
            const uint4 b = *reinterpret_cast<const uint4 *>(mat + i0 + 4);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = i0 + e < total ? mat[i0 + e] : 0u;
        }
        long long s = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) s += v[e];
        long long tot;
        long long ex = block_exclusive_scan(s, sh, &tot);
        if (threadIdx.x < 32) {
            long long excl = 0;
            if (t == 0) {
                if (lane == 0) *reinterpret_cast<volatile unsigned long long *>(&tstat[0]) = kScanPrefix | (unsigned long long)tot;
            } else {
                if (lane == 0) {
                    __threadfence();
                    *reinterpret_cast<volatile unsigned long long *>(&tstat[t]) = kScanAgg | (unsigned long long)tot;
                }
                for (int j = t - 1;; j -= 32) {
                    const int idx = j - lane;
                    unsigned long long w;
                    do {
                        w = kScanPrefix;
                        if (idx >= 0) w = *reinterpret_cast<volatile unsigned long long *>(&tstat[idx]);
                    } while (!__all_sync(0xffffffffu, (w >> 62) != 0));
                    const unsigned pm = __ballot_sync(0xffffffffu, (w >> 62) == 2);
                    const int stop = pm ? __ffs(pm) - 1 : 31;
                    long long val = lane <= stop ? (long long)(w & kScanVal) : 0;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                    excl += val;
                    if (pm) break;
                }
                if (lane == 0) {
                    __threadfence();
                    *reinterpret_cast<volatile unsigned long long *>(&tstat[t]) =
                        kScanPrefix | (unsigned long long)(excl + tot);
                }
            }
            if (lane == 0) s_excl = excl;
        }
        __syncthreads();
        ex += s_excl;
        if (i0 + E <= total) {
            long long o[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                o[e] = ex;
                ex += v[e];
            }
#pragma unroll
            for (int e = 0; e < E; e += 2)
                *reinterpret_cast<longlong2 *>(moff + i0 + e) = make_longlong2(o[e], o[e + 1]);
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (i0 + e < total) moff[i0 + e] = ex;
                ex += v[e];
            }
        }
        __syncthreads();   // s_tile / s_excl reuse
    }
    KS_TL(24, 8, 0);
}

// start of class c inside segment g (relative), c in [0, rows]; rows -> len
__device__ __forceinline__ long long class_start(const Seg &g, const long long *moff, long long base_i, int c)
{
    if (c >= g.rows) return g.len;
    return moff[(c & 1) ? mat_eq(g, c >> 1) : mat_gap(g, c >> 1, 0)] - base_i;
}

// ---------------------------------------------------------------------------
// scatter: classify again and send each key straight to its class slot:
// slot = atomicAdd(cursor[gap]) on a shared-memory cursor seeded with the
// chunk's offset from the scanned count matrix (32-bit, relative to the
// segment start).  No tile staging: on B200 the direct 8-byte scatter into
// the L2-resident destination costs fewer shared-memory wavefronts than
// staging runs (ncu: staged 1.56 wavefronts/key, smem-bound).  Equality
// runs (odd classes) are not written: the finish pass fills them, so only
// gap classes carry a cursor.
// ---------------------------------------------------------------------------
#ifndef KS_ST_HINT
#define KS_ST_HINT 0      // cache hint of the scattered stores (0 default, 1 .cg, 2 .cs, 3 .wt)
#endif
__device__ __forceinline__ void scatter_store(double *p, double v)
{
#if KS_ST_HINT == 1
    __stcg(p, v);
#elif KS_ST_HINT == 2
    __stcs(p, v);
#elif KS_ST_HINT == 3
    __stwt(p, v);
#else
    *p = v;
#endif
}

#ifndef KS_OUT_HINT
#define KS_OUT_HINT 0     // cache hint of the segment sorters' final stores (0 default, 1 .cs evict-first)
#endif
// final sorted keys: never read again by the sort
__device__ __forceinline__ void out_store(double *p, double v)
{
#if KS_OUT_HINT == 1
    __stcs(p, v);
#else
    *p = v;
#endif
}

#ifndef KS_LOCAL_CS
#define KS_LOCAL_CS 0     // 1: the local partition's scatter loads (last read of its source) are evict-first
#endif
#ifndef KS_SEG_CS
#define KS_SEG_CS 0       // 1: the two-buffer segment sorters' loads (last read of the segment) are evict-first
#endif
__device__ __forceinline__ double ld_local_last(const double *p)
{
#if KS_LOCAL_CS
    return __ldcs(p);
#else
    return __ldcg(p);
#endif
}
template <bool kSingle>
__device__ __forceinline__ double ld_seg(const double *p)
{
#if KS_SEG_CS
    if (!kSingle) return __ldcs(p);
#endif
    return __ldcg(p);
}

struct ScatterSmem {
    PassSmem P;
    unsigned cursor[kPMax + 1];   // next slot per gap class, relative to the segment start
    Seg sg;
};

__global__ void __launch_bounds__(kPassThreads, KS_SCAT_MINB) k_scatter(const Seg *segs, const int *chunk_seg,
                                                          const DevStatus *cst, const double *src, double *dst,
                                                          const double *piv_pool, const unsigned *lut_pool,
                                                          const long long *moff, const unsigned *mat, int pf)
{
    KS_PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScatterSmem &S = *reinterpret_cast<ScatterSmem *>(smem_raw);
    constexpr int U = 8;
    if (abort_requested(cst)) return;   // non-finite key or both signed zeros: write nothing
    int cached = -1;
    const int nchunks = cst->nchunks, chunk = cst->chunk;
    for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int s = chunk_seg[ch];
        __syncthreads();
#if KS_PF_EARLY   // descriptor first, the cursors and destination prefetches next, the tables last
        const bool fresh = s != cached;
        if (fresh) {
            if (threadIdx.x == 0) S.sg = segs[s];
            __syncthreads();
        }
#else
        if (s != cached) {
            load_seg(segs, s, piv_pool, lut_pool, S.sg, S.P);
            cached = s;
        }
#endif
        const Seg &g = S.sg;
        const int j = ch - g.ch_off;
        const long long base = g.start + (long long)j * chunk;
        const int cnt = (int)min((long long)chunk, g.len - (long long)j * chunk);
        const long long base_i = moff[g.mat_off];
        const int T = g.T;
        const double lo = g.lo, scale = g.scale;
        double *out = dst + g.start;
        for (int q0 = 0; q0 <= g.k; q0 += 4 * blockDim.x) {   // 4 gaps per thread in flight
            long long off[4];
            unsigned cnt[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = q0 + u * blockDim.x + threadIdx.x;
                const long long e = mat_gap(g, q, j);
                off[u] = q <= g.k ? moff[e] : base_i;
                cnt[u] = q <= g.k ? mat[e] : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = q0 + u * blockDim.x + threadIdx.x;
                if (q <= g.k) {
                    const unsigned c0 = (unsigned)(off[u] - base_i);
                    S.cursor[q] = c0;
#if KS_PREFETCH
                    // pull this chunk's destination run of gap q into L2 ahead of the
                    // 8-byte stores (a partial-sector store that misses L2 waits for a fill);
                    // not when the whole pass is L2-resident anyway (pf == 0)
                    if (pf) l2_prefetch_lines(out + c0, 8ull * cnt[u]);
#endif
                }
            }
        }
#if KS_PF_EARLY
        if (fresh) {
            load_seg_tables(piv_pool, lut_pool, g, S.P);
            cached = s;
        }
#endif
        __syncthreads();
        const double *in = src + base + threadIdx.x;
        int i0 = 0;
        for (; i0 + U * kPassThreads <= cnt; i0 += U * kPassThreads) {
            double v[U];
#pragma unroll
#if KS_SRC_CS   // last read of the source at this level: evict-first, so the prefetched destination stays
            for (int u = 0; u < U; ++u) v[u] = __ldcs(in + i0 + u * kPassThreads);
#else
            for (int u = 0; u < U; ++u) v[u] = in[i0 + u * kPassThreads];
#endif
#if KS_SBATCH
#pragma unroll
            for (int g0 = 0; g0 < U; g0 += KS_SBATCH) {
                int c[KS_SBATCH];
                classify_batch<KS_SBATCH>(v + g0, c, S.P.piv, S.P.lut, lo, scale, T);
                unsigned slot[KS_SBATCH];
#pragma unroll
                for (int u = 0; u < KS_SBATCH; ++u) slot[u] = (c[u] & 1) ? 0u : atomicAdd(&S.cursor[c[u] >> 1], 1u);
#pragma unroll
                for (int u = 0; u < KS_SBATCH; ++u)
                    if (!(c[u] & 1)) scatter_store(out + slot[u], v[g0 + u]);
            }
#elif KS_BATCH
            int c[U];
            classify_batch<U>(v, c, S.P.piv, S.P.lut, lo, scale, T);
            unsigned slot[U];
#pragma unroll
            for (int u = 0; u < U; ++u) slot[u] = (c[u] & 1) ? 0u : atomicAdd(&S.cursor[c[u] >> 1], 1u);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (!(c[u] & 1)) out[slot[u]] = v[u];
#else
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = classify(v[u], S.P.piv, S.P.lut, lo, scale, T);
#if KS_SCATTER_EXP == 1   // experiment: slots taken, stores coalesced (wrong output)
                if (!(c & 1)) {
                    const unsigned sl = atomicAdd(&S.cursor[c >> 1], 1u);
                    out[(base - g.start) + i0 + u * kPassThreads + threadIdx.x] = v[u] + (double)(sl & 1);
                }
#elif KS_SCATTER_EXP == 2   // experiment: no slots, stores coalesced (wrong output)
                if (!(c & 1)) out[(base - g.start) + i0 + u * kPassThreads + threadIdx.x] = v[u];
#elif KS_SCATTER_EXP == 3   // experiment: slots taken, scattered stores of L2-resident lines (wrong output)
                if (!(c & 1)) out[atomicAdd(&S.cursor[c >> 1], 1u) & 0x3fffff] = v[u];
#else
                if (!(c & 1)) scatter_store(out + atomicAdd(&S.cursor[c >> 1], 1u), v[u]);
#endif
            }
#endif
        }
        if (i0 < cnt) {   // the last partial block, loads still batched
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kPassThreads + threadIdx.x;
                v[u] = i < cnt ? src[base + i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kPassThreads + threadIdx.x;
                if (i < cnt) {
                    const int c = classify(v[u], S.P.piv, S.P.lut, lo, scale, T);
                    if (!(c & 1)) scatter_store(out + atomicAdd(&S.cursor[c >> 1], 1u), v[u]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Staged partition pass (KS_STAGED): the count and scatter kernels of a
// global pass rebuilt around 128-bit loads, a branch-free classification,
// a shared-memory staging of every chunk in gap order and TMA bulk stores.
//
//   count:   per chunk, 2 keys per 16-byte load, class of every key
//            (classify_group: one LUT probe + at most two pivot probes, no
//            divergent branch), shared-memory histogram -> count-matrix
//            column; every key's class is also stored (2 B, KS_CLS) so the
//            scatter needs neither the pivot tables nor a second classification.
//   scatter: per chunk (= one tile, <= kStageMax keys, 1 CTA per SM):
//            A. gap table: this chunk's gap counts and destinations from the
//               count matrix (fetched during the previous chunk's copy-out),
//               exclusive block scan -> each gap run's start in the tile,
//               placed at its destination's index parity (one spare slot per
//               gap) so the run's 16-byte granules line up on both sides;
//            B. keys (16-byte loads, evict-first: last read of the source at
//               this level) and classes (4-byte loads) -> tile slot
//               atomicAdd(cur[gap]): the tile ends up ordered by gap;
//            C. every gap run leaves the tile by ONE TMA bulk copy
//               (cp.async.bulk.global.shared::cta) -- an odd head / tail key
//               by a plain store -- asynchronously, while the next chunk's
//               table is fetched.
//   Equality runs (odd classes) are never moved (filled later), as before.
// Replaces the per-key 8-byte scattered stores of k_scatter and its 80 MB
// destination prefetch (sort_core.py:94-101 is the reference's element move).
// Measured (C0, ncu): scatter 85 -> 71 us; DRAM 241 -> 144 MB per launch.
// ---------------------------------------------------------------------------
// Classes of G keys (see classify), batched so that the G lookup chains
// overlap: all bucket indices, then all LUT probes, then two pivot probes per
// key (pivots of later buckets are > v and the NaN sentinels compare false,
// so the probes need no bound checks), then the class arithmetic.  A bucket
// holding 3+ pivots (rare with T >= 2P) is finished afterwards by a short
// loop for the keys that need it.  kMap: 0 linear bucket map, 1 bit-image
// map, 2 single bucket (see lut_bucket) -- hoisted out of the key loops.
template <int kMap>
__device__ __forceinline__ int bucket_of(double v, double lo, double scale, unsigned long long olo, int T)
{
    if (kMap == 2) return 0;
    double t;
    if (kMap == 0) {
        t = (v - lo) * scale;
    } else {
        const unsigned long long ov = ord_bits(v);
        t = ov >= olo ? (double)(ov - olo) * -scale : -1.0;
    }
    const int x = __double2int_rz(t);
    return min(max(x, 0), T - 1);
}

struct PassMap {
    double lo, scale;
    unsigned long long olo;
    int T;
};

template <int kMap, int G>
__device__ __forceinline__ void classify_group(const double *v, int *c, const double *piv, const unsigned *lut,
                                               const PassMap &M)
{
    unsigned e[G];
#pragma unroll
    for (int u = 0; u < G; ++u) e[u] = lut[bucket_of<kMap>(v[u], M.lo, M.scale, M.olo, M.T)];
    double p0[G], p1[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
        // probes only where the bucket holds pivots (predicated loads: lanes of
        // pivot-free buckets -- most of them -- add no shared-memory traffic)
        const int a = (int)(e[u] & 0xffffu), b = (int)(e[u] >> 16);
        p0[u] = CUDART_INF;
        p1[u] = CUDART_INF;
        if (b > a) p0[u] = piv[a];
        if (b > a + 1) p1[u] = piv[a + 1];
    }
    unsigned slow = 0;
#pragma unroll
    for (int u = 0; u < G; ++u) {
        const int a = (int)(e[u] & 0xffffu), b = (int)(e[u] >> 16);
        const int r = a + (p0[u] < v[u] ? 1 : 0) + (p1[u] < v[u] ? 1 : 0);
        const int eq = (p0[u] == v[u] || p1[u] == v[u]) ? 1 : 0;
        c[u] = 2 * r + eq;
        slow |= (b - a > 2 ? 1u : 0u) << u;
    }
    if (slow) {
#pragma unroll
        for (int u = 0; u < G; ++u) {
            if (!((slow >> u) & 1u)) continue;
            const int a = (int)(e[u] & 0xffffu), b = (int)(e[u] >> 16);
            // pivots a+2 .. b-1 (sorted): how many lie below the key, and whether one equals it --
            // a binary search (a bucket can hold hundreds of pivots when the keys sit in a few narrow
            // clusters far apart: a linear scan made such inputs 4x slower than uniform ones)
            int lo_i = a + 2, hi_i = b;
#pragma unroll 1
            while (lo_i < hi_i) {
                const int mid = (lo_i + hi_i) >> 1;
                if (piv[mid] < v[u]) lo_i = mid + 1; else hi_i = mid;
            }
            const int r = lo_i - (a + 2);
            const int eq = (lo_i < b && piv[lo_i] == v[u]) ? 1 : 0;
            c[u] += 2 * r + ((c[u] & 1) ? 0 : eq);
        }
    }
}

// f(keys[G], index of keys[0] relative to in, number valid) over in[0, cnt):
// groups of G = 4 keys from two 16-byte loads (the first key peeled when in is
// not 16-byte aligned), kU2 pairs in flight per thread; ragged ends come as
// partial groups.  kCS: evict-first loads.
template <int kT, int kU2, bool kCS, typename F>
__device__ __forceinline__ void for_chunk_groups(const double *in, int cnt, F &&f)
{
    static_assert(kU2 % 2 == 0, "groups of two pairs");
    int i0 = 0;
    if ((reinterpret_cast<unsigned long long>(in) & 15ull) != 0 && cnt > 0) {
        if (threadIdx.x == 0) {
            double v[4] = {kCS ? __ldcs(in) : in[0], 0.0, 0.0, 0.0};
            f(v, 0, 1);
        }
        i0 = 1;
    }
    const double2 *in2 = reinterpret_cast<const double2 *>(in + i0);
    const int np = (cnt - i0) >> 1;
    int p0 = 0;
    for (; p0 + kU2 * kT <= np; p0 += kU2 * kT) {
        double2 w[kU2];
#pragma unroll
        for (int u = 0; u < kU2; ++u) {
            const double2 *p = in2 + p0 + u * kT + threadIdx.x;
            w[u] = kCS ? __ldcs(p) : *p;
        }
#pragma unroll
        for (int u = 0; u < kU2; u += 2) {
            double v[4] = {w[u].x, w[u].y, w[u + 1].x, w[u + 1].y};
            // (the two pairs are kT pairs apart: two index bases)
            f(v, i0 + 2 * (p0 + u * kT + (int)threadIdx.x), -(i0 + 2 * (p0 + (u + 1) * kT + (int)threadIdx.x)));
        }
    }
    for (int p = p0 + (int)threadIdx.x; p < np; p += kT) {
        const double2 w = kCS ? __ldcs(in2 + p) : in2[p];
        double v[4] = {w.x, w.y, 0.0, 0.0};
        f(v, i0 + 2 * p, 2);
    }
    const int last = i0 + 2 * np;   // an odd key left at the end
    if (last < cnt && threadIdx.x == kT - 1) {
        double v[4] = {kCS ? __ldcs(in + last) : in[last], 0.0, 0.0, 0.0};
        f(v, last, 1);
    }
}
// (the functor's third argument: n > 0 -> keys[0..n) at index i, consecutive;
//  n <= 0 -> a full group of two pairs at indices i, i+1 and -n, -n+1)
__device__ __forceinline__ long long group_index(int i, int n, int u)
{
    return n > 0 ? (long long)(i + u) : (long long)(u < 2 ? i + u : -n + (u - 2));
}

// one pass's classification with the bucket map hoisted: calls body.template
// operator()<kMap>() for the segment's map kind
template <typename B>
__device__ __forceinline__ void with_map(const PassMap &M, B &&body)
{
    if (M.T <= 1) body(std::integral_constant<int, 2>());
    else if (M.scale >= 0.0) body(std::integral_constant<int, 0>());
    else body(std::integral_constant<int, 1>());
}

#ifndef KS_COUNT2_MINB
#define KS_COUNT2_MINB 2
#endif
template <bool kGate>
__global__ void __launch_bounds__(kCount2Threads, KS_COUNT2_MINB) k_count2(const Seg *segs, const int *chunk_seg,
                                                             const DevStatus *cst, const double *src,
                                                             const double *piv_pool, const unsigned *lut_pool,
                                                             unsigned *mat, DevStatus *st, unsigned short *cls)
{
    KS_PDL_ENTRY();
    KS_TL_T0;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CountSmem &CS = *reinterpret_cast<CountSmem *>(smem_raw);
    PassSmem &P = CS.P;
    unsigned *hist = CS.hist;
    Seg &sg = CS.sg;
    int cached = -1;
    long long bad = LLONG_MAX;
    unsigned pz = 0, nz = 0;
    const int nchunks = cst->nchunks, chunk = cst->chunk;
    for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int s = chunk_seg[ch];
        __syncthreads();
        if (s != cached) {
            load_seg(segs, s, piv_pool, lut_pool, sg, P);
            cached = s;
        }
        for (int c = threadIdx.x; c < sg.rows; c += blockDim.x) hist[c] = 0;
        __syncthreads();
        const int j = ch - sg.ch_off;
        const long long base = sg.start + (long long)j * chunk;
        const int cnt = (int)min((long long)chunk, sg.len - (long long)j * chunk);
        const PassMap M{sg.lo, sg.scale, ord_bits(sg.lo), sg.T};
        with_map(M, [&](auto mk) {
            constexpr int kMap = decltype(mk)::value;
            for_chunk_groups<kCount2Threads, 4, false>(src + base, cnt, [&](const double *v, int i, int nv) {
                // level 0 also gates: non-finite keys (sort_core.py:50-59) and signed zeros
                if (kGate) {
                    bool odd = false;
#pragma unroll
                    for (int u = 0; u < 4; ++u) odd |= (nv <= 0 || u < nv) && !(fabs(v[u]) <= DBL_MAX && v[u] != 0.0);
                    if (odd) {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (nv <= 0 || u < nv) gate_one(v[u], base + group_index(i, nv, u), bad, pz, nz);
                    }
                }
                int c[4];
                classify_group<kMap, 4>(v, c, P.piv, P.lut, M);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (nv <= 0 || u < nv) atomicAdd(&hist[c[u]], 1u);
                if (KS_CLS) {   // each key's class for the scatter (pairs: 4-byte stores)
                    unsigned short *cb = cls + base;
                    if (nv <= 0 && !((base + i) & 1)) {   // (parity uniform over the pass: 4-byte aligned)
                        *reinterpret_cast<unsigned *>(cb + i) = (unsigned)c[0] | ((unsigned)c[1] << 16);
                        *reinterpret_cast<unsigned *>(cb - nv) = (unsigned)c[2] | ((unsigned)c[3] << 16);
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (nv <= 0 || u < nv) cb[group_index(i, nv, u)] = (unsigned short)c[u];
                    }
                }
            });
        });
        __syncthreads();
        for (int c = threadIdx.x; c < sg.rows; c += blockDim.x) {
            if (!(c & 1)) mat[mat_gap(sg, c >> 1, j)] = hist[c];
            else if (hist[c]) atomicAdd(&mat[mat_eq(sg, c >> 1)], hist[c]);   // (zeroed by k_pivots)
        }
    }
    if (kGate) gate_flush(bad, pz, nz, st);
    KS_TL(23, 8, 0);
}

struct Scatter2Smem {
#if !KS_CLS
    PassSmem P;                  // (with KS_CLS the classes come from the count pass: no tables)
#endif
    unsigned cur[kPMax + 1];     // next tile slot per gap
    unsigned delta[kPMax + 1];   // destination (relative to the segment start) - tile position, per gap
    unsigned sh[33];
    unsigned total;
    Seg sg;
#if KS_SCAT_TMA
    alignas(16) double stage[kStageMax + kPMax + 2];   // gap runs, each started at its destination's index parity
#else
    alignas(16) double stage[kStageMax];           // the chunk's gap keys in gap order
#endif
#if KS_CLS && !KS_SCAT_TMA
    unsigned dsti[kStageMax];          // destination (relative to the segment start) of each tile position
#elif !KS_CLS
    unsigned short cls[kStageMax];     // gap of each tile position
#endif
};

__global__ void __launch_bounds__(kScat2Threads, 1) k_scatter2(const Seg *segs, const int *chunk_seg,
                                                              const DevStatus *cst, const double *src, double *dst,
                                                              const double *piv_pool, const unsigned *lut_pool,
                                                              const long long *moff, const unsigned *mat,
                                                              const unsigned short *cls, int pf)
{
    KS_PDL_ENTRY();
    KS_TL_T0;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Scatter2Smem &S = *reinterpret_cast<Scatter2Smem *>(smem_raw);
    static_assert(2 * kScat2Threads >= kPMax + 1, "two gaps per thread in the gap table");
    if (abort_requested(cst)) return;   // non-finite key, both signed zeros or bad offsets: write nothing
    int cached = -1;
    const int nchunks = cst->nchunks, chunk = cst->chunk;
    const int tid = threadIdx.x;
    // gap table of a chunk: gaps 2*tid, 2*tid+1 (contiguous per thread for the
    // scan); the next chunk's is fetched during this chunk's copy-out when it
    // belongs to the same segment (its L2 latency then overlaps the stores)
    unsigned c2[2] = {0u, 0u};
    long long o2[2] = {0, 0};
    int have = -1;
    auto fetch_table = [&](const Seg &g, int jj, long long bi) {   // (bi: the value of a padding gap)
        const int ng = g.k + 1;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int q = 2 * tid + u;
            const long long e = mat_gap(g, q, jj);
            c2[u] = q < ng ? __ldcg(mat + e) : 0u;
            o2[u] = q < ng ? __ldcg(moff + e) : bi;   // (base subtracted at use: no stall at the fetch)
        }
    };
    // L2 prefetch of the chunk's destination runs: a run boundary leaves a
    // partially written sector, and a write that misses L2 is slow (the
    // round-1 scatter measured 156 -> 103 us from the same prefetch)
    auto prefetch_runs = [&](const Seg &g, long long bi) {
        if (!pf) return;
        const double *o = dst + g.start;
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (c2[u]) l2_prefetch_lines(o + (o2[u] - bi), 8ull * c2[u]);
    };
    for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
#ifdef KS_TIMELINE
        const unsigned long long ph_t0 = tl_now();
        unsigned long long ph_t1 = ph_t0, ph_t2 = ph_t0;
#endif
        const int s = chunk_seg[ch];
        __syncthreads();   // the previous tile's copy-out is done
        if (s != cached) {
#if KS_CLS
            if (tid == 0) S.sg = segs[s];
            __syncthreads();
#else
            load_seg(segs, s, piv_pool, lut_pool, S.sg, S.P);
#endif
            cached = s;
        }
        const Seg &g = S.sg;
        const int j = ch - g.ch_off;
        const long long base = g.start + (long long)j * chunk;
        const int cnt = (int)min((long long)chunk, g.len - (long long)j * chunk);
        const long long base_i = moff[g.mat_off];
        // A. gap table -> run starts in the tile (cur) and destination deltas
        const int ng = g.k + 1;
        if (have != ch) {
            fetch_table(g, j, base_i);
            prefetch_runs(g, base_i);
        }
        unsigned tot;
#if KS_SCAT_TMA
        // one spare slot per gap: each run starts in the tile at its destination's
        // index parity, so the run's 16-byte granules line up on both sides
        unsigned ps[2];
        {
            unsigned ex = block_exclusive_scan_u32(c2[0] + c2[1] + 2u, S.sh, &tot);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int q = 2 * tid + u;
                const unsigned long long a = (unsigned long long)(g.start + (o2[u] - base_i));
                ps[u] = ex + ((ex ^ (unsigned)a) & 1u);
                if (q < ng) S.cur[q] = ps[u];
                ex += c2[u] + 1u;
            }
        }
#else
        unsigned ex = block_exclusive_scan_u32(c2[0] + c2[1], S.sh, &tot);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int q = 2 * tid + u;
            if (q < ng) {
                S.cur[q] = ex;
                S.delta[q] = (unsigned)(o2[u] - base_i - (long long)ex);
            }
            ex += c2[u];
        }
#endif
#if KS_SCAT_TMA
        // a tile without a single gap key (all its keys equal pivots: few distinct values)
        // has nothing to move -- its keys and classes are not even read
        if (tot == 2u * (unsigned)kScat2Threads) {
            have = -1;
            continue;
        }
        // the previous tile's bulk copies have read the buffer (they overlapped this tile's table)
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
        __syncthreads();
        // B. stage the chunk's gap keys in gap order
#ifdef KS_TIMELINE
        ph_t1 = tl_now();
#endif
#if KS_CLS
        {
            // keys by 16-byte loads and their classes (from the count pass) by
            // 4-byte loads, kU2 pairs in flight per thread
            constexpr int kU2 = 4, kT = kScat2Threads;
            const double *in = src + base;
            const unsigned short *cin = cls + base;
            auto place = [&](double v, unsigned c) {
                if (!(c & 1u)) {
                    const unsigned q = c >> 1;
                    const unsigned slot = atomicAdd(&S.cur[q], 1u);
                    S.stage[slot] = v;
#if !KS_SCAT_TMA
                    S.dsti[slot] = S.delta[q] + slot;
#endif
                }
            };
            int i0 = 0;
            if ((reinterpret_cast<unsigned long long>(in) & 15ull) != 0) {
                if (tid == 0) place(KS_SRC_CS ? __ldcs(in) : in[0], cin[0]);
                i0 = 1;
            }
            const bool c4 = !((base + i0) & 1);   // class pairs 4-byte aligned (uniform)
            const double2 *in2 = reinterpret_cast<const double2 *>(in + i0);
            const int np = (cnt - i0) >> 1;
            auto cpair = [&](int p) -> unsigned {
                const unsigned short *cp = cin + i0 + 2 * p;
                return c4 ? __ldcs(reinterpret_cast<const unsigned *>(cp))
                          : (unsigned)__ldcs(cp) | ((unsigned)__ldcs(cp + 1) << 16);
            };
            int p0 = 0;
            for (; p0 + kU2 * kT <= np; p0 += kU2 * kT) {
                double2 w[kU2];
                unsigned cc[kU2];
#pragma unroll
                for (int u = 0; u < kU2; ++u) {
                    const int p = p0 + u * kT + tid;
                    w[u] = KS_SRC_CS ? __ldcs(in2 + p) : in2[p];
                    cc[u] = cpair(p);
                }
#pragma unroll
                for (int u = 0; u < kU2; ++u) {
                    place(w[u].x, cc[u] & 0xffffu);
                    place(w[u].y, cc[u] >> 16);
                }
            }
            for (int p = p0 + tid; p < np; p += kT) {
                const double2 w = KS_SRC_CS ? __ldcs(in2 + p) : in2[p];
                const unsigned cc = cpair(p);
                place(w.x, cc & 0xffffu);
                place(w.y, cc >> 16);
            }
            const int last = i0 + 2 * np;
            if (last < cnt && tid == kT - 1) place(KS_SRC_CS ? __ldcs(in + last) : in[last], cin[last]);
        }
#else
        const PassMap M{g.lo, g.scale, ord_bits(g.lo), g.T};
        with_map(M, [&](auto mk) {
            constexpr int kMap = decltype(mk)::value;
            for_chunk_groups<kScat2Threads, 4, KS_SRC_CS != 0>(src + base, cnt, [&](const double *v, int, int nv) {
                int c[4];
                classify_group<kMap, 4>(v, c, S.P.piv, S.P.lut, M);
                unsigned slot[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    slot[u] = ((nv <= 0 || u < nv) && !(c[u] & 1)) ? atomicAdd(&S.cur[c[u] >> 1], 1u) : ~0u;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (slot[u] != ~0u) {
                        S.stage[slot[u]] = v[u];
                        S.cls[slot[u]] = (unsigned short)(c[u] >> 1);
                    }
            });
        });
#endif
#if KS_SCAT_TMA
        // this chunk's runs (in registers) before the next chunk's table replaces them
        const unsigned rc[2] = {c2[0], c2[1]};
        const long long ro[2] = {o2[0] - base_i, o2[1] - base_i};
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // staged keys -> visible to the bulk copies
#endif
        __syncthreads();
#ifdef KS_TIMELINE
        ph_t2 = tl_now();
#endif
        have = -1;
        {
            const int nx = ch + (int)gridDim.x;
            if (nx < nchunks && nx - g.ch_off < g.nch) {   // next chunk in the same segment
                fetch_table(g, nx - g.ch_off, base_i);
                prefetch_runs(g, base_i);
                have = nx;
#if KS_SRC_PF
                // the next tile's keys and classes into L2 while this tile's runs leave:
                // its staging loads (two dependent DRAM round trips per thread) then hit L2
                if (tid == 0) {
                    const long long nb = g.start + (long long)(nx - g.ch_off) * chunk;
                    const long long nc = min((long long)chunk, g.len - (long long)(nx - g.ch_off) * chunk);
                    l2_prefetch(src + nb, 8ull * (unsigned long long)nc);
                    l2_prefetch(cls + nb, 2ull * (unsigned long long)nc);
                }
#endif
            }
        }
        // C. copy-out in tile order: lane l of a warp writes position w + l, so
        //    a warp store covers 32 consecutive destinations of the runs it
        //    crosses (whole sectors except at run ends)
        double *out = dst + g.start;
#if KS_SCAT_TMA
        // C'. every run leaves by one bulk copy (an odd head / tail key by a plain store)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int n = (int)rc[u];
            if (n == 0) continue;
            const unsigned sp = ps[u];
            double *o = out + ro[u];
            const int head = (int)((g.start + ro[u]) & 1);
            const int mid = (n - head) & ~1;
            if (head) o[0] = S.stage[sp];
            if (mid > 0)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o + head),
                             "r"((unsigned)__cvta_generic_to_shared(&S.stage[sp + head])), "r"(8u * (unsigned)mid)
                             : "memory");
            if (head + mid < n) o[head + mid] = S.stage[sp + head + mid];
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        (void)tot;
#ifdef KS_TIMELINE
        if (blockIdx.x < 4 && threadIdx.x == 0) {   // phases of a few CTAs: A table+scan, B staging, C copy-out issue
            tl_rec(50, 0, cnt, ph_t0);
            const unsigned long long t1 = tl_now();
            (void)t1;
            tl_rec(51, 0, (long long)(ph_t1 - ph_t0), ph_t0);
            tl_rec(52, 0, (long long)(ph_t2 - ph_t1), ph_t1);
        }
#endif
#else
        const int tot2 = (int)tot;
#pragma unroll 4
#if KS_CLS
        for (int i = tid; i < tot2; i += kScat2Threads) out[S.dsti[i]] = S.stage[i];
#else
        for (int i = tid; i < tot2; i += kScat2Threads) out[S.delta[S.cls[i]] + (unsigned)i] = S.stage[i];
#endif
#endif
    }
#if KS_SCAT_TMA
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
    KS_TL(26, 8, 0);
}

// ---------------------------------------------------------------------------
// emission of finishing work (shared by the global plan and the local
// partitioner).  Each thread owns one pivot j: the gap below it (class 2j,
// gl keys at ag) and its equality run (class 2j+1, el keys at ae).
//  * gap <= kUnitMax (+ its short equality run)  -> one warp unit
//  * kUnitMax < gap <= kLocalMax                 -> local-partition segment
//  * gap > kLocalMax                             -> next global pass
//  * equality run (any length)                   -> fill (never scattered)
// Lists are reserved per CTA with one atomic each.
// ---------------------------------------------------------------------------
struct EmitOut {
    long long unit_keys, fill_keys, items;
};

struct EmitArgs {
    Seg *gnext;        // next global level (> kLocalMax)
    int *ngnext;
    int gcap;
    LeafQ Q;           // local / sort queues of the leaf kernel
    Item *units;       // warp units (<= kUnitMax keys) and long fills
    int ucap;
    double *keys;      // user buffer: short equality runs and tiny gaps are written here directly
    const double *tmp;
    int in_leaf;       // emitting inside the leaf launch: local children go to the sort queue
    int defer;         // running concurrently with the scatter: no reads of the scattered data and no
                       // writes to the scatter's source -- tiny gaps become units, pivot runs fill items
    int merge_cand;    // merging (see emit_pairs): pairs up to this many keys are candidates,
    int merge_t;       // ... grouped by floor(run prefix / merge_t); 0: kMergeCand / kMergeT
    int to_leaf;       // one small array: every segment of kUnitMax < len <= kSortMax keys goes to the
                       // leaf kernel's sort queue (one ~n/SMs-key group per SM, one wave) instead of the lists
};

// packed per-thread counts for one block scan (11 bits each; blocks <= 1024 threads):
// units + fill items (<= 2 per thread), local items, global segments, sort items
constexpr int kPkU = 0, kPkL = 16, kPkG = 27, kPkS = 38, kPkLB = 49;   // (units: 16 bits)
constexpr int kFillPiece = 4096;   // long fills are split so that many warps write them
__device__ __forceinline__ long long pk_get(long long x, int sh, int bits) { return (x >> sh) & ((1ll << bits) - 1); }

// sort up to kTinyGap keys with one thread (src may equal dst)
__device__ __forceinline__ void tiny_sort_copy(const double *src, double *dst, int m)
{
    double a[kTinyGap];
    for (int i = 0; i < m; ++i) {
        const double x = src[i];
        int j = i;
        while (j > 0 && a[j - 1] > x) {
            a[j] = a[j - 1];
            --j;
        }
        a[j] = x;
    }
    for (int i = 0; i < m; ++i) dst[i] = a[i];
}

// Emission of one partition's classes, one pivot pair (gap 2j, run 2j+1) per thread:
//  * gap <= kTinyGap                        -> sorted right here
//  * kTinyGap < gap <= kUnitMax             -> warp unit
//  * kUnitMax < gap <= kSortMax             -> sort queue
//  * kSortMax < gap <= kLocalMax            -> local queue
//  * gap > kLocalMax                        -> next global pass
//  * equality run <= kFillDirect            -> written right here; longer -> fill item
//
// Merging: consecutive pairs of <= kMergeCand keys (gap + a short equality
// run) are grouped, within runs of such pairs, by floor(run prefix / kMergeT),
// and a group of two or more pairs is sorted as ONE small segment (its pivots'
// runs included: they are written into the data buffer too), so the segment
// sorter sees fewer, larger segments.  Groups hold < kMergeT + kMergeCand keys.
// `mg` is block-sized shared scratch.
#ifndef KS_MERGE
#define KS_MERGE 1
#endif
#ifndef KS_MERGE_CAND
#define KS_MERGE_CAND (2 * sort_cap(1) / 3)
#endif
#ifndef KS_MERGE_T
#define KS_MERGE_T (sort_cap(1) / 3)
#endif
constexpr int kMergeCand = KS_MERGE_CAND, kMergeT = KS_MERGE_T;
static_assert(kMergeCand + kMergeT <= sort_cap(1) && kMergeCand <= sort_cap(1), "merged groups are small segments");
__device__ __forceinline__ bool mg_prev_cand(int *mg, bool cand)
{
    mg[threadIdx.x] = cand ? 1 : 0;
    __syncthreads();
    const bool p = threadIdx.x > 0 && mg[threadIdx.x - 1] != 0;
    __syncthreads();
    return p;
}
__device__ __forceinline__ long long block_inclusive_max(long long x, long long *sh)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = y > inc ? y : inc;
    }
    if (lane == 31) sh[wid] = inc;
    __syncthreads();
    long long w = -1;
    for (int q = 0; q < wid && q < nw; ++q) w = sh[q] > w ? sh[q] : w;
    __syncthreads();
    return w > inc ? w : inc;
}

__device__ __forceinline__ double block_inclusive_max_f64(double x, long long *sh)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = y > inc ? y : inc;
    }
    double *shd = reinterpret_cast<double *>(sh);
    if (lane == 31) shd[wid] = inc;
    __syncthreads();
    double w = -CUDART_INF;
    for (int q = 0; q < wid && q < nw; ++q) w = shd[q] > w ? shd[q] : w;
    __syncthreads();
    return w > inc ? w : inc;
}

__device__ EmitOut emit_pairs(bool have, long long ag, long long gl, long long ae, long long el, double pv, int dst_id,
                              const EmitArgs &A, DevStatus *st, long long *sh, long long *sbase, int *mg, double blo,
                              double bhi, long long plen)
{
    const int stall = 4 * gl > 3 * plen ? 1 : 0;   // this gap kept > 3/4 of the parent's keys
    int u_gap = 0, s_gap = 0, l_gap = 0, g_gap = 0, t_gap = 0;
    long long s_ag = ag, s_gl = gl;   // the sort-queue item of this thread (its gap, or the merged group it closes)
    double s_blo = blo;
    bool merged = false;
#if KS_MERGE
    if (KS_MERGE == 2 || !A.in_leaf) {   // (block-uniform; in the leaf it costs more than it saves)
        const long long sz = gl + el;
        const int mcand = A.merge_t > 0 ? A.merge_cand : kMergeCand, mt = A.merge_t > 0 ? A.merge_t : kMergeT;
        const bool cand = have && sz <= mcand && el <= kFillDirect;
        const long long x = block_exclusive_scan(cand ? sz : 0, sh, nullptr);   // (non-candidates add 0)
        const bool prev_cand = mg_prev_cand(mg, cand);
        // prefix at the start of this pair's run: X is non-decreasing, so the
        // latest run start carries the largest X
        const long long xr = block_inclusive_max(cand && !prev_cand ? x : -1, sh);
        const int key = cand ? (int)((x - xr) / mt) : -1;
        mg[threadIdx.x] = key;
        __syncthreads();
        const bool leader = cand && (threadIdx.x == 0 || mg[threadIdx.x - 1] != key);
        const bool last = cand && (threadIdx.x + 1 == (int)blockDim.x || mg[threadIdx.x + 1] != key);
        const long long agl = block_inclusive_max(leader ? ag : -1, sh);   // gaps are in order: latest leader
        const double glo = block_inclusive_max_f64(leader ? blo : -CUDART_INF, sh);   // ... and so are their bounds
        merged = cand && !(leader && last);
        if (merged) {
            if (dst_id && el > 0)   // the run is part of the merged segment's data
                for (long long i = 0; i < el; ++i) const_cast<double *>(A.tmp)[ae + i] = pv;
            if (last) {
                const long long len = ag + gl + el - agl;
                if (A.to_leaf && len > kUnitMax) {   // (the group's last thread queues it below)
                    s_gap = 1;
                    s_ag = agl;
                    s_gl = len;
                    s_blo = glo;
                } else
                    small_push(A.Q, make_bseg(agl, len, dst_id, glo, bhi), st);
            }
        }
        __syncthreads();   // mg reuse
    }
#endif
    if (have && !merged && (gl >= 2 || (gl == 1 && dst_id == 1))) {
        if (gl <= kTinyGap && !A.defer) {
            tiny_sort_copy((dst_id ? A.tmp : A.keys) + ag, A.keys + ag, (int)gl);
            t_gap = 1;
        }
        else if (gl <= kUnitMax) u_gap = 1;
        else if (gl <= sort_cap(1) && !A.to_leaf) small_push(A.Q, make_bseg(ag, gl, dst_id, blo, bhi), st);
        else if (gl <= kSortMax) s_gap = 1;
        else if (gl <= kLocalMax) l_gap = 1;
        else g_gap = 1;
    }
    // pivot runs: written here when short (a merged group's run is its data:
    // in tmp above, or here when the group lives in keys), else fill items
    const bool direct = have && el > 0 && el <= kFillDirect && (merged ? dst_id == 0 : !A.defer);
    if (direct)
        for (long long i = 0; i < el; ++i) A.keys[ae + i] = pv;
    const int f_eq = (have && el > 0 && !merged && !direct) ? (int)((el + kFillPiece - 1) / kFillPiece) : 0;   // fill pieces
    const int nu = u_gap + f_eq;
    // the plan stores big local items at the front of the local queue, the others from
    // the back: the leaf launch takes them front to back (longest first)
    const int lb_gap = (l_gap && !A.in_leaf && gl > kLocalBig) ? 1 : 0;
    if (lb_gap) l_gap = 0;
    const long long pk = ((long long)nu << kPkU) | ((long long)l_gap << kPkL) | ((long long)g_gap << kPkG) |
                         ((long long)s_gap << kPkS) | ((long long)lb_gap << kPkLB);
    long long tpk;
    const long long xpk = block_exclusive_scan(pk, sh, &tpk);
    if (threadIdx.x == 0) {
        const int tu = (int)pk_get(tpk, kPkU, 16), tl = (int)pk_get(tpk, kPkL, 11);
        const int tg = (int)pk_get(tpk, kPkG, 11), ts = (int)pk_get(tpk, kPkS, 11);
        const int tlb = (int)pk_get(tpk, kPkLB, 11);
        if (tl + tlb) atomicAdd(&st->pending, tl + tlb);   // before the slots become claimable
        sbase[4] = tlb ? atomicAdd(&st->lqb_claim, tlb) : 0;
        sbase[0] = tu ? atomicAdd(&st->nunits, tu) : 0;
        sbase[1] = tl ? atomicAdd(A.in_leaf ? &st->sq_claim : &st->lq_claim, tl) : 0;
        sbase[2] = tg ? atomicAdd(A.ngnext, tg) : 0;
        sbase[3] = ts ? atomicAdd(&st->sq_claim, ts) : 0;
    }
    __syncthreads();
    long long ui = sbase[0] + pk_get(xpk, kPkU, 16);
    if (u_gap) {
        if (ui < A.ucap) A.units[ui] = make_item(ag, gl, kItemUnit, dst_id); else st->overflow = 3;
        ++ui;
    }
    for (int f = 0; f < f_eq; ++f, ++ui) {   // fill pieces of <= kFillPiece keys
        const long long off = (long long)f * kFillPiece;
        Item it = make_item(ae + off, min((long long)kFillPiece, el - off), kItemFill, dst_id);
        it.value = pv;
        if (ui < A.ucap) A.units[ui] = it; else st->overflow = 3;
    }
    if (s_gap)
        q_publish(A.Q.sq, A.Q.sq_ready, A.Q.scap, (int)(sbase[3] + pk_get(xpk, kPkS, 11)),
                  with_kind(make_bseg(s_ag, s_gl, dst_id, s_blo, bhi), kItemSort), q_epoch(A.Q));
    if (l_gap) {
        const int i = (int)(sbase[1] + pk_get(xpk, kPkL, 11));
        Seg c = with_kind(make_bseg(ag, gl, dst_id, blo, bhi), kItemLocal);
        c.stall = stall;
        if (A.in_leaf) q_publish(A.Q.sq, A.Q.sq_ready, A.Q.scap, i, c, q_epoch(A.Q));
        else if (i < A.Q.lcap) A.Q.lq[A.Q.lcap - 1 - i] = c; else st->overflow = 7;   // (read after this launch)
    }
    if (lb_gap) {
        const int i = (int)(sbase[4] + pk_get(xpk, kPkLB, 11));
        Seg c = with_kind(make_bseg(ag, gl, dst_id, blo, bhi), kItemLocal);
        c.stall = stall;
        if (i < A.Q.lcap) A.Q.lq[i] = c; else st->overflow = 7;
    }
    if (g_gap) {
        const long long gi = sbase[2] + pk_get(xpk, kPkG, 11);
        Seg c = make_seg(ag, gl, dst_id);
        c.stall = stall;
        if (gi < A.gcap) A.gnext[gi] = c; else st->overflow = 4;
    }
    // keys in fills / units (block totals; segments < 2^31 keys)
    long long tk;
    block_exclusive_scan((have ? el : 0) | (((u_gap | t_gap) ? gl : 0) << 32), sh, &tk);
    EmitOut o;
    o.unit_keys = tk >> 32;
    o.fill_keys = tk & 0xffffffffll;
    o.items = pk_get(tpk, kPkU, 16);
    return o;
}

__device__ __forceinline__ void account_partition(DevStatus *st, long long len, const EmitOut &o, bool local)
{
    // algorithmic bytes: count reads 8B/key; scatter reads 8B/key and writes 8B
    // per key it places; units read+write 16B/key; fills write 8B/key
    add_bytes(st, local ? kPhLeaf : kPhCount, 8ull * len);
    add_bytes(st, local ? kPhLeaf : kPhScatter, 8ull * len + 8ull * (len - o.fill_keys));
    add_bytes(st, kPhLeaf, 16ull * o.unit_keys + 8ull * o.fill_keys);
    atomicAdd(&st->keys_partitioned, (unsigned long long)len);
    atomicAdd(&st->keys_leaf, (unsigned long long)o.unit_keys);
    atomicAdd(&st->leaves, (unsigned long long)o.items);
}

// ---------------------------------------------------------------------------
// plan (global pass): class extents from the scanned count matrix
// ---------------------------------------------------------------------------
#ifndef KS_PLAN_THREADS
#define KS_PLAN_THREADS 128
#endif
constexpr int kPlanThreads = KS_PLAN_THREADS;
constexpr int kPlanChunks = (kPMax + 1 + kPlanThreads - 1) / kPlanThreads;   // grid.y: pivot-pair chunks

// One CTA per (segment, chunk of kPlanThreads pivot pairs): gap 2j and
// equality run 2j+1 for j in the chunk (j = k: the last gap).
// chained: launched programmatically behind the scatter (deferred emission:
// it needs only the scan and the pivots), it runs on the SMs the scatter's
// CTAs leave; it completes only after the scatter (griddepcontrol.wait at the end).
__global__ void __launch_bounds__(kPlanThreads) k_plan(const Seg *segs, const int *nseg, const double *piv_pool,
                                                       const long long *moff, EmitArgs A, DevStatus *st, int dst_id,
                                                       int chained)
{
    if (chained)
        asm volatile("griddepcontrol.launch_dependents;" :::);
    else
        KS_PDL_ENTRY();
    KS_TL_T0;
    __shared__ long long sh[33];
    __shared__ long long sbase[5];
    __shared__ int s_mg[kPlanThreads];
    if (abort_requested(st)) {
        if (chained) asm volatile("griddepcontrol.wait;" ::: "memory");
        return;
    }
    const int ns = *nseg;
    const int j0 = blockIdx.y * kPlanThreads;
    for (int s = blockIdx.x; s < ns; s += gridDim.x) {
        const Seg g = segs[s];
        if (j0 > g.k) continue;   // block-uniform
        __syncthreads();
        const long long base_i = moff[g.mat_off];
        const int j = j0 + threadIdx.x;
        const bool have = j <= g.k;
        long long ag = 0, gl = 0, ae = 0, el = 0;
        double pv = 0.0;
        if (have) {
            ag = class_start(g, moff, base_i, 2 * j);
            ae = class_start(g, moff, base_i, 2 * j + 1);
            gl = ae - ag;
            if (j < g.k) {
                el = class_start(g, moff, base_i, 2 * j + 2) - ae;
                pv = piv_pool[g.piv_off + j];
            }
        }
        // value range of gap j: (piv[j-1], piv[j]); the ends of the segment: unknown
        const double blo = (have && j > 0) ? piv_pool[g.piv_off + j - 1] : -CUDART_INF;
        const double bhi = (have && j < g.k) ? pv : CUDART_INF;
        const EmitOut o = emit_pairs(have, g.start + ag, gl, g.start + ae, el, pv, dst_id, A, st, sh, sbase, s_mg, blo,
                                     bhi, g.len);
        if (threadIdx.x == 0) {
            // keys of this chunk's classes [2 j0, 2 min(j0 + kPlanThreads, k + 1))
            const int jend = min(j0 + kPlanThreads, g.k + 1);
            const long long len = class_start(g, moff, base_i, 2 * jend) - class_start(g, moff, base_i, 2 * j0);
            account_partition(st, len, o, false);
        }
    }
    KS_TL(25, 8, 0);
    if (chained) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------------------
// local partition: one CTA takes one segment (<= kLocalMax keys, L2-resident)
// and performs the same K-sort multi-level partition without any grid-wide
// step: pivots, shared-memory class histogram, scan, scatter into the other
// buffer, emission of units / next-round segments.  CTAs pull segments from
// a device work counter.
// ---------------------------------------------------------------------------
struct LocalSmem {
    PivotScratch<kPMaxLocal + 1> W;
    double piv[kPMaxLocal + kPivPad];
    unsigned lut[kLutMaxLocal];
    unsigned hist[kRowsMaxLocal + 1];
    unsigned cursor[kRowsMaxLocal + 1];
    long long sh[33];
    long long sbase[5];
    int mg[kLocalThreads];
};

// Partition one local segment (in global memory, L2-resident) with its first
// P keys, classes scattered into the other buffer, children emitted to the
// queues (the same K-sort step as a global pass, by one CTA).  Loads bypass L1:
// the segment may have been written by another SM during this launch.
__device__ void local_one(LocalSmem &L, const Seg &g, const EmitArgs &A, DevStatus *st, double *keys,
                          const double *tmp)
{
    const double *src = (g.src ? tmp : keys) + g.start;
    double *dst = (g.src ? keys : const_cast<double *>(tmp)) + g.start;
    const int dst_id = g.src ? 0 : 1;
    const int m = (int)g.len;
    const int P = pivots_for(m, kPMaxLocal, kKeysPerPivotLocal);
    int k, T;
    double lo, scale;
    KS_TR_DECL;
    build_pivots(src, P, lut_for(P, kLutMaxLocal), L.piv, L.lut, L.W, k, T, lo, scale, pivot_stride(g.stall, m, P));
    KS_TR(0);
    const int rows = 2 * k + 1;
    for (int c = threadIdx.x; c < rows; c += blockDim.x) L.hist[c] = 0;
    __syncthreads();
    constexpr int U = 8;
    int i0 = 0;
    for (; i0 + U * kLocalThreads <= m; i0 += U * kLocalThreads) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcg(src + i0 + u * kLocalThreads + threadIdx.x);
#pragma unroll
        for (int u = 0; u < U; ++u) atomicAdd(&L.hist[classify(v[u], L.piv, L.lut, lo, scale, T)], 1u);
    }
    for (int i = i0 + threadIdx.x; i < m; i += kLocalThreads)
        atomicAdd(&L.hist[classify(__ldcg(src + i), L.piv, L.lut, lo, scale, T)], 1u);
    __syncthreads();
    KS_TR(1);
    {   // exclusive scan of the class histogram -> class starts (2 classes per thread)
        const int c0 = 2 * threadIdx.x;
        const unsigned h0 = c0 < rows ? L.hist[c0] : 0u;
        const unsigned h1 = c0 + 1 < rows ? L.hist[c0 + 1] : 0u;
        const long long ex = block_exclusive_scan((long long)h0 + h1, L.sh, nullptr);
        if (c0 < rows) L.cursor[c0] = (unsigned)ex;
        if (c0 + 1 < rows) L.cursor[c0 + 1] = (unsigned)ex + h0;
    }
    __syncthreads();
    i0 = 0;
    for (; i0 + U * kLocalThreads <= m; i0 += U * kLocalThreads) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_local_last(src + i0 + u * kLocalThreads + threadIdx.x);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = classify(v[u], L.piv, L.lut, lo, scale, T);
            if (!(c & 1)) dst[atomicAdd(&L.cursor[c], 1u)] = v[u];
        }
    }
    for (int i = i0 + threadIdx.x; i < m; i += kLocalThreads) {
        const double v = ld_local_last(src + i);
        const int c = classify(v, L.piv, L.lut, lo, scale, T);
        if (!(c & 1)) dst[atomicAdd(&L.cursor[c], 1u)] = v;
    }
    __threadfence();   // children are published below and may be taken by other SMs at once
    __syncthreads();
    KS_TR(2);
    // class starts = cursor - (keys written); emit per pivot pair
    const int j = threadIdx.x;
    const bool have = j <= k;
    long long ag = 0, gl = 0, ae = 0, el = 0;
    double pv = 0.0;
    if (have) {
        gl = L.hist[2 * j];
        ag = (long long)L.cursor[2 * j] - gl;
        if (j < k) {
            el = L.hist[2 * j + 1];
            ae = (long long)L.cursor[2 * j + 1];   // equality runs are not scattered: cursor = start
            pv = L.piv[j];
        }
    }
    // value range of gap j: (piv[j-1], piv[j]), the segment's own bounds at its ends
    const double blo = (have && j > 0) ? L.piv[j - 1] : (g.bnd ? g.lo : -CUDART_INF);
    const double bhi = (have && j < k) ? pv : (g.bnd ? g.scale : CUDART_INF);
    const EmitOut o = emit_pairs(have, g.start + ag, gl, g.start + ae, el, pv, dst_id, A, st, L.sh, L.sbase, L.mg, blo,
                                 bhi, g.len);
    if (threadIdx.x == 0) account_partition(st, g.len, o, true);
    KS_TR(3);
#ifdef KS_TRACE
    if (threadIdx.x == 0) { atomicAdd(&g_trace[4], 1ull); atomicAdd(&g_trace[5], (unsigned long long)m); }
#endif
}

// ---------------------------------------------------------------------------
// finish (units): one warp per item, many warps per SM.  A unit (a gap and
// its pivot run, <= 512 keys) is loaded coalesced, transposed through the
// warp's shared slice into registers (lane l holds keys l*E..l*E+E-1),
// sorted by the bitonic network (in-register compare-exchange + warp-shuffle
// merges) and stored coalesced into the user buffer.  Fills are written.
// ---------------------------------------------------------------------------
template <int E>
__device__ __forceinline__ void warp_unit_sort(const double *__restrict__ in, double *__restrict__ out, int m,
                                               double *sm)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = e * 32 + lane;
        sm[sidx(i)] = i < m ? in[i] : CUDART_INF;
    }
    __syncwarp();
    double x[E];
#pragma unroll
    for (int r = 0; r < E; ++r) x[r] = sm[sidx(lane * E + r)];
    warp_bitonic_sort<E>(x);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < E; ++r) sm[sidx(lane * E + r)] = x[r];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = e * 32 + lane;
        if (i < m) out[i] = sm[sidx(i)];
    }
    __syncwarp();
}

// One finishing item by one warp: a fill, or a unit (<= kUnitMax keys) sorted
// in registers through the warp's shared slice `sm` (sidx_size(kUnitMax) doubles).
__device__ void finish_item(const Item &it, double *keys, const double *tmp, double *sm)
{
    const int lane = threadIdx.x & 31;
    double *out = keys + it.start;
    const int m = it.len;
    if (it.kind == kItemFill) {
        for (int i = lane; i < m; i += 32) out[i] = it.value;
        return;
    }
    const double *in = (it.src ? tmp : keys) + it.start;
    if (m <= 2) {
        if (lane == 0) {
            const double a = in[0];
            if (m == 2) {
                const double b = in[1];
                out[0] = b < a ? b : a;
                out[1] = b < a ? a : b;
            } else {
                out[0] = a;
            }
        }
    } else if (m <= 32) {
        warp_unit_sort<1>(in, out, m, sm);
    } else if (m <= 64) {
        warp_unit_sort<2>(in, out, m, sm);
    } else if (m <= 128) {
        warp_unit_sort<4>(in, out, m, sm);
    } else if (m <= 256) {
        warp_unit_sort<8>(in, out, m, sm);
    } else {
        warp_unit_sort<16>(in, out, m, sm);
    }
}

// ---------------------------------------------------------------------------
// segment sorter: one CTA sorts one whole segment (kUnitMax < len <=
// kSortMax) on chip and writes it to its final place in the user buffer.
//   1. the segment is read once, coalesced, into registers (kSortPer keys
//      per thread); block min / max
//   2. interpolation buckets b(v) = (v - min) * B / (max - min), B ~ len / 2:
//      the map is monotone in v (see lut_bucket), so bucket order is value
//      order; shared-memory histogram, scan, scatter into the staging buffer
//   3. buckets of <= kThreadSortMax keys: insertion sort by one thread;
//      larger ones: constant-run check, then a warp bitonic network
//      (<= kUnitMax keys); larger non-constant buckets (skewed data) are
//      handed back to the local partitioner, whose first-key pivots do not
//      depend on the value distribution
//   4. coalesced write-back.
// ---------------------------------------------------------------------------
constexpr int kMidCap = 384;   // listed 5..kThreadSortMax-key buckets (single buffer); beyond: the owner sorts
// (5.3% of the B = len/2 buckets hold 5..16 keys: the leaf's 20K-key class needs ~540 entries)
__host__ __device__ constexpr int mid_cap(int c) { return c == 2 ? 1536 : kMidCap; }
constexpr int kMid16Cap = 32;  // ... of them for 9..16-key buckets (rare: Poisson(2) puts 0.02% of buckets there)
#ifndef KS_MID_NET
#define KS_MID_NET 28  // bit c: size class c sorts its 5..8-key buckets with one thread each and an 8-key
#endif                 // network (else a half-warp's ranks). Classes 2, 3, 4 -- the throughput-bound sorters:
                       // C0 -2%, C4 -3.6%; classes 0 / 1 serve latency-bound small calls: C1 +5% with it
template <int C>
struct SortSmem {
    static constexpr int kT = sort_threads(C), kCap = sort_cap(C), kLam = sort_lambda(C);
    // single buffer: the keys are read from global memory (L2) once per pass
    // instead of being held in `a` -- half the shared memory, more sorters per SM
    static constexpr bool kSingle = C == 3 || C == 4 || (C == 2 && KS_SINGLE2);
    // class 0 also finishes the warp units in `a` + `b` (kUnitScratch doubles)
    static constexpr int kUnitScratch = (kT / 32) * sidx_size(kUnitMax);
    static constexpr int kA = !kSingle ? kCap : (C == 4 && kUnitScratch > kCap ? kUnitScratch - kCap : 1);
    static constexpr int kBuckets = kCap / kLam;            // interpolation buckets
    static constexpr int kPB = kBuckets / kT;               // buckets per thread in the scan
    static constexpr int kBigCap = kCap / (kThreadSortMax + 1) + 1;
    double a[kA];          // the segment as loaded (single buffer: unused, or unit scratch)
    alignas(16) double b[kCap + 2];   // bucket order, from b[start & 1] (sorted in place; TMA source)
    unsigned cur[kBuckets];
    int big[kBigCap];
    double red[3][32];     // block min / max / scaled sum
    double bounds[2];      // lo, scale
    int bits;              // bucket map in the order-preserving bit image (wide segments)
    unsigned sh[33];
    int nbig;
    int nmid;              // buckets of 5..8 keys (listed in the free `a` buffer)
    int nmid16;            // buckets of 9..kThreadSortMax keys (listed behind them)
    int nhb;               // hand-back buckets (published once the segment is written)
    int hb[kCap / (kUnitMax + 1) + 1];
    int mid[kSingle ? mid_cap(C) : 1];   // (single buffer: no free `a` for the list)
};

// f(i, key) for every key of in[0, m), kLU loads in flight per thread (L2 only)
template <int kT, int kLU, typename F>
__device__ __forceinline__ void for_keys(const double *in, int m, F &&f)
{
    for (int i0 = 0; i0 < m; i0 += kLU * kT) {
        double x[kLU];
#pragma unroll
        for (int u = 0; u < kLU; ++u) {
            const int i = i0 + u * kT + (int)threadIdx.x;
            x[u] = i < m ? __ldcg(in + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kLU; ++u) {
            const int i = i0 + u * kT + (int)threadIdx.x;
            if (i < m) f(i, x[u]);
        }
    }
}

__device__ __forceinline__ int sort_bucket(double v, double lo, double scale, int B)
{
    const int x = __double2int_rz((v - lo) * scale);
    return min(max(x, 0), B - 1);
}

// Bucket map of the segment sorter: linear in the value, or -- when the
// segment spans many binades (log-like data: linear buckets would overflow) --
// linear in the order-preserving bit image.  Both are monotone in v.
struct BucketMap {
    double lo, scale;
    unsigned long long ulo;
    int bits;
    int B;
    __device__ __forceinline__ int operator()(double v) const
    {
        if (!bits) return sort_bucket(v, lo, scale, B);
        const int x = __double2int_rz((double)(ord_bits(v) - ulo) * scale);
        return min(max(x, 0), B - 1);
    }
};

__device__ __forceinline__ void smem_insertion_sort(double *a, int s)
{
    for (int i = 1; i < s; ++i) {
        const double x = a[i];
        int j = i - 1;
        double y = a[j];
        while (y > x) {
            a[j + 1] = y;
            if (--j < 0) break;
            y = a[j];
        }
        a[j + 1] = x;
    }
}

template <int E>
__device__ __forceinline__ void warp_sort_inplace(double *a, int s)
{
    const int lane = threadIdx.x & 31;
    double x[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int i = lane * E + r;
        x[r] = i < s ? a[i] : CUDART_INF;
    }
    warp_bitonic_sort<E>(x);
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int i = lane * E + r;
        if (i < s) a[i] = x[r];
    }
}

// One warp sorts one bucket in place; false if the bucket is too large (and
// not constant).  Kept out of line: its E = 16 network must not raise the
// register allocation of the streaming loops around it.
__device__ __noinline__ bool warp_sort_bucket(double *a, int sz)
{
    const int lane = threadIdx.x & 31;
    const double f = a[0];
    bool same = true;
    for (int i = lane; i < sz; i += 32) same &= (a[i] == f);
    if (__all_sync(0xffffffffu, same)) return true;
    if (sz <= 32) warp_sort_inplace<1>(a, sz);
    else if (sz <= 64) warp_sort_inplace<2>(a, sz);
    else if (sz <= 128) warp_sort_inplace<4>(a, sz);
    else if (sz <= 256) warp_sort_inplace<8>(a, sz);
    else if (sz <= kUnitMax) warp_sort_inplace<16>(a, sz);
    else return false;
    return true;
}

// Sort one segment (kUnitMax < len <= kSortMax) on chip and write it to its
// final place in the user buffer (see the segment-sorter notes above).
// Item pipeline of the small-segment sorters, run by thread 0 at two points
// of each segment so that it never waits: the next item's claim (an atomic
// issued before the segment) is used after the load phase to start an
// asynchronous copy of its descriptor into shared memory, and after the
// scatter phase the copy is complete and its key ranges are prefetched into L2.
struct NoFeed {
    __device__ __forceinline__ void after_load() {}
    __device__ __forceinline__ void after_scatter() {}
};
struct SegFeed {
    const Seg *list;
    int n;
    int d;           // claimed next item (thread 0)
    Seg *slot;       // its descriptor in shared memory
    int *sidx;
    const double *keys, *tmp;
    bool done;
    bool pf;         // per-item L2 prefetches (off for small, L2-resident calls)
    __device__ __forceinline__ void after_load()
    {
        if (threadIdx.x != 0) return;
        *sidx = d;
        if (d < n) {
            static_assert(sizeof(Seg) % 16 == 0, "descriptor copied in 16-byte pieces");
            const char *src = reinterpret_cast<const char *>(list + d);
            const unsigned dst = (unsigned)__cvta_generic_to_shared(slot);
#pragma unroll
            for (int o = 0; o < (int)sizeof(Seg); o += 16)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + o), "l"(src + o) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    }
    __device__ __forceinline__ void after_scatter()
    {
        if (done) return;
        done = true;
        if (threadIdx.x != 0 || d >= n) return;
        asm volatile("cp.async.wait_all;" ::: "memory");
#if KS_PREFETCH
        if (!pf) return;
        const Seg &g = *slot;
        l2_prefetch((g.src ? tmp : keys) + g.start, 8ull * g.len);
        if (g.src) l2_prefetch(keys + g.start, 8ull * g.len);
#endif
    }
};

template <int C, typename Feed = NoFeed>
__device__ void segsort_one(SortSmem<C> &S, const Seg &g, const LeafQ &Q, DevStatus *st, double *keys,
                            const double *tmp, Feed &&feed = NoFeed{})
{
#ifdef KS_TRACE
    long long tr_t0 = clock64();
#define KS_TRS(slot)                                                                    \
    do {                                                                                \
        if (threadIdx.x == 0) {                                                         \
            long long t1_ = clock64();                                                  \
            atomicAdd(&g_trace[16 + 5 * (C == 3 ? 1 : (C == 4 ? 0 : C)) + (slot)], (unsigned long long)(t1_ - tr_t0)); \
            tr_t0 = t1_;                                                                \
        }                                                                               \
    } while (0)
#else
#define KS_TRS(slot)
#endif
    using Smem = SortSmem<C>;
    constexpr int kT = Smem::kT;
    constexpr int kWarps = kT / 32;
    static_assert(Smem::kPB * kT == Smem::kBuckets, "whole buckets per thread");
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long start = g.start;
    const int m = (int)g.len;
    // bucket-order buffer placed at the segment's global index parity: bb[i] and
    // out[i] share their 16-byte alignment (the sorted segment leaves by TMA)
    double *const bb = S.b + (KS_SEG_TMA ? (int)(start & 1) : 0);
    const double *in = (g.src ? tmp : keys) + start;
    double *out = keys + start;
    constexpr int kLU = kT >= 1024 ? KS_LU1024 : 8;   // loads in flight per thread (one round trip for most segments)
    int B = m / Smem::kLam;
    B = B < 1 ? 1 : (B > Smem::kBuckets ? Smem::kBuckets : B);
    // Bounded item (its keys lie between two of the parent's pivots): the
    // bucket map is known before the load, so the histogram is built while
    // loading (no min / max pass, one barrier fewer).  Else: load + min / max.
    double fscale = 0.0;
    const bool fused = KS_FUSED_HIST && g.bnd && g.scale > g.lo &&
                       !((g.lo > 0.0 && g.scale > 64.0 * g.lo) || (g.scale < 0.0 && g.lo < 64.0 * g.scale)) &&
                       isfinite(fscale = (double)B / (g.scale - g.lo)) && fscale > 0.0;
    if (fused) {
#pragma unroll 1
        for (int b = tid; b < B; b += kT) S.cur[b] = 0u;
        if (tid == 0) {
            S.nbig = 0;
            S.nhb = 0;
        }
        __syncthreads();
        const BucketMap fmap{g.lo, fscale, 0ull, 0, B};
        for (int i0 = 0; i0 < m; i0 += kLU * kT) {
            double x[kLU];
#pragma unroll
            for (int u = 0; u < kLU; ++u) {
                const int i = i0 + u * kT + tid;
                x[u] = i < m ? ld_seg<Smem::kSingle>(in + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kLU; ++u) {
                const int i = i0 + u * kT + tid;
                if (i < m) {
                    if (!Smem::kSingle) S.a[i] = x[u];
                    atomicAdd(&S.cur[fmap(x[u])], 1u);
                }
            }
        }
        __syncthreads();
    }
    double mn = CUDART_INF, mx = -CUDART_INF, sm16 = 0.0;   // (sm16: sum of key * 2^-16, for the mean)
    for (int i0 = 0; !fused && i0 < m; i0 += kLU * kT) {
        double x[kLU];
#pragma unroll
        for (int u = 0; u < kLU; ++u) {
            const int i = i0 + u * kT + tid;
            x[u] = i < m ? ld_seg<Smem::kSingle>(in + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kLU; ++u) {
            const int i = i0 + u * kT + tid;
            if (i < m) {
                if (!Smem::kSingle) S.a[i] = x[u];
                mn = x[u] < mn ? x[u] : mn;
                mx = x[u] > mx ? x[u] : mx;
                sm16 += x[u] * 0x1p-16;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double p = __shfl_xor_sync(0xffffffffu, mn, o), q = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = p < mn ? p : mn;
        mx = q > mx ? q : mx;
        sm16 += __shfl_xor_sync(0xffffffffu, sm16, o);
    }
    if (!fused) {
    if (lane == 0) {
        S.red[0][wid] = mn;
        S.red[1][wid] = mx;
        S.red[2][wid] = sm16;
    }
#pragma unroll 1
    for (int b = tid; b < B; b += kT) S.cur[b] = 0u;
    if (tid == 0) {
        S.nbig = 0;
        S.nhb = 0;
    }
    __syncthreads();
    if (wid == 0) {   // block min / max and the bucket scale, broadcast through shared memory
        mn = lane < kWarps ? S.red[0][lane] : CUDART_INF;
        mx = lane < kWarps ? S.red[1][lane] : -CUDART_INF;
        sm16 = lane < kWarps ? S.red[2][lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double p = __shfl_xor_sync(0xffffffffu, mn, o), q = __shfl_xor_sync(0xffffffffu, mx, o);
            mn = p < mn ? p : mn;
            mx = q > mx ? q : mx;
            sm16 += __shfl_xor_sync(0xffffffffu, sm16, o);
        }
        if (lane == 0) {
            double scale = mx > mn ? (double)B / (mx - mn) : -1.0;            // -1: constant segment
            int bits = 0;
            // many binades: log-like data (bit-image buckets) -- unless the keys do not crowd the
            // small-magnitude end: a mean at least 1/8 of the range away from it (uniform keys down
            // to ~0: the array's lowest gap) keeps the linear map
            const double mean16 = sm16 / (double)m, lo16 = mn * 0x1p-16, hi16 = mx * 0x1p-16;
            const bool spread = mn > 0.0 ? (mean16 - lo16 > (hi16 - lo16) * 0.125) : (hi16 - mean16 > (hi16 - lo16) * 0.125);
            const bool wide = ((mn > 0.0 && mx > 64.0 * mn) || (mx < 0.0 && mn < 64.0 * mx)) && !(KS_SPREAD && spread);
            if (mx > mn && (wide || !(scale > 0.0) || isinf(scale))) {
                bits = 1;   // many binades, or a range the linear map cannot hold
                scale = (double)B / (double)(ord_bits(mx) - ord_bits(mn));
                if (!(scale > 0.0) || isinf(scale)) scale = 0.0;
            }
            S.bounds[0] = mn;
            S.bounds[1] = scale;
            S.bits = bits;
        }
    }
    __syncthreads();
    }
    const double lo = fused ? g.lo : S.bounds[0];
    const double scale = fused ? fscale : S.bounds[1];
    const int bits = fused ? 0 : S.bits;
    KS_TRS(0);   // load + min/max
    feed.after_load();
    if (scale < 0.0) {   // constant segment: already sorted
        if (g.src) {
#pragma unroll 1
            for (int i = tid; i < m; i += kT) out_store(out + (i), Smem::kSingle ? __ldcg(in + i) : S.a[i]);
        }
        feed.after_scatter();
    } else {
        if (scale == 0.0) B = 1;   // one bucket: the warp path (or the partitioner) takes it
        const BucketMap bmap{lo, scale, ord_bits(lo), bits, B};
        // 2. bucket histogram (unless built while loading), scan, scatter a -> b
        if (!fused) {
#pragma unroll 1
            if (Smem::kSingle)
                for_keys<kT, kLU>(in, m, [&](int, double x) { atomicAdd(&S.cur[bmap(x)], 1u); });
            else
                for (int i = tid; i < m; i += kT) atomicAdd(&S.cur[bmap(S.a[i])], 1u);
            __syncthreads();
        }
        KS_TRS(1);   // histogram
#if KS_SEG_TMA
        // the previous segment's bulk store has read bb (rewritten by this
        // segment's scatter, after the scan's barriers): waited as late as possible
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
        {
            const int b0 = tid * Smem::kPB;
            unsigned c[Smem::kPB];
            unsigned t = 0;
#pragma unroll
            for (int e = 0; e < Smem::kPB; ++e) {
                c[e] = b0 + e < B ? S.cur[b0 + e] : 0u;
                t += c[e];
            }
            unsigned ex = block_exclusive_scan_u32(t, S.sh, nullptr);
            unsigned bigmask = 0;
#pragma unroll
            for (int e = 0; e < Smem::kPB; ++e) {
                if (b0 + e < B) S.cur[b0 + e] = ex;
                ex += c[e];
                bigmask |= (c[e] > (unsigned)kThreadSortMax ? 1u : 0u) << e;
            }
            while (bigmask) {   // rare: buckets for the warp path
                const int e = __ffs(bigmask) - 1;
                bigmask &= bigmask - 1;
                S.big[atomicAdd(&S.nbig, 1)] = b0 + e;
            }
        }
        __syncthreads();
        if (Smem::kSingle) {
            for_keys<kT, kLU>(in, m, [&](int, double x) { bb[atomicAdd(&S.cur[bmap(x)], 1u)] = x; });
        } else {
#pragma unroll 1
            for (int i = tid; i < m; i += kT) {
                const double x = S.a[i];
                bb[atomicAdd(&S.cur[bmap(x)], 1u)] = x;
            }
        }
        __syncthreads();
        feed.after_scatter();
        KS_TRS(2);   // scan + scatter
        // 3. cur[b] is now the end of bucket b.  Buckets of more than
        //    kThreadSortMax keys (listed by the scan; none for smooth
        //    inputs) are sorted in place by one warp each.
        const int nbig = S.nbig;
        if (nbig) {
            for (int q = wid; q < nbig; q += kWarps) {
                const int b = S.big[q];
                const int s0 = b ? (int)S.cur[b - 1] : 0;
                const int sz = (int)S.cur[b] - s0;
                if (!warp_sort_bucket(bb + s0, sz) && lane == 0)   // skewed: back to the first-key partitioner
                    S.hb[atomicAdd(&S.nhb, 1)] = b;
            }
            __syncthreads();
        }
#if KS_RANK_LEAF
        // 4. every key of a small bucket takes its rank inside the bucket
        //    (ties by position: equal keys are bitwise equal here) and is
        //    written straight to its final place
#pragma unroll 1
        for (int i = tid; i < m; i += kT) {
            const double x = bb[i];
            const int bk = bmap(x);
            const int e = (int)S.cur[bk];
            const int s0 = bk ? (int)S.cur[bk - 1] : 0;
            int pos = i;
            if (e - s0 > 1 && e - s0 <= kThreadSortMax) {
                int r = s0;
#pragma unroll 1
                for (int j = s0; j < e; ++j) {
                    const double y = bb[j];
                    r += (y < x || (y == x && j < i)) ? 1 : 0;
                }
                pos = r;
            }
            out_store(out + (pos), x);
        }
#else
        // 4a. one thread per bucket: <= 4 keys -> sorting network in registers,
        //     stored straight to the final place; 5..kThreadSortMax keys ->
        //     listed (the `a` buffer is free now) for 4b
        int *mid = Smem::kSingle ? S.mid : reinterpret_cast<int *>(S.a);
        // 5..8-key buckets from the front, 9..16 behind them (KS_MID_NET; else one list)
        constexpr bool kNet = ((KS_MID_NET >> C) & 1) != 0;
        constexpr int kMid8Cap = (Smem::kSingle ? mid_cap(C) : 2 * Smem::kA) - (kNet ? kMid16Cap : 0);
        int *mid16 = mid + kMid8Cap;
        if (tid == 0) {
            S.nmid = 0;
            S.nmid16 = 0;
        }
        __syncthreads();
#pragma unroll 1
        for (int b0 = tid; b0 < B; b0 += 2 * kT) {   // two buckets in flight per thread
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int b = b0 + h * kT;
                if (b >= B) break;
                const int s0 = b ? (int)S.cur[b - 1] : 0;
                const int sz = (int)S.cur[b] - s0;
                if (sz == 0 || sz > kThreadSortMax) continue;
                if (sz > 4) {
                    const bool big16 = kNet && sz > 8;
                    const int q = atomicAdd(big16 ? &S.nmid16 : &S.nmid, 1);
                    if (q < (big16 ? kMid16Cap : kMid8Cap)) {
                        (big16 ? mid16 : mid)[q] = b;
                    } else {   // list full: the owner sorts it
                        smem_insertion_sort(bb + s0, sz);
                        if (!KS_SEG_TMA)
                            for (int i = 0; i < sz; ++i) out_store(out + (s0 + i), bb[s0 + i]);
                    }
                    continue;
                }
                const double *x = bb + s0;
                double x0 = x[0], x1 = sz > 1 ? x[1] : CUDART_INF, x2 = sz > 2 ? x[2] : CUDART_INF,
                       x3 = sz > 3 ? x[3] : CUDART_INF;
                cas(x0, x1, true);
                cas(x2, x3, true);
                cas(x0, x2, true);
                cas(x1, x3, true);
                cas(x1, x2, true);
                double *o = KS_SEG_TMA ? bb + s0 : out + s0;   // (in place: the bulk store writes it)
                o[0] = x0;
                if (sz > 1) o[1] = x1;
                if (sz > 2) o[2] = x2;
                if (sz > 3) o[3] = x3;
            }
        }
        __syncthreads();
        // 4b. 5..kThreadSortMax keys: a half-warp per bucket, lane l takes key l
        //     to its rank in the bucket (ties by position) -- no serial chain
        //     (was: one thread per bucket, insertion sort; 0.377 -> 0.368 ms at C0)
        int nmid;
        if constexpr (kNet) {
            // 4b. 5..8 keys: one thread per bucket, 19-comparator 8-key network in
            //     registers (+inf padding), in place; the rare 9..16-key buckets by
            //     half-warp ranks below (a half-warp per 5..8-key bucket left most
            //     lanes idle: 20% of the sorter's warp instructions for 15% of the keys)
            {
                const int n8 = min(S.nmid, kMid8Cap);
    #pragma unroll 1
                for (int q = tid; q < n8; q += kT) {
                    const int b = mid[q];
                    const int s0 = b ? (int)S.cur[b - 1] : 0;
                    const int sz = (int)S.cur[b] - s0;
                    double *x = bb + s0;
                    double v[8];
    #pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = i < sz ? x[i] : CUDART_INF;
                    cas(v[0], v[2], true); cas(v[1], v[3], true); cas(v[4], v[6], true); cas(v[5], v[7], true);
                    cas(v[0], v[4], true); cas(v[1], v[5], true); cas(v[2], v[6], true); cas(v[3], v[7], true);
                    cas(v[0], v[1], true); cas(v[2], v[3], true); cas(v[4], v[5], true); cas(v[6], v[7], true);
                    cas(v[2], v[4], true); cas(v[3], v[5], true);
                    cas(v[1], v[4], true); cas(v[3], v[6], true);
                    cas(v[1], v[2], true); cas(v[3], v[4], true); cas(v[5], v[6], true);
                    double *o = KS_SEG_TMA ? x : out + s0;
    #pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if (i < sz) o[i] = v[i];
                }
            }
            nmid = min(S.nmid16, kMid16Cap);
            mid = mid16;
        } else {
            nmid = Smem::kSingle ? min(S.nmid, kMid8Cap) : S.nmid;
        }
#if KS_MID_RANK
        static_assert(kThreadSortMax <= 16, "one half-warp lane per key");
#if KS_SEG_TMA
        // in place: both half-warps of a warp run the same iterations, every
        // lane reads before any lane of its warp writes
#pragma unroll 1
        for (int q0 = (tid >> 5) * 2; q0 < nmid; q0 += kT / 16) {
            const int q = q0 + ((tid >> 4) & 1), l = tid & 15;
            int s0 = 0, sz = 0, r = 0;
            double v = 0.0;
            if (q < nmid) {
                const int b = mid[q];
                s0 = b ? (int)S.cur[b - 1] : 0;
                sz = (int)S.cur[b] - s0;
                if (l < sz) {
                    const double *x = bb + s0;
                    v = x[l];
#pragma unroll 4
                    for (int j = 0; j < sz; ++j) {
                        const double y = x[j];
                        r += (y < v || (y == v && j < l)) ? 1 : 0;
                    }
                }
            }
            __syncwarp();
            if (l < sz) bb[s0 + r] = v;
            __syncwarp();
        }
#else
#pragma unroll 1
        for (int q = tid >> 4; q < nmid; q += kT / 16) {
            const int b = mid[q], l = tid & 15;
            const int s0 = b ? (int)S.cur[b - 1] : 0;
            const int sz = (int)S.cur[b] - s0;
            if (l < sz) {
                const double *x = bb + s0;
                const double v = x[l];
                int r = 0;
#pragma unroll 4
                for (int j = 0; j < sz; ++j) {
                    const double y = x[j];
                    r += (y < v || (y == v && j < l)) ? 1 : 0;
                }
                out_store(out + (s0 + r), v);
            }
        }
#endif
#else
#pragma unroll 1
        for (int q = tid; q < nmid; q += kT) {
            const int b = mid[q];
            const int s0 = b ? (int)S.cur[b - 1] : 0;
            const int sz = (int)S.cur[b] - s0;
            smem_insertion_sort(bb + s0, sz);
            for (int i = 0; i < sz; ++i) out_store(out + (s0 + i), bb[s0 + i]);
        }
#endif
        // 4c. large buckets (sorted by warps above, or handed back): coalesced copy
        for (int q = wid; q < nbig && !KS_SEG_TMA; q += kWarps) {
            const int b = S.big[q];
            const int s0 = b ? (int)S.cur[b - 1] : 0;
            const int sz = (int)S.cur[b] - s0;
            for (int i = lane; i < sz; i += 32) out_store(out + (s0 + i), bb[s0 + i]);
        }
#endif
#if KS_SEG_TMA
        // 5. the sorted segment (bb) leaves by one TMA bulk copy (an odd head /
        //    tail key by a plain store); bb is rewritten only by the next
        //    segment's scatter, after its wait for this copy's reads
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        {
            const int h = (int)(start & 1), midn = (m - h) & ~1;
            if (tid == 0 && midn > 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + h),
                             "r"((unsigned)__cvta_generic_to_shared(bb + h)), "r"(8u * (unsigned)midn)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            if (tid == (kT > 32 ? 32 : 0) && h) out[0] = bb[0];
            if (tid == kT - 1 && h + midn < m) out[h + midn] = bb[h + midn];
        }
#endif
        // hand-backs are published only once their keys are in place
        __syncthreads();
        KS_TRS(3);   // big buckets + in-bucket order + write
#if KS_SEG_TMA
        if (S.nhb) {   // (rare) hand-backs are published once the bulk store has landed
            if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            __syncthreads();
        }
#endif
        if (tid < S.nhb) {
            const int b = S.hb[tid];
            const int s0 = b ? (int)S.cur[b - 1] : 0;
            __threadfence();
            hb_push(Q, make_seg(start + s0, (int)S.cur[b] - s0, 0), st);
        }
    }
#ifdef KS_TRACE
    if (threadIdx.x == 0) atomicAdd(&g_trace[16 + 5 * (C == 3 ? 1 : (C == 4 ? 0 : C)) + 4], 1ull);
#endif
#undef KS_TRS
}

// Small segments (size classes 0 and 1): persistent CTAs of the class's own
// shape pull them from a counter after the leaf launch.  Hand-backs go to the
// next leaf launch's queue.
template <int C>
__global__ void __launch_bounds__(sort_threads(C), C == 0 ? KS_MINB0 : (C == 3 ? KS_MINB3 : (C == 4 ? KS_MINB4 : KS_MINB1)))
    k_segsort(const Seg *list, const int *count, int *next, LeafQ Q, DevStatus *st, double *keys, const double *tmp,
              const Item *units, int chained, const Seg *list0, const int *count0, int *next0, int drain0)
{
    // chained: launched programmatically behind the leaf kernel (or behind the
    // other list sorter) and started on the SMs its CTAs leave.  The lists are
    // final once no local partition is queued or running (`pending`, released
    // by the partitioner after its list entries); the grid ahead must still
    // complete before this one does (griddepcontrol.wait at the end).
    if (chained) {
        asm volatile("griddepcontrol.launch_dependents;" :::);
        if (threadIdx.x == 0)
            while (ld_acquire_s32(&st->pending) != 0) __nanosleep(256);
        __syncthreads();
    } else {
        KS_PDL_ENTRY();
    }
    KS_TL_T0;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem<C> &S = *reinterpret_cast<SortSmem<C> *>(smem_raw);
    __shared__ int s_item;
    if (abort_requested(st)) {
        if (chained) asm volatile("griddepcontrol.wait;" ::: "memory");
        return;
    }
    unsigned long long keys_sorted = 0, segs_sorted = 0;
    // thread 0 claims one item ahead and pulls its input and output ranges into
    // L2 while the current one is sorted (a cold segment otherwise costs two
    // DRAM round trips to load and a fill stall per partially written sector)
    const bool pf = !st->no_item_pf;
    __shared__ __align__(16) Seg s_seg[2];
    __shared__ int s_idx[2];
    (void)s_item;
    auto run_list = [&](const Seg *lst, int n, int *nxt) {
        auto prefetch = [&](int d) {
#if KS_PREFETCH
            if (d < n && pf) {
                const Seg g = lst[d];
                l2_prefetch((g.src ? tmp : keys) + g.start, 8ull * g.len);
                if (g.src) l2_prefetch(keys + g.start, 8ull * g.len);
            }
#endif
        };
        // descriptors of the current and the next item in shared memory (see SegFeed)
        __syncthreads();
        if (threadIdx.x == 0) {
            const int d = atomicAdd(nxt, 1);
            s_idx[0] = d;
            if (d < n) {
                s_seg[0] = lst[d];
                prefetch(d);
            }
        }
        for (int slot = 0;; slot ^= 1) {
            __syncthreads();
            if (s_idx[slot] >= n) break;
            const Seg g = s_seg[slot];
            SegFeed f{lst, n, 0, &s_seg[slot ^ 1], &s_idx[slot ^ 1], keys, tmp, false, pf};
            if (threadIdx.x == 0) f.d = atomicAdd(nxt, 1);   // (used after the load phase)
            KS_TL_T0;
            segsort_one<C>(S, g, Q, st, keys, tmp, f);
            f.after_scatter();   // (no-op unless the segment took no scatter path)
            KS_TL(10 + C, 1, g.len);
            keys_sorted += (unsigned long long)g.len;
            segs_sorted += 1;
        }
    };
    run_list(list, *count, next);
    // one large array: the class-0 list after the class-1 list in the same
    // launch (it fills the class-1 sorters' tail; as a kernel of its own behind
    // them it was the sort's last 30 us for 3 us of work)
    if (drain0) run_list(list0, *count0, next0);
#if KS_SEG_TMA
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // (S reused / freed next)
#endif
    if (threadIdx.x == 0 && segs_sorted) {
        add_bytes(st, kPhLeaf, 16ull * keys_sorted);
        atomicAdd(&st->keys_leaf, keys_sorted);
        atomicAdd(&st->leaves, segs_sorted);
    }
    KS_TL(10 + C, 8, keys_sorted);
    if (C == 0 || C == 4 || drain0) {   // the last kernel of the launch also finishes the warp units and fills
        constexpr int kW = sort_threads(C) / 32;
        static_assert(kW * sidx_size(kUnitMax) <= SortSmem<C>::kA + SortSmem<C>::kCap, "unit scratch fits a + b");
        __syncthreads();
        double *sm = (SortSmem<C>::kA > 1 ? S.a : S.b) + (threadIdx.x >> 5) * sidx_size(kUnitMax);   // (a, b contiguous)
        // claimed warp by warp: the CTAs that run out of segments first take them all,
        // the last CTAs find none left (a fixed share per CTA put ~8 us of unit
        // sorts behind the last segment)
        const int nu = st->nunits;
        for (;;) {
            int d = 0;
            if ((threadIdx.x & 31) == 0) d = atomicAdd(&st->unit_next, 1);
            d = __shfl_sync(0xffffffffu, d, 0);
            if (d >= nu) break;
            finish_item(units[d], keys, tmp, sm);
            __syncwarp();
        }
    }
    if (chained) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------------------
// leaf kernel: one persistent CTA per SM drains the local queue (biggest work
// first: each local partition feeds the sort queue) and then the sort queue,
// in one launch -- the long local partitions overlap the segment sorts, and
// the segment sorter's hand-backs are picked up without a host round trip.
// The launch ends when no item is queued or running.
// ---------------------------------------------------------------------------
constexpr int kLeafThreads = 1024;
static_assert(kLocalThreads == kLeafThreads, "the local partitioner runs inside the leaf kernel");
static_assert(sort_threads(2) == kLeafThreads, "the segment sorter runs inside the leaf kernel");

struct LeafCtl {
    Seg seg;
    int kind;   // -1 done, 0 local partition, 1 segment sort
};
constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
constexpr size_t kLeafSmem = cmax(sizeof(SortSmem<2>), sizeof(LocalSmem)) + sizeof(LeafCtl) + 64;
template <int C>
constexpr size_t sort_smem() { return sizeof(SortSmem<C>); }

__global__ void __launch_bounds__(kLeafThreads, 1) k_leaf(EmitArgs A, DevStatus *st, double *keys,
                                                         const double *tmp)
{
    KS_PDL_ENTRY();
    KS_TL_T0;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LeafCtl &ctl = *reinterpret_cast<LeafCtl *>(smem_raw + (kLeafSmem - sizeof(LeafCtl) - 64));
    if (abort_requested(st)) return;
    const LeafQ &Q = A.Q;
    unsigned long long keys_sorted = 0, segs_sorted = 0;
#ifdef KS_TRACE
    long long tr_t0 = clock64();
#endif
    // the plan's local items (all published before this launch): a fixed set
    // (written by the plan, i.e. before this launch: big ones at the front, the rest at the back)
    const int lq_nb = *reinterpret_cast<volatile int *>(&st->lqb_claim);
    const unsigned long long ep = q_epoch(Q);   // (thread 0: ready tags of this launch)
    const int lq_n = lq_nb + *reinterpret_cast<volatile int *>(&st->lq_claim);
    // nothing queued for this launch (small inputs: every gap went to the list
    // sorters): leave at once, the chained list sorters take the SMs
    if (lq_n == 0 && *reinterpret_cast<volatile int *>(&st->sq_claim) == 0) return;
    bool local_phase = true;   // (thread 0 only)
    for (;;) {
        KS_TL_T0;
        if (threadIdx.x == 0) {
            int kind = -1;
            // 1. the plan's local partitions, biggest work first: one ticket each
            if (local_phase) {
                const int idx = atomicAdd(&st->lq_head, 1);
                if (idx < lq_n) {
                    const int slot = idx < lq_nb ? idx : Q.lcap - 1 - (idx - lq_nb);
                    const Seg *q = Q.lq + slot;
                    ctl.seg = load_item(q);
                    kind = kItemLocal;
                } else {
                    local_phase = false;
                }
            }
            // 2. the sort queue: take a ticket, wait until it is published or no
            //    more can come (no local partition queued or running: during a
            //    launch only those produce items -- hand-backs wait for the next
            //    launch -- so the CTA leaves and its SM goes to the list sorters)
            if (kind < 0) {
                const int idx = atomicAdd(&st->sq_head, 1);
                const int slot = idx % Q.scap;
                for (;;) {
                    if (ld_acquire_u64(&Q.sq_ready[slot]) == q_tag(ep, idx)) {
                        const Seg *q = Q.sq + slot;
                        ctl.seg = load_item(q);
                        kind = __ldcg(&q->k);
                        break;
                    }
                    if (idx >= ld_acquire_s32(&st->sq_claim) && ld_acquire_s32(&st->pending) == 0 &&
                        idx >= ld_acquire_s32(&st->sq_claim))
                        break;   // (claims are made before a partition leaves `pending`)
                    __nanosleep(64);
                }
            }
            ctl.kind = kind;
        }
        __syncthreads();
        KS_TR(13);   // item fetch (incl. waiting for work)
        const int kind = ctl.kind;
        KS_TL(2, -1, kind);   // (kind -1: the final wait for pending == 0)
        if (kind < 0) break;
        const Seg g = ctl.seg;
        {
        KS_TL_T0;
        if (kind == kItemLocal) {
            local_one(*reinterpret_cast<LocalSmem *>(smem_raw), g, A, st, keys, tmp);
            KS_TR(14);
        } else {
            segsort_one<2>(*reinterpret_cast<SortSmem<2> *>(smem_raw), g, Q, st, keys, tmp);
#if KS_SEG_TMA
            // the next item may be a local partition, whose tables overlay S.b
            if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
            keys_sorted += (unsigned long long)g.len;
            segs_sorted += 1;
            KS_TR(15);
        }
        KS_TL(2, kind, g.len);
        }
        if (kind == kItemLocal) __threadfence();   // (its children and list entries before `pending` drops)
        __syncthreads();   // this item's children are published; smem free for the next one
        if (threadIdx.x == 0 && kind == kItemLocal) {
            __threadfence();
            atomicSub(&st->pending, 1);
        }
    }
#if KS_SEG_TMA
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
    if (threadIdx.x == 0 && segs_sorted) {
        add_bytes(st, kPhLeaf, 16ull * keys_sorted);
        atomicAdd(&st->keys_leaf, keys_sorted);
        atomicAdd(&st->leaves, segs_sorted);
    }
    KS_TL(2, 8, keys_sorted);
}

// ---------------------------------------------------------------------------
// One small array in ONE cooperative launch (kInitLocalMax < n <= sms *
// kSmallChunk): the eleven dependent launches of the general schedule (rank,
// LUT, count, scan, scatter || plan, leaf, two list sorters, reset) cost
// 3-10 us each whatever the size.  Here every SM takes one contiguous chunk
// of the input and the same K-sort pass runs between grid barriers:
//   0. the first P keys (K-sort's pivots) ranked, a few per CTA; status reset
//      -- barrier --
//   1. distinct pivots in shared memory; every key of the chunk classified by
//      binary search (class 2r: gap below pivot r, 2r+1: equal to pivot r),
//      gated (non-finite, signed zeros) and counted; the chunk's offset
//      inside each gap taken from an atomicAdd on the gap's total (arrival
//      order is as good as chunk order: equal keys are bitwise equal and every
//      gap is sorted below)
//      -- barrier --
//   2. class starts by a scan of the 2k+1 class sizes (every CTA, in shared
//      memory); gap keys scattered to tmp (equality runs are never moved)
//      -- barrier --
//   3. CTA b sorts the gaps that start in [b n/G, (b+1) n/G) on chip
//      (segsort_one, consecutive gaps merged up to kSortMax keys with their
//      pivots' runs) into the user buffer and fills the equality runs.
// Rare leftovers -- a gap above kSortMax keys, a skewed bucket the on-chip
// sorter hands back -- go to the next level's lists; k_leaf_reset behind this
// kernel publishes the status and the host / device loop continues as usual.
// ---------------------------------------------------------------------------
#ifndef KS_SMALL_KPP
#define KS_SMALL_KPP 1024
#endif
#ifndef KS_SMALL_CHUNK
#define KS_SMALL_CHUNK 33792
#endif
constexpr int kSmallChunk = KS_SMALL_CHUNK;   // keys per CTA (their classes are kept in shared memory)
constexpr int kSmallTab = 128;       // gaps per batch of the sort phase
constexpr int kSmallLut = 1024;      // value buckets of the classification's search-range table
struct SmallWords {                  // scratch in the offsets array
    double sorted[kPMax + 1];        // the ranked first P keys
    double piv[kPMax + 2];           // distinct pivots
    unsigned gtot[kPMax + 1];        // keys per gap
    unsigned etot[kPMax + 1];        // keys per equality run
    unsigned cs[2 * kPMax + 4];      // class starts; cs[2k+1] = n
    int k;
};
struct SmallSmem {                   // phases 0-2 (overlaid by SortSmem<2> in phase 3)
    double piv[kPMax + 2];
    unsigned cs[2 * kPMax + 4];      // class histogram of the chunk, then the class starts
    unsigned off[kPMax + 1];         // next destination per gap
    unsigned short cls[kSmallChunk];
    unsigned short lut[kSmallLut + 2];   // lut[t]: pivots whose value bucket is below t (search range of a key in bucket t)
    long long sh[33];
    unsigned shu[33];
};
struct SmallTab {                    // behind SortSmem<2>: the gaps of the current batch
    unsigned gs[kSmallTab], ge[kSmallTab], nx[kSmallTab];   // gap start, gap end (= run start), run end
    double pv[kSmallTab], plo[kSmallTab];                   // the gap's pivot (upper bound), lower bound
    int j0, j1;
    unsigned lo, hi;           // my destination range [b n / G, (b + 1) n / G)
    unsigned pre_start, pre_end;   // the part inside my range of the equality run of the last gap that starts before it
    double pre_pv;
    unsigned maxgap;
};
constexpr size_t kSmallSmemBytes = cmax(sizeof(SortSmem<2>), sizeof(SmallSmem)) + sizeof(SmallTab) + 64;
static_assert(kSmallSmemBytes <= 227 * 1024, "k_small's shared memory");
static_assert(sizeof(SmallSmem) <= sizeof(SortSmem<2>), "the tab sits behind the sorter's buffers");

__global__ void __launch_bounds__(kLeafThreads, 1) k_small(double *keys, double *tmp, long long n, InitLists Lst,
                                                          DevStatus *st, unsigned long long magic, SmallWords *W,
                                                          Seg *gnext, int gnext_cap)
{
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmallSmem &S = *reinterpret_cast<SmallSmem *>(smem_raw);
    SortSmem<2> &SS = *reinterpret_cast<SortSmem<2> *>(smem_raw);
    SmallTab &T = *reinterpret_cast<SmallTab *>(smem_raw + ((sizeof(SortSmem<2>) + 15) & ~size_t(15)));
    const LeafQ &Q = Lst.Q;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int G = gridDim.x, b = blockIdx.x;
    const int P = pivots_for(n, kPMax, KS_SMALL_KPP);   // (more pivots than the general pass: evener shares per CTA)
#ifdef KS_TIMELINE
    unsigned long long tl_p = tl_now();
#define KS_TLP(id)                                   \
    do {                                             \
        if (threadIdx.x == 0) tl_rec(id, 8, 0, tl_p); \
        tl_p = tl_now();                             \
    } while (0)
#else
#define KS_TLP(id)
#endif
    // ---- 0. rank the first P keys; reset the status and the totals ------------------
    if (tid == 0) {   // my chunk into L2 while the pivots are ranked (its loads come two barriers later)
        const long long ch0 = (n + G - 1) / G, b0 = (long long)b * ch0;
        if (b0 < n) l2_prefetch(keys + b0, 8ull * (unsigned long long)min(ch0, n - b0));
    }
    for (int i = tid; i < P; i += kLeafThreads) S.piv[i] = __ldcg(keys + i);
    __syncthreads();
    {
        const int per = (P + G - 1) / G;
        for (int q = wid; q < per; q += kLeafThreads / 32) {
            const int i = b * per + q;
            if (i >= P) break;
            const double v = S.piv[i];
            int r = 0;
            for (int j = lane; j < P; j += 32) {
                const double y = S.piv[j];
                r += (y < v || (y == v && j < i)) ? 1 : 0;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
            if (lane == 0) W->sorted[r] = v;   // (NaN keys -- rejected by the gate -- may collide; all in range)
        }
    }
    if (b == G - 1) {
        seq_advance(Q, magic);
        unsigned long long *w = reinterpret_cast<unsigned long long *>(st);
        for (int i = tid; i < (int)(sizeof(DevStatus) / 8); i += kLeafThreads) w[i] = 0ull;
        __syncthreads();
        if (tid == 0) {
            st->bad_index = kNoIndex;
            st->no_item_pf = 1;
            st->npasses = 1;
        }
    }
    if (b == 0)
        for (int i = tid; i <= P; i += kLeafThreads) W->gtot[i] = W->etot[i] = 0u;
    __threadfence();
    KS_TLP(40);
    grid.sync();
    KS_TLP(44);
    // ---- 1. pivots, classify + gate + count, chunk offsets ---------------------------
    long long carry = 0;
    for (int base = 0; base < P; base += kLeafThreads) {
        const int i = base + tid;
        const double v = i < P ? __ldcg(W->sorted + i) : 0.0;
        const int keep = (i < P && (i == 0 || v != __ldcg(W->sorted + i - 1))) ? 1 : 0;
        long long tot;
        const long long pos = block_exclusive_scan(keep, S.sh, &tot);
        if (keep) S.piv[carry + pos] = v;
        carry += tot;
    }
    const int k = (int)carry;
    const int rows = 2 * k + 1;
    for (int c = tid; c < rows + 1; c += kLeafThreads) S.cs[c] = 0u;
    // search-range table: value buckets t(v) = (v - piv[0]) * scale (monotone in v, saturating, NaN -> 0);
    // pivots of lower buckets are below a key of bucket t, pivots of higher ones above it
    const double lut_lo = k > 0 ? S.piv[0] : 0.0;
    double lut_scale = k > 1 ? (double)kSmallLut / (S.piv[k - 1] - lut_lo) : 0.0;
    if (!(lut_scale > 0.0) || !isfinite(lut_scale)) lut_scale = 0.0;   // (one bucket: plain binary search)
    auto vbucket = [&](double v) { return min(max(__double2int_rz((v - lut_lo) * lut_scale), 0), kSmallLut - 1); };
    for (int t = tid; t <= kSmallLut; t += kLeafThreads) {
        int lo = 0, hi = k;   // first pivot whose bucket is >= t
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (vbucket(S.piv[mid]) < t) lo = mid + 1; else hi = mid;
        }
        S.lut[t] = (unsigned short)lo;
    }
    __syncthreads();
    const long long chunk = (n + G - 1) / G;
    const long long base = (long long)b * chunk;
    const int cnt = (int)max(0ll, min(chunk, n - base));
    {
        long long bad = LLONG_MAX;
        unsigned pz = 0, nz = 0;
        constexpr int kU = 4;
        for (int i0 = 0; i0 < cnt; i0 += kU * kLeafThreads) {
            double v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int i = i0 + u * kLeafThreads + tid;
                v[u] = i < cnt ? __ldcg(keys + base + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int i = i0 + u * kLeafThreads + tid;
                if (i >= cnt) continue;
                gate_one(v[u], base + i, bad, pz, nz);
                const int tb = vbucket(v[u]);
                int lo = S.lut[tb], hi = S.lut[tb + 1];
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (S.piv[mid] < v[u]) lo = mid + 1; else hi = mid;
                }
                const int c = 2 * lo + ((lo < k && S.piv[lo] == v[u]) ? 1 : 0);
                S.cls[i] = (unsigned short)c;
                atomicAdd(&S.cs[c], 1u);
            }
        }
        gate_flush(bad, pz, nz, st);
    }
    __syncthreads();
    for (int g0 = 0; g0 <= k; g0 += 2 * kLeafThreads) {   // (two atomics in flight per thread)
        const int ga = g0 + tid, gb = g0 + kLeafThreads + tid;
        const unsigned ha = ga <= k ? S.cs[2 * ga] : 0u, hb = gb <= k ? S.cs[2 * gb] : 0u;
        const unsigned pa = ha ? atomicAdd(&W->gtot[ga], ha) : 0u;
        const unsigned pb = hb ? atomicAdd(&W->gtot[gb], hb) : 0u;
        if (ga <= k) S.off[ga] = pa;
        if (gb <= k) S.off[gb] = pb;
    }
    for (int j = tid; j < k; j += kLeafThreads) {
        const unsigned h = S.cs[2 * j + 1];
        if (h) atomicAdd(&W->etot[j], h);
    }
    __threadfence();
    KS_TLP(41);
    grid.sync();
    KS_TLP(44);
    // ---- 2. class starts, scatter ------------------------------------------------------
    const bool ab = abort_requested(st);   // (every CTA's gate flags are in: uniform over the grid)
    {
        // sizes of classes 0..2k -> starts (4 per thread, one block scan); cs[2k+1] = n
        unsigned sz[4];
        unsigned t = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = 4 * tid + e;
            sz[e] = c < rows ? ((c & 1) ? __ldcg(&W->etot[c >> 1]) : __ldcg(&W->gtot[c >> 1])) : 0u;
            t += sz[e];
        }
        unsigned ex = block_exclusive_scan_u32(t, S.shu, nullptr);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = 4 * tid + e;
            if (c <= rows) S.cs[c] = ex;
            ex += sz[e];
        }
    }
    if (tid == 0) T.maxgap = 0u;
    __syncthreads();
    for (int g = tid; g <= k; g += kLeafThreads) {
        S.off[g] += S.cs[2 * g];
        atomicMax(&T.maxgap, S.cs[2 * g + 1] - S.cs[2 * g]);
    }
    if (b == 0) {   // for the later batches of the sort phase
        for (int c = tid; c <= rows; c += kLeafThreads) W->cs[c] = S.cs[c];
        for (int j = tid; j < k; j += kLeafThreads) W->piv[j] = S.piv[j];
        if (tid == 0) W->k = k;
    }
    __syncthreads();
    // One gap kept > 3/4 of the keys (presorted, reversed, organ-pipe inputs: the first P keys
    // are no sample of the array): this level is void -- the keys go to tmp as they are and the
    // whole array becomes one stalled segment of the next level, whose pivots are sampled
    // across it (the stall guard of the general pass).
    const bool degenerate = 4ull * T.maxgap > 3ull * (unsigned long long)n;
    if (!ab) {
        constexpr int kU = 4;
        for (int i0 = 0; i0 < cnt; i0 += kU * kLeafThreads) {
            double v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int i = i0 + u * kLeafThreads + tid;
                v[u] = i < cnt ? __ldcg(keys + base + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int i = i0 + u * kLeafThreads + tid;
                if (i >= cnt) continue;
                const unsigned c = S.cls[i];
                if (degenerate) tmp[base + i] = v[u];
                else if (!(c & 1u)) tmp[atomicAdd(&S.off[c >> 1], 1u)] = v[u];
            }
        }
        if (degenerate && b == 0 && tid == 0) {
            Seg c = make_seg(0, n, 1);
            c.stall = 1;
            if (gnext_cap >= 1) gnext[0] = c; else st->overflow = 4;
            st->nseg[1] = 1;
            add_bytes(st, kPhCount, 8ull * (unsigned long long)n);
            add_bytes(st, kPhScatter, 16ull * (unsigned long long)n);
        }
    }
    // my gaps: those that start in [b n / G, (b + 1) n / G); the first batch's table from shared memory
    {
        const unsigned lo_b = (unsigned)(((long long)b * n) / G), hi_b = (unsigned)(((long long)(b + 1) * n) / G);
        if (tid == 0) {
            int lo = 0, hi = k + 1;   // first gap j with cs[2j] >= lo_b
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (S.cs[2 * mid] < lo_b) lo = mid + 1; else hi = mid;
            }
            int j0 = lo;
            hi = k + 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (S.cs[2 * mid] < hi_b) lo = mid + 1; else hi = mid;
            }
            // (a gap of zero keys at the very end starts at n: the last CTA takes it, it has no work)
            T.j0 = degenerate ? 0 : j0;
            T.j1 = degenerate ? 0 : (b == G - 1 ? k + 1 : lo);
            T.lo = lo_b;
            T.hi = b == G - 1 ? (unsigned)n : hi_b;
            // the equality run between the last gap that starts before my range and gap j0 (the first
            // that starts inside it): its owner fills what lies in its own range, I fill my part
            T.pre_start = T.pre_end = lo_b;
            T.pre_pv = 0.0;
            if (!degenerate && j0 >= 1 && j0 - 1 < k) {
                const unsigned r0 = max(S.cs[2 * (j0 - 1) + 1], lo_b), r1 = min(S.cs[2 * (j0 - 1) + 2], T.hi);
                if (r1 > r0) {
                    T.pre_start = r0;
                    T.pre_end = r1;
                    T.pre_pv = S.piv[j0 - 1];
                }
            }
        }
        __syncthreads();
        const int j0 = T.j0, j1 = T.j1;
        for (int t = tid; t < kSmallTab && j0 + t < j1; t += kLeafThreads) {
            const int j = j0 + t;
            T.gs[t] = S.cs[2 * j];
            T.ge[t] = S.cs[2 * j + 1];
            T.nx[t] = j < k ? S.cs[2 * j + 2] : S.cs[2 * j + 1];
            T.pv[t] = j < k ? S.piv[j] : CUDART_INF;
            T.plo[t] = j > 0 ? S.piv[j - 1] : -CUDART_INF;
        }
    }
    __threadfence();
    KS_TLP(42);
    grid.sync();
    KS_TLP(44);
    if (ab) return;
    // ---- 3. sort my gaps ---------------------------------------------------------------
    const int j0 = T.j0, j1 = T.j1;
    const unsigned my_hi = T.hi;
    unsigned long long keys_sorted = 0, segs_sorted = 0, keys_filled = 0;
    // long equality runs are filled range by range: each CTA writes the part inside its own range
    for (unsigned i = T.pre_start + tid; i < T.pre_end; i += kLeafThreads) keys[i] = T.pre_pv;
    keys_filled += T.pre_end - T.pre_start;
    for (int jb = j0; jb < j1; jb += kSmallTab) {
        const int nt = min(kSmallTab, j1 - jb);
        if (jb > j0) {   // later batches: from the arrays CTA 0 left in global memory
            __syncthreads();
            const int kk = __ldcg(&W->k);
            for (int t = tid; t < nt; t += kLeafThreads) {
                const int j = jb + t;
                T.gs[t] = __ldcg(&W->cs[2 * j]);
                T.ge[t] = __ldcg(&W->cs[2 * j + 1]);
                T.nx[t] = j < kk ? __ldcg(&W->cs[2 * j + 2]) : T.ge[t];
                T.pv[t] = j < kk ? __ldcg(&W->piv[j]) : CUDART_INF;
                T.plo[t] = j > 0 ? __ldcg(&W->piv[j - 1]) : -CUDART_INF;
            }
            __syncthreads();
        }
        int t = 0;
        while (t < nt) {   // (uniform over the CTA)
            const unsigned a = T.gs[t];
            unsigned e = T.ge[t];
            int u = t + 1;
            const bool big = e - a > (unsigned)kSortMax;
            if (!big)
                while (u < nt && T.ge[u] - a <= (unsigned)kSortMax) e = T.ge[u++];
            // equality runs: inside the group they are part of its data (tmp); the last one is final
            // (a final run that leaves my range is continued by the CTAs it reaches into)
            for (int q = t; q < u; ++q) {
                const bool inside = q + 1 < u;
                const unsigned r0 = T.ge[q], r1 = inside ? T.nx[q] : min(T.nx[q], max(my_hi, r0));
                double *dstp = inside ? tmp : keys;
                const double pv = T.pv[q];
                for (unsigned i = r0 + tid; i < r1; i += kLeafThreads) dstp[i] = pv;
                keys_filled += r1 - r0;
            }
            const unsigned len = e - a;
            if (big) {   // (rare) more keys than the on-chip sorter holds: the next level takes the gap
                if (tid == 0) {
                    Seg c = make_seg(a, len, 1);
                    c.stall = 4ll * len > 3ll * n ? 1 : 0;   // (presorted, reversed, ...: sampled pivots next)
                    if (len > (unsigned)kLocalMax) {
                        const int gi = atomicAdd(&st->nseg[1], 1);
                        if (gi < gnext_cap) gnext[gi] = c; else st->overflow = 4;
                    } else
                        hb_push(Q, c, st);
                }
            } else if (len > (unsigned)kUnitMax) {
                __syncthreads();   // the fills above and the previous segment's buffers
                segsort_one<2>(SS, make_bseg(a, len, 1, T.plo[t], T.pv[u - 1]), Q, st, keys, tmp);
                keys_sorted += len;
                segs_sorted += 1;
                __syncthreads();
            } else if (len > 0) {
                __syncthreads();
                if (wid == 0) finish_item(make_item(a, len, kItemUnit, 1), keys, tmp, SS.b);
                keys_sorted += len;
                segs_sorted += 1;
                __syncthreads();
            }
            t = u;
        }
    }
    KS_TLP(43);
#undef KS_TLP
    if (tid == 0) {
        add_bytes(st, kPhLeaf, 16ull * keys_sorted + 8ull * keys_filled);
        atomicAdd(&st->keys_leaf, keys_sorted);
        atomicAdd(&st->leaves, segs_sorted);
        if (b == 0 && !degenerate) {
            add_bytes(st, kPhCount, 8ull * (unsigned long long)n);
            add_bytes(st, kPhScatter, 16ull * (unsigned long long)n);
            atomicAdd(&st->keys_partitioned, (unsigned long long)n);
        }
    }
}

// ---------------------------------------------------------------------------
// host plumbing
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// self-check build (KS_CHECK): multiset fingerprint (sum and xor of the bit
// patterns) of the input and of the output, and per-segment sortedness
// ---------------------------------------------------------------------------
struct CheckWords {
    unsigned long long in_sum, in_xor, out_sum, out_xor, unsorted, bad_tile, pad_[2];
};
__global__ void k_check_sum(const double *keys, long long n, unsigned long long *sum, unsigned long long *x)
{
    unsigned long long s = 0, z = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long b = __double_as_longlong(keys[i]);
        s += b;
        z ^= b;
    }
    atomicAdd(sum, s);
    atomicXor(x, z);
}
__global__ void k_check_sorted(const double *keys, long long n, const long long *off, long long nseg,
                               unsigned long long *bad)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x + 1; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (keys[i - 1] <= keys[i]) continue;
        bool boundary = false;   // i starts a segment: no order across segments
        if (off != nullptr) {
            long long lo = 0, hi = nseg;   // any s with off[s] == i
            while (lo < hi) {
                const long long mid = (lo + hi) >> 1;
                if (off[mid] < i) lo = mid + 1; else hi = mid;
            }
            boundary = lo <= nseg && off[lo] == i;
        }
        if (!boundary) atomicAdd(bad, 1ull);
    }
}

static int sm_count()
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

#define KS_CK(x)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) {                                                          \
            fprintf(stderr, "ksort: %s failed: %s\n", #x, cudaGetErrorString(e_));        \
            cudaGetLastError(); /* a non-sticky error must not fail the next call */      \
            return KS_CUDA_ERROR;                                                         \
        }                                                                                 \
    } while (0)

// Launch bookkeeping: counts kernels per phase and, with KS_FLAG_PROFILE,
// brackets each launch with CUDA events on the launching stream.
class Launcher {
  public:
    Launcher(cudaStream_t st, bool prof) : st_(st), prof_(prof) {}
    ~Launcher()
    {
        for (auto &r : recs_) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
    }
    template <typename F>
    void run(int phase, F &&launch)
    {
        Rec r{phase, nullptr, nullptr};
        if (prof_) {
            cudaEventCreate(&r.a);
            cudaEventCreate(&r.b);
            cudaEventRecord(r.a, st_);
        }
        launch();
        if (prof_) {
            cudaEventRecord(r.b, st_);
            recs_.push_back(r);
        }
        ++launches_[phase];
        ++total_;
    }
    void collect(float ms[8], int launches[8]) const
    {
        for (int p = 0; p < 8; ++p) {
            ms[p] = 0.f;
            launches[p] = launches_[p];
        }
        for (const auto &r : recs_) {
            float t = 0.f;
            if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) ms[r.phase] += t;
        }
    }
    int total() const { return total_; }

  private:
    struct Rec {
        int phase;
        cudaEvent_t a, b;
    };
    cudaStream_t st_;
    bool prof_;
    std::vector<Rec> recs_;
    int launches_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int total_ = 0;
};

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its predecessor runs; KS_PDL_ENTRY() in every kernel waits
// for the predecessor's completion before touching its results.
constexpr bool kPdlHeavy = KS_PDL_HEAVY != 0;
// set while the device loop's body is captured: a conditional body holds plain
// kernel / memset nodes only (no programmatic edges, no forked side streams)
static thread_local bool t_in_body = false;

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args &&...args)
{
    if (t_in_body) pdl = false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (KS_PDL && pdl) ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
static cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                          Args &&...args)
{
    return launch_pdl(true, kern, grid, block, smem, stream, std::forward<Args>(args)...);
}

// Small reset kernel (replaces memset nodes, which would break the PDL chain).
struct IntPtrs {
    int *p[8];
};
__global__ void k_set_ints(IntPtrs z)
{
    KS_PDL_ENTRY();
    if (threadIdx.x < 8 && z.p[threadIdx.x]) *z.p[threadIdx.x] = 0;
}

// Status block mirrored into mapped (zero-copy) host memory by the last kernel
// of a leaf launch, then a release of `flag`: the host polls the flag instead
// of queueing a device-to-host copy and synchronising the stream.
struct HostStatus {
    DevStatus st;
    unsigned long long flag;
};

// status block -> mapped host memory, then the flag (one CTA, all threads)
__device__ void publish_status(const DevStatus *st, HostStatus *out)
{
    __syncthreads();
    const unsigned long long *src = reinterpret_cast<const unsigned long long *>(st);
    unsigned long long *dst = reinterpret_cast<unsigned long long *>(&out->st);
    for (int i = threadIdx.x; i < (int)(sizeof(DevStatus) / 8); i += blockDim.x) dst[i] = src[i];
    __syncthreads();   // (the block's stores are ordered before thread 0's system-scope release)
    if (threadIdx.x == 0) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&out->flag), "l"(1ull) : "memory");
}

// End of a leaf launch (all its sorters done): queue and list counters reset,
// the sorters' hand-backs become the next launch's local items.  The host gets
// the status (`out`): after every launch (host loop), or -- under the device
// loop (`use_cond`: this kernel also sets the WHILE node's condition) -- once,
// when no work is left.  gnext: the next level's segment table.
__global__ void k_leaf_reset(LeafQ Q, DevStatus *st, HostStatus *out, cudaGraphConditionalHandle cond, int use_cond,
                             int gnext)
{
    KS_PDL_ENTRY();
    KS_TL_T0;
    const int nhb = min(st->nhb, Q.hb_cap);
    for (int i = threadIdx.x; i < nhb; i += blockDim.x) Q.lq[Q.lcap - 1 - i] = with_kind(Q.hb[i], kItemLocal);
    if (threadIdx.x == 0) {
        st->lq_claim = nhb;
        st->pending = nhb;
        st->nhb = 0;
        st->lq_head = st->lqb_claim = st->sq_claim = st->sq_head = 0;
        st->nsmall[0] = st->nsmall[1] = st->small_next[0] = st->small_next[1] = st->nunits = st->unit_next = 0;
        ++st->nleaves;
    }
    // Device-resident recursion (the reference's worklist, sort_core.py:184-198):
    // more levels while segments or hand-backs are left and the call stands
    __shared__ int s_pub;
    if (threadIdx.x == 0) {
        const bool ab = st->bad_index != kNoIndex || (st->pos_zero && st->neg_zero) || st->bad_arg || st->overflow;
        const bool more = !ab && (st->nseg[gnext] > 0 || nhb > 0);
        if (use_cond) cudaGraphSetConditional(cond, more ? 1u : 0u);
        st->done = more ? 0 : 1;
        s_pub = out != nullptr && (!use_cond || (!more && !st->published));
        if (s_pub && use_cond) st->published = 1;
    }
    __syncthreads();
    if (s_pub) publish_status(st, out);
    KS_TL(27, 8, 0);
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

FastLayout fast_layout(long long n, long long nseg0)
{
    FastLayout L{};
    L.n = n;
    L.seg_cap = (int)(n / (kInitLocalMax + 1) + 2);              // global-pass segments (level 0: > kInitLocalMax)
    // leaf queues: queued items are disjoint ranges of > kUnitMax keys, plus CTAs in flight
    L.lq_cap = (int)(n / (kUnitMax + 1) + nseg0 + 4096);
    L.sq_cap = L.lq_cap;
    L.small_cap[0] = (int)(n / (kUnitMax + 1) + nseg0 + 2);      // disjoint ranges per leaf launch
    L.small_cap[1] = (int)(n / (sort_cap(0) + 1) + nseg0 + 2);
    L.hb_cap = (int)(n / (kUnitMax + 1) + nseg0 + 2);              // hand-backs: disjoint ranges of > kUnitMax keys
    const long long psum = n / kKeysPerPivot + L.seg_cap + 1;    // sum of P_i over one global pass
    L.piv_cap = (int)(psum + L.seg_cap + 1);                     // + one NaN sentinel per segment
    L.lut_cap = (int)(16 * psum + kLutMax);                      // sum of T_i (T_i < 16 P_i)
    // chunks of one pass: sum over segments of cdiv(len, chunk), chunk >= max(kChunkMin, total / items)
    const long long nch = std::max(std::min(n / kChunkMin, (long long)kChunkItemsMax), n / kChunk) + 1;
    L.ch_cap = (int)(nch + L.seg_cap + 1);
    // sum of (P_s + 1)(nch_s + 1) over segments, P_s + 1 <= min(kPMax + 1, len / kKeysPerPivot + 2)
    L.mat_cap = (psum + L.seg_cap) * 2 + (long long)(kPMax + 1) * (nch + 4);
    // warp units and fill items of one leaf launch: disjoint final ranges of > kTinyGap keys
    L.unit_cap = (int)(2 * (n / (kTinyGap + 1)) + n / kFillPiece + nseg0 + 4096);
    L.bsum_cap = cdiv(L.mat_cap, kScanBlock) + 1;
    size_t off = 0;
    L.o_status = off; off = align_up(off + sizeof(DevStatus) + sizeof(CallSeq));   // (CallSeq right behind)
    L.o_seg[0] = off; off = align_up(off + sizeof(Seg) * L.seg_cap);
    L.o_seg[1] = off; off = align_up(off + sizeof(Seg) * L.seg_cap);
    L.o_lq_ready = off; off = align_up(off + sizeof(unsigned long long) * L.lq_cap);   // (ready words contiguous:
    L.o_sq_ready = off; off = align_up(off + sizeof(unsigned long long) * L.sq_cap);   //  one clear per call)
    L.o_lq = off; off = align_up(off + sizeof(Seg) * L.lq_cap);
    L.o_sq = off; off = align_up(off + sizeof(Seg) * L.sq_cap);
    L.o_small[0] = off; off = align_up(off + sizeof(Seg) * L.small_cap[0]);
    L.o_small[1] = off; off = align_up(off + sizeof(Seg) * L.small_cap[1]);
    L.o_hb = off; off = align_up(off + sizeof(Seg) * L.hb_cap);
    L.o_chunk = off; off = align_up(off + sizeof(int) * L.ch_cap);
    L.o_piv = off; off = align_up(off + sizeof(double) * L.piv_cap);
    L.o_lut = off; off = align_up(off + sizeof(unsigned) * L.lut_cap);
    L.o_mat = off; off = align_up(off + sizeof(unsigned) * L.mat_cap);
    L.o_moff = off; off = align_up(off + sizeof(long long) * L.mat_cap);
    L.o_bsum = off; off = align_up(off + sizeof(long long) * L.bsum_cap);
    L.o_units = off; off = align_up(off + sizeof(Item) * L.unit_cap);
    L.o_tmp = off; off = align_up(off + sizeof(double) * (size_t)n);
    L.o_cls = off; off = align_up(off + ((KS_STAGED && KS_CLS) ? sizeof(unsigned short) * (size_t)n : 0));
    L.o_check = off; off = align_up(off + (KS_CHECK ? 64 : 0));
    L.total = off;
    return L;
}

// Per-device launch shapes and kernel attributes, set up once per process
// (cudaFuncSetAttribute / occupancy queries cost host time on every call).
struct EngineCfg {
    int sms, g_count, g_scatter, g_leaf, g_small[2], g_small3, g_small4;
    int g_count2, g_scatter2;
    int coop_ok;   // k_small can run: cooperative launches supported and one CTA per SM fits
};

static const EngineCfg *engine_cfg()
{
    static std::mutex mu;
    static EngineCfg cfgs[64];
    static bool ready[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (ready[dev]) return &cfgs[dev];
    EngineCfg c{};
    bool ok = true;
    auto smem = [&](auto kern, size_t bytes) {
        ok = ok && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess;
    };
    smem(k_scatter, sizeof(ScatterSmem));
    smem(k_pivots, sizeof(PivotsSmem));
    smem(k_count<true>, sizeof(CountSmem));
    smem(k_count<false>, sizeof(CountSmem));
    if (KS_STAGED) {
        smem(k_count2<true>, sizeof(CountSmem));
        smem(k_count2<false>, sizeof(CountSmem));
        smem(k_scatter2, sizeof(Scatter2Smem));
    }
    smem(k_leaf, kLeafSmem);
    const bool small_attr = cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)kSmallSmemBytes) == cudaSuccess;
    if (!small_attr) cudaGetLastError();   // (the general schedule serves every size)
    smem(k_segsort<0>, sort_smem<0>());
    smem(k_segsort<1>, sort_smem<1>());
    smem(k_segsort<3>, sort_smem<3>());
    smem(k_segsort<4>, sort_smem<4>());
    if (!ok) {
        fprintf(stderr, "ksort: cudaFuncSetAttribute failed: %s\n", cudaGetErrorString(cudaGetLastError()));
        return nullptr;
    }
    c.sms = sm_count();
    auto grid = [&](auto kern, int threads, size_t bytes) {
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, bytes);
        return c.sms * (occ > 0 ? occ : 1);
    };
    c.g_count = grid(k_count<false>, kCountThreads, sizeof(CountSmem));
    c.g_scatter = grid(k_scatter, kPassThreads, sizeof(ScatterSmem));
    if (KS_STAGED) {
        c.g_count2 = grid(k_count2<false>, kCount2Threads, sizeof(CountSmem));
        c.g_scatter2 = grid(k_scatter2, kScat2Threads, sizeof(Scatter2Smem));
    }
    c.g_leaf = grid(k_leaf, kLeafThreads, kLeafSmem);
    c.g_small[0] = grid(k_segsort<0>, sort_threads(0), sort_smem<0>());
    c.g_small[1] = grid(k_segsort<1>, sort_threads(1), sort_smem<1>());
    c.g_small3 = grid(k_segsort<3>, sort_threads(3), sort_smem<3>());
    c.g_small4 = grid(k_segsort<4>, sort_threads(4), sort_smem<4>());
    {
        int coop = 0, occ = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        if (small_attr) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_small, kLeafThreads, kSmallSmemBytes);
        c.coop_ok = (small_attr && coop && occ >= 1) ? 1 : 0;
    }
    cfgs[dev] = c;
    ready[dev] = true;
    return &cfgs[dev];
}

// CUDA-graph cache of the speculative schedule.  Its launches depend only on
// the buffers and sizes of the call (the device decides everything else), so a
// repeated call with the same (keys, offsets, workspace, n) replays one graph
// instead of ~20 launches.  Captured on an internal stream (the caller's may
// be the legacy default stream, which cannot capture) and launched on the
// caller's stream.  Small LRU, one per process.
struct GraphKey {
    const void *keys, *d_off, *ws;
    long long n, nseg0;
    size_t ws_bytes;
    const void *hs;   // the calling thread's mapped status block (baked into the graph)
    bool operator==(const GraphKey &o) const
    {
        return keys == o.keys && d_off == o.d_off && ws == o.ws && n == o.n && nseg0 == o.nseg0 &&
               ws_bytes == o.ws_bytes && hs == o.hs;
    }
};
// The executable graph is reference-counted: a thread that evicts an entry
// never destroys a graph another thread has just looked up and is launching.
using GraphExecPtr = std::shared_ptr<CUgraphExec_st>;
struct GraphEntry {
    GraphKey key;
    int dev;
    GraphExecPtr exec;
    int level, gcur, leaves_run, epoch, launches;
    bool has_loop;   // the recursion's remaining levels run in a WHILE node
    unsigned long long last_use;
};
static std::mutex g_graph_mu;
static std::vector<GraphEntry> g_graphs;
static unsigned long long g_graph_clock = 0;
constexpr size_t kGraphCacheMax = 8;

// Copies out of the cache under the lock.  A graph is captured on the second
// call with the same key (a one-off call runs the launches directly: capture
// and instantiation would cost more than they save).
static bool graph_lookup(const GraphKey &k, GraphEntry *out, bool *seen_before)
{
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_graph_mu);
    for (auto &e : g_graphs)
        if (e.dev == dev && e.key == k) {
            e.last_use = ++g_graph_clock;
            *out = e;
            return true;
        }
    static GraphKey seen[kGraphCacheMax];
    static int seen_dev[kGraphCacheMax];
    static size_t seen_next = 0;
    *seen_before = false;
    for (size_t i = 0; i < kGraphCacheMax; ++i)
        if (seen[i] == k && seen_dev[i] == dev) *seen_before = true;
    if (!*seen_before) {
        seen[seen_next % kGraphCacheMax] = k;
        seen_dev[seen_next % kGraphCacheMax] = dev;
        ++seen_next;
    }
    return false;
}

// Keys whose sorts needed more than the speculative levels (presorted,
// reversed, organ-pipe ... inputs): their graphs carry the device loop.  Other
// graphs leave it out -- its WHILE node costs ~5 us per call (measured: C0
// 0.321 -> 0.329 ms) -- and fall back to the host loop if ever needed, which
// marks the key and drops the graph so that the next call recaptures it.
static std::vector<std::pair<GraphKey, int>> g_loop_keys;
static bool key_wants_loop(const GraphKey &k, int dev)
{
    std::lock_guard<std::mutex> lock(g_graph_mu);
    for (auto &x : g_loop_keys)
        if (x.first == k && x.second == dev) return true;
    return false;
}
static void key_mark_loop(const GraphKey &k, int dev)
{
    std::lock_guard<std::mutex> lock(g_graph_mu);
    for (size_t i = 0; i < g_graphs.size(); ++i)
        if (g_graphs[i].dev == dev && g_graphs[i].key == k && !g_graphs[i].has_loop) {
            g_graphs.erase(g_graphs.begin() + i);
            break;
        }
    for (auto &x : g_loop_keys)
        if (x.first == k && x.second == dev) return;
    if (g_loop_keys.size() >= 4 * kGraphCacheMax) g_loop_keys.erase(g_loop_keys.begin());
    g_loop_keys.emplace_back(k, dev);
}

static void graph_store(GraphEntry e)
{
    cudaGetDevice(&e.dev);
    std::lock_guard<std::mutex> lock(g_graph_mu);
    e.last_use = ++g_graph_clock;
    if (g_graphs.size() >= kGraphCacheMax) {
        size_t victim = 0;
        for (size_t i = 1; i < g_graphs.size(); ++i)
            if (g_graphs[i].last_use < g_graphs[victim].last_use) victim = i;
        g_graphs.erase(g_graphs.begin() + victim);
    }
    g_graphs.push_back(e);
}

// Per-thread pinned host copy of the status block (the one read per call).
struct PinnedStatus {
    DevStatus *p = nullptr;
    ~PinnedStatus()
    {
        if (p) cudaFreeHost(p);
    }
};
// Per host thread: a mapped pinned status block (the graph bakes its device
// address in; the graph key carries it, so a graph only ever signals the
// thread that captured it).
struct MappedStatus {
    HostStatus *h = nullptr;
    HostStatus *d = nullptr;
    ~MappedStatus()
    {
        if (h) cudaFreeHost(h);
    }
};
static MappedStatus *mapped_status()
{
    static thread_local MappedStatus ms;
    if (ms.h == nullptr) {
        HostStatus *h = nullptr;
        if (cudaHostAlloc(reinterpret_cast<void **>(&h), sizeof(HostStatus), cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        HostStatus *d = nullptr;
        if (cudaHostGetDevicePointer(reinterpret_cast<void **>(&d), h, 0) != cudaSuccess) {
            cudaGetLastError();
            cudaFreeHost(h);
            return nullptr;
        }
        ms.h = h;
        ms.d = d;
    }
    return &ms;
}

static DevStatus *pinned_status()
{
    static thread_local PinnedStatus ps;
    if (ps.p == nullptr && cudaMallocHost(reinterpret_cast<void **>(&ps.p), sizeof(DevStatus)) != cudaSuccess) {
        cudaGetLastError();
        ps.p = nullptr;
    }
    return ps.p;
}

// Side stream + fork/join events of the calling thread on the current device
// (thread-local: concurrent sorts from different threads never share them).
struct ForkRes {
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
static const ForkRes *fork_res()
{
    if (t_in_body) return nullptr;
    static thread_local ForkRes res[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    ForkRes &r = res[dev];
    if (r.side == nullptr) {
        if (cudaStreamCreateWithFlags(&r.side, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            r = ForkRes{};
            return nullptr;
        }
    }
    return &r;
}

// Capture stream of the calling thread on the current device (thread-local like
// fork_res: two threads capturing their graphs at once never share a stream).
struct CaptureStream {
    cudaStream_t s = nullptr;
};
static cudaStream_t capture_stream()
{
    static thread_local CaptureStream cs[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (cs[dev].s == nullptr && cudaStreamCreateWithFlags(&cs[dev].s, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        cs[dev].s = nullptr;
    }
    return cs[dev].s;
}

static cudaStream_t body_stream()   // captures the device loop's body (per thread and device)
{
    static thread_local CaptureStream cs[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (cs[dev].s == nullptr && cudaStreamCreateWithFlags(&cs[dev].s, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        cs[dev].s = nullptr;
    }
    return cs[dev].s;
}
static std::atomic<int> g_dloop_broken{0};   // a failed device-loop capture: graphs without it from then on
static bool device_loop_ok() { return g_dloop_broken.load() == 0; }

// Staged scatter tiles per SM in one pass.  A tile costs ~3-4 us of fixed work
// (class table, scan, one bulk copy per gap run), so one array gets as few
// tiles per SM as its size allows (tile capacity kStageMax keys: 1 below 2.4M
// keys, 2 below 4.8M, 3 below 7.4M -- 5.5M keys -5%, 6M -4%, 7M -1% against 4);
// larger arrays and batches keep KS_STAGE_ITEMS_PER_SM.
#ifndef KS_TO_LEAF
#define KS_TO_LEAF 0   // measured: 1M +10%, 2M -3% (stragglers: groups up to 2x n / SMs keys); off
#endif
#ifndef KS_TO_LEAF_DIV
#define KS_TO_LEAF_DIV 1
#endif
#ifndef KS_TO_LEAF_CAND4
#define KS_TO_LEAF_CAND4 4
#endif
#ifndef KS_TO_LEAF_MAX_N
#define KS_TO_LEAF_MAX_N 2400000
#endif
#ifndef KS_COOP
#define KS_COOP 1
#endif
#ifndef KS_COOP_MIN_N
#define KS_COOP_MIN_N 2048
#endif
#ifndef KS_COOP_MAX_N
#define KS_COOP_MAX_N 5000000
#endif
#ifndef KS_IPSM1_MAX_N
#define KS_IPSM1_MAX_N 2400000
#endif
#ifndef KS_IPSM2_MAX_N
#define KS_IPSM2_MAX_N 4800000
#endif
#ifndef KS_IPSM3_MAX_N
#define KS_IPSM3_MAX_N 7400000
#endif
static int stage_items_per_sm(long long n, bool batch)
{
    if (batch) return KS_STAGE_ITEMS_PER_SM;
    if (n <= KS_IPSM1_MAX_N) return 1;
    if (n <= KS_IPSM2_MAX_N) return std::min(2, KS_STAGE_ITEMS_PER_SM);
    if (n <= KS_IPSM3_MAX_N) return std::min(3, KS_STAGE_ITEMS_PER_SM);
    return KS_STAGE_ITEMS_PER_SM;
}

int fast_sort(double *keys, long long n, const long long *d_off, long long nseg0, void *ws, size_t ws_bytes,
              cudaStream_t user_stream, bool profile, FastResult *res, double *h_out)
{
    cudaStream_t stream = user_stream;   // (the capture stream while a graph is being recorded)
    FastLayout L = fast_layout(n, nseg0);
    if (ws_bytes < L.total) return KS_WORKSPACE_SMALL;
    if (L.sq_cap >= (1 << kTagIdxBits)) return KS_BAD_ARG;   // (ready tags hold 25-bit claim indices: n < 1.7e10)
    char *w = static_cast<char *>(ws);
    DevStatus *st = reinterpret_cast<DevStatus *>(w + L.o_status);
    Seg *segs[2] = {reinterpret_cast<Seg *>(w + L.o_seg[0]), reinterpret_cast<Seg *>(w + L.o_seg[1])};
    int *chunk_seg = reinterpret_cast<int *>(w + L.o_chunk);
    double *piv = reinterpret_cast<double *>(w + L.o_piv);
    unsigned *lut = reinterpret_cast<unsigned *>(w + L.o_lut);
    unsigned *mat = reinterpret_cast<unsigned *>(w + L.o_mat);
    long long *moff = reinterpret_cast<long long *>(w + L.o_moff);
    long long *bsum = reinterpret_cast<long long *>(w + L.o_bsum);
    Item *units = reinterpret_cast<Item *>(w + L.o_units);
    double *tmp = reinterpret_cast<double *>(w + L.o_tmp);
    unsigned short *cls16 = reinterpret_cast<unsigned short *>(w + L.o_cls);
    LeafQ Q{reinterpret_cast<Seg *>(w + L.o_lq), reinterpret_cast<unsigned long long *>(w + L.o_lq_ready), L.lq_cap,
            reinterpret_cast<Seg *>(w + L.o_sq), reinterpret_cast<unsigned long long *>(w + L.o_sq_ready), L.sq_cap,
            1, {reinterpret_cast<Seg *>(w + L.o_small[0]), reinterpret_cast<Seg *>(w + L.o_small[1])},
            {L.small_cap[0], L.small_cap[1]}, reinterpret_cast<Seg *>(w + L.o_hb), L.hb_cap,
            reinterpret_cast<unsigned *>(w + L.o_status + sizeof(DevStatus))};
    // workspace layout signature (ready words of another layout are stale)
    const unsigned long long ws_magic = 0x4b53525459ull ^ ((unsigned long long)n * 0x9E3779B97F4A7C15ull) ^
                                        ((unsigned long long)nseg0 << 40) ^ (unsigned long long)L.total;

    const EngineCfg *cfg = engine_cfg();
    if (cfg == nullptr) return KS_CUDA_ERROR;
    const int sms = cfg->sms;
    // with the plan forked next to the scatter, the scatter leaves room for the
    // plan's CTAs (level 0: kPlanChunks of them) so that both are resident at once
    const int g_count = cfg->g_count, g_leaf = cfg->g_leaf;
    const int g_scatter = (KS_PLAN_FORK && !profile) ? std::max(cfg->sms, cfg->g_scatter - KS_FORK_ROOM) : cfg->g_scatter;
    const int g_scan = sms * 2;
    // chunks per pass: the staged scatter gives every SM KS_STAGE_ITEMS_PER_SM tiles
    const int pass_items = KS_STAGED ? sms * stage_items_per_sm(n, d_off != nullptr) : std::min(g_count, g_scatter);
    const int g_pivots = sms;
    Launcher K(stream, profile);

    DevStatus h{};
    DevStatus *hp = pinned_status();   // (a pageable destination would add a staged copy)
    // device calls end with the status in mapped host memory (polled; no copy,
    // no stream synchronisation); host destinations (h_out) still synchronise
    // for their copy, profiled calls keep the plain path
    MappedStatus *ms = (KS_MAPPED_STATUS && h_out == nullptr && !profile && !KS_CHECK) ? mapped_status() : nullptr;
    HostStatus *hs_dev = ms ? ms->d : nullptr;
    volatile unsigned long long *hs_flag = ms ? &ms->h->flag : nullptr;
    if (hs_flag) *hs_flag = 0ull;
    int syncs = 0;
    auto sync_status = [&]() -> int {
        KS_CK(cudaGetLastError());
        ++syncs;
        if (hs_flag != nullptr) {
            bool got = false;
            for (unsigned it = 1;; ++it) {
                if (*hs_flag != 0ull) {
                    got = true;
                    break;
                }
                if ((it & 255u) == 0u) {   // a failed launch never raises the flag
                    const cudaError_t q = cudaStreamQuery(stream);
                    if (q == cudaErrorNotReady) continue;
                    if (q != cudaSuccess) return KS_CUDA_ERROR;
                    got = *hs_flag != 0ull;
                    break;
                }
            }
            std::atomic_thread_fence(std::memory_order_acquire);
            if (got) {
                h = ms->h->st;
                *hs_flag = 0ull;   // (armed for the next leaf launch of this call)
                return (h.overflow && !h.bad_arg) ? KS_CUDA_ERROR : KS_OK;
            }
        }
        KS_CK(cudaMemcpyAsync(hp ? hp : &h, st, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream));
        KS_CK(cudaStreamSynchronize(stream));
        if (hp) h = *hp;
        // (an aborted call -- invalid offsets, NaN, mixed zeros -- may leave
        // queued items behind; its own code takes precedence)
        return (h.overflow && !h.bad_arg) ? KS_CUDA_ERROR : KS_OK;
    };
    auto aborted = [&]() { return h.bad_index != kNoIndex || (h.pos_zero && h.neg_zero) || h.bad_arg; };

    const InitLists Lst{segs[0], Q, units, L.seg_cap, L.unit_cap};
    // one small array: rank, count, scatter and the on-chip sorts in one cooperative launch
    const bool coop = KS_COOP && cfg->coop_ok && !profile && d_off == nullptr && n > KS_COOP_MIN_N && n <= KS_COOP_MAX_N &&
                      n <= (long long)sms * kSmallChunk && sizeof(SmallWords) <= sizeof(long long) * (size_t)L.mat_cap &&
                      L.seg_cap >= 1;
    // level 0 of one array: its first P keys ranked into `sorted` (scratch in the
    // offsets array, written only later by the scan)
    bool rank_done = false;
    auto launch_rank = [&](cudaStream_t s) {
        const int P0 = pivots_for(n, kPMax);
        K.run(kPhPivots, [&] {
            launch_pdl(s == stream, k_pivot_rank, dim3((P0 * kRankParts + kRankThreads - 1) / kRankThreads),
                       dim3(kRankThreads), 0, s, keys, P0, reinterpret_cast<double *>(moff));
        });
    };
    auto init_launch = [&]() {
        // batches: queue ready words cleared here, status and call sequence reset
        // (a single array: the init kernel advances the call sequence instead)
        if (d_off != nullptr) {
            cudaMemsetAsync(Q.sq_ready, 0, sizeof(unsigned long long) * L.sq_cap, stream);
            cudaMemsetAsync(st, 0, sizeof(DevStatus) + sizeof(CallSeq), stream);
            cudaMemsetAsync(&st->bad_index, 0xff, sizeof(unsigned long long), stream);
        }
        if (d_off == nullptr) {
            if (n > kInitLocalMax) {   // (+ the level-0 pass bookkeeping)
                // the first P keys ranked, then one launch for the init, the level-0
                // layout and the pivot LUT (PDL: its CTAs wait at griddepcontrol.wait)
                launch_rank(stream);
                K.run(kPhPivots, [&] {
                    launch(k_front_lut, dim3(kLutCtas + 1), dim3(kPivotThreads), 0, stream, n, Lst, st, L.mat_cap, L.ch_cap,
                           L.piv_cap, L.lut_cap, mat, (const long long *)moff,
                           reinterpret_cast<unsigned long long *>(bsum), pass_items, ws_magic,
                           (const double *)reinterpret_cast<double *>(moff), piv, lut, chunk_seg);
                });
                rank_done = true;
            } else
                K.run(kPhGate, [&] { launch(k_init_single, dim3(1), dim3(64), 0, stream, n, Lst, st, ws_magic); });
            if (n <= kInitLocalMax)
                K.run(kPhGate, [&] { launch(k_gate_segments, dim3(sms * 2), dim3(256), 0, stream, keys, nullptr, 0, n, n, st); });
        } else {
            K.run(kPhGate, [&] { launch(k_init_segmented, dim3(sms), dim3(256), 0, stream, d_off, nseg0, n, Lst, st); });
            K.run(kPhGate, [&] { launch(k_gate_segments, dim3(sms * 4), dim3(256), 0, stream, keys, d_off, nseg0, 0, n, st); });
        }
    };

    // The schedule is launched speculatively without host round-trips: global
    // passes read their segment counts on the device (and exit at once when
    // empty), the leaf kernel drains its queues by itself.  One status read at
    // the end; inputs that need more global passes (adversarial shapes:
    // presorted, few distinct values, ...) continue in a synchronising loop.
    int level = 0, gcur = 0, leaves_run = 0;
    cudaGraphConditionalHandle cond_h{};
    bool cond_on = false;            // capturing the device loop: k_leaf_reset sets its condition
    // queue ready words cleared before a level (its plan publishes sort items)
    auto clear_ready = [&]() { cudaMemsetAsync(Q.sq_ready, 0, sizeof(unsigned long long) * L.sq_cap, stream); };
    const int scatter_pf = n >= KS_PF_MIN_N ? 1 : 0;
    // One small array (latency bound: ~1K-key gaps, fewer list items than sorter
    // CTAs): the plan merges consecutive gaps into groups of about n / SMs keys
    // and queues them for the leaf kernel, whose 1024-thread sorter finishes one
    // group per SM in a single wave (1M keys: 30 -> ~12 us for the sorts).
    const int to_leaf = (KS_TO_LEAF && d_off == nullptr && n <= KS_TO_LEAF_MAX_N) ? 1 : 0;
    const int leaf_merge_t = to_leaf ? (int)std::min<long long>(std::max<long long>(n / (sms * KS_TO_LEAF_DIV), 1024), kSortMax / 2 - 256) : 0;
    const int leaf_merge_cand = to_leaf ? std::max(leaf_merge_t * KS_TO_LEAF_CAND4 / 4, 1024) : 0;
    auto global_pass = [&]() {
        const double *src = (level & 1) ? tmp : keys;
        double *dst = (level & 1) ? keys : tmp;
        const int dst_id = (level & 1) ? 0 : 1;
        int *nseg_cur = &st->nseg[gcur];
        // segments at this level: known on the host at level 0, else bounded by the table size
        // (level 0 of one large array: its layout comes from k_front_lut; a
        // small array's first pass -- only ever the device loop's no-op -- is generic)
        const bool first_single = level == 0 && d_off == nullptr && n > kInitLocalMax;
        const long long seg_bound = level == 0 ? (d_off == nullptr ? 1 : nseg0) : L.seg_cap;
        const int gx = (int)(seg_bound < g_pivots ? seg_bound : g_pivots);
        int *nseg_next = &st->nseg[gcur ^ 1];
        // (chained into the scatter's tail for one large array; forked beside the
        // scatter otherwise -- measured: 10M -0.7% chained, 1M and 500 x 100K -1.6% / -0.5% forked)
        const int plan_mode = (profile || t_in_body) ? 0
                              : (KS_PLAN_FORK == 2 && (d_off != nullptr || n < KS_SINGLE_MIN_N)) ? 1 : KS_PLAN_FORK;
        const ForkRes *fr = plan_mode == 1 ? fork_res() : nullptr;
        EmitArgs A{segs[gcur ^ 1], nseg_next, L.seg_cap, Q, units, L.unit_cap, keys, tmp, 0, plan_mode ? 1 : 0,
                   leaf_merge_cand, leaf_merge_t, to_leaf};
        if (!first_single)   // (done by k_front_lut)
            K.run(kPhPivots, [&] {
                launch(k_seg_offsets, dim3(1), dim3(1024), 0, stream, segs[gcur], nseg_cur, st, L.mat_cap, L.ch_cap,
                       L.piv_cap, L.lut_cap, mat, moff, reinterpret_cast<unsigned long long *>(bsum), nseg_next,
                       pass_items);
            });
        if (first_single) {   // one segment, known P: pivots and LUT built by k_front_lut
        } else {
            K.run(kPhPivots, [&] {
                launch(k_pivots, dim3(gx), dim3(kPivotThreads), sizeof(PivotsSmem), stream, segs[gcur], nseg_cur, src,
                       piv, lut, chunk_seg, mat);
            });
        }
        if (KS_STAGED) {
            K.run(kPhCount, [&] {
                launch_pdl(kPdlHeavy, level == 0 ? k_count2<true> : k_count2<false>, dim3(cfg->g_count2),
                           dim3(kCount2Threads), sizeof(CountSmem), stream, segs[gcur], chunk_seg, st, src, piv, lut,
                           mat, st, cls16);
            });
        } else if (level == 0)
            K.run(kPhCount, [&] {
                launch_pdl(kPdlHeavy, k_count<true>, dim3(g_count), dim3(kCountThreads), sizeof(CountSmem), stream, segs[gcur],
                       chunk_seg, st, src, piv, lut, mat, st);
            });
        else
            K.run(kPhCount, [&] {
                launch_pdl(kPdlHeavy, k_count<false>, dim3(g_count), dim3(kCountThreads), sizeof(CountSmem), stream, segs[gcur],
                       chunk_seg, st, src, piv, lut, mat, st);
            });
#if KS_SCAN3
        K.run(kPhScan, [&] { launch(k_scan_reduce, dim3(g_scan), dim3(kScanThreads), 0, stream, mat, st, bsum); });
        K.run(kPhScan, [&] { launch(k_scan_bsums, dim3(1), dim3(1024), 0, stream, bsum, st); });
        K.run(kPhScan, [&] { launch(k_scan_apply, dim3(g_scan), dim3(kScanThreads), 0, stream, mat, st, bsum, moff); });
#else
        K.run(kPhScan, [&] {
            launch(k_scan_lookback, dim3(g_scan), dim3(kScanThreads), 0, stream, mat, st,
                   reinterpret_cast<unsigned long long *>(bsum), moff);
        });
#endif
        auto launch_scatter = [&]() {
            if (KS_STAGED)
                K.run(kPhScatter, [&] {
                    launch_pdl(kPdlHeavy, k_scatter2, dim3(cfg->g_scatter2), dim3(kScat2Threads), sizeof(Scatter2Smem),
                               stream, segs[gcur], chunk_seg, st, src, dst, piv, lut, moff, mat,
                               (const unsigned short *)cls16, KS_STAGED_PF ? scatter_pf : 0);
                });
            else
                K.run(kPhScatter, [&] {
                    launch_pdl(kPdlHeavy, k_scatter, dim3(g_scatter), dim3(kPassThreads), sizeof(ScatterSmem), stream,
                               segs[gcur], chunk_seg, st, src, dst, piv, lut, moff, mat, scatter_pf);
                });
        };
        if (fr != nullptr) {
            // the plan needs only the scanned offsets and the pivots: it runs on a
            // side stream next to the scatter (fork / join; inside the captured graph too)
            cudaEventRecord(fr->fork, stream);
            cudaStreamWaitEvent(fr->side, fr->fork, 0);
            K.run(kPhPlan, [&] {
                launch_pdl(false, k_plan, dim3(gx, kPlanChunks), dim3(kPlanThreads), 0, fr->side, segs[gcur], nseg_cur, piv,
                           moff, A, st, dst_id, 0);
            });
            launch_scatter();
            cudaEventRecord(fr->join, fr->side);
            cudaStreamWaitEvent(stream, fr->join, 0);
        } else {
            // (chained: the plan's CTAs take the SMs the scatter's leave -- forked, they
            // held 16 SMs at the scatter's start and those scatter CTAs ended 10 us late)
            launch_scatter();
            K.run(kPhPlan, [&] {
                launch(k_plan, dim3(gx, kPlanChunks), dim3(kPlanThreads), 0, stream, segs[gcur], nseg_cur, piv, moff, A,
                       st, dst_id, plan_mode == 2 ? 1 : 0);
            });
        }
        ++level;
        gcur ^= 1;
    };
    // leaf launch: queues -> sorted ranges; then the small segments by their own
    // CTA shapes (hand-backs go to the next leaf epoch), the warp units and fills
    // sig: mapped status block the launch's last kernel signals (nullptr: none);
    // clear: the queue's ready words are cleared first (a launch whose epoch
    // may repeat: the device loop's body, the host loop after a replay)
    auto leaf = [&](HostStatus *sig) {
        EmitArgs A{segs[gcur], &st->nseg[gcur], L.seg_cap, Q, units, L.unit_cap, keys, tmp, 1, 0, 0, 0, 0};
        K.run(kPhLeaf, [&] { launch_pdl(kPdlHeavy, k_leaf, dim3(g_leaf), dim3(kLeafThreads), kLeafSmem, stream, A, st, keys, tmp); });
        // the list sorters: chained behind the leaf kernel (programmatic launch),
        // their CTAs take the SMs the leaf's CTAs leave once no local partition is
        // left (the lists are final then; see k_segsort).
        // class-1 list: on large inputs (many segments per CTA slot) the
        // single-buffer sorter (3 per SM, 256 threads) has the higher throughput;
        // on smaller ones the 512-thread sorter's shorter per-segment latency wins
        // (measured: 10M keys -2.4%, 500 x 100K -4.0%; 7M +4.4%, 1M +10%)
        // the two lists are disjoint ranges: on smaller inputs and batches the
        // class-0 sorter (which also finishes the warp units and fills) runs on
        // the side stream next to the class-1 sorter and fills the SMs the
        // class-1 launch's tail leaves idle (measured: 100K keys -12%, 500 x 100K
        // -2.3%); for one large array it is chained behind the class-1 sorter
        const bool chain = KS_LEAF_CHAIN && !profile && !t_in_body;
        const bool sort_fork = KS_SORT_FORK && !profile && (n < KS_SINGLE_MIN_N || d_off != nullptr);
        const ForkRes *fr = sort_fork ? fork_res() : nullptr;
        cudaStream_t s0 = stream;
        if (fr != nullptr) {
            cudaEventRecord(fr->fork, stream);
            cudaStreamWaitEvent(fr->side, fr->fork, 0);
            s0 = fr->side;
        }
        const int ch1 = chain ? 1 : 0, ch0 = (chain && s0 == stream) ? 1 : 0;
        // one large array: the class-1 sorters also drain the class-0 list (and finish the units)
        const int drain0 = (KS_DRAIN0 && n >= KS_SINGLE_MIN_N && fr == nullptr) ? 1 : 0;
        if (n >= KS_SINGLE_MIN_N)
            K.run(kPhLeaf, [&] {
                launch_pdl(chain, k_segsort<3>, dim3(cfg->g_small3), dim3(sort_threads(3)), sort_smem<3>(), stream,
                           Q.small[1], &st->nsmall[1], &st->small_next[1], Q, st, keys, tmp, units, ch1,
                           Q.small[0], &st->nsmall[0], &st->small_next[0], drain0);
            });
        else
            K.run(kPhLeaf, [&] {
                launch_pdl(chain, k_segsort<1>, dim3(cfg->g_small[1]), dim3(sort_threads(1)), sort_smem<1>(), stream,
                           Q.small[1], &st->nsmall[1], &st->small_next[1], Q, st, keys, tmp, units, ch1,
                           Q.small[0], &st->nsmall[0], &st->small_next[0], 0);
            });
        if (drain0) {
        } else if (n >= KS_SINGLE_MIN_N)   // (same trade-off for the class-0 list: 8 single-buffer sorters per SM)
            K.run(kPhLeaf, [&] {
                launch_pdl(ch0 != 0, k_segsort<4>, dim3(cfg->g_small4), dim3(sort_threads(4)), sort_smem<4>(), s0,
                           Q.small[0], &st->nsmall[0], &st->small_next[0], Q, st, keys, tmp, units, ch0,
                           (const Seg *)nullptr, (const int *)nullptr, (int *)nullptr, 0);
            });
        else
            K.run(kPhLeaf, [&] {
                launch_pdl(ch0 != 0, k_segsort<0>, dim3(cfg->g_small[0]), dim3(sort_threads(0)), sort_smem<0>(), s0,
                           Q.small[0], &st->nsmall[0], &st->small_next[0], Q, st, keys, tmp, units, ch0,
                           (const Seg *)nullptr, (const int *)nullptr, (int *)nullptr, 0);
            });
        if (fr != nullptr) {
            cudaEventRecord(fr->join, fr->side);
            cudaStreamWaitEvent(stream, fr->join, 0);
        }
        K.run(kPhGate, [&] {
            launch(k_leaf_reset, dim3(1), dim3(256), 0, stream, Q, st, sig, cond_h, cond_on ? 1 : 0, gcur);
        });
        ++Q.epoch;
        ++leaves_run;
    };
    HostStatus *sig_spec = hs_dev;   // the status block the schedule's leaf launches signal
    bool dloop_failed = false;
    CheckWords *cw = reinterpret_cast<CheckWords *>(w + L.o_check);
    auto spec = [&]() {
        if (KS_CHECK) {
            cudaMemsetAsync(cw, 0, sizeof(CheckWords), stream);
            k_check_sum<<<sms * 4, 256, 0, stream>>>(keys, n, &cw->in_sum, &cw->in_xor);
        }
        if (coop) {
            // one small array: the whole first level in one cooperative launch (see k_small)
            K.run(kPhLeaf, [&] {
                cudaLaunchConfig_t lc = {};
                lc.gridDim = dim3(sms);
                lc.blockDim = dim3(kLeafThreads);
                lc.dynamicSmemBytes = kSmallSmemBytes;
                lc.stream = stream;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                cudaLaunchKernelEx(&lc, k_small, keys, tmp, n, Lst, st, ws_magic, reinterpret_cast<SmallWords *>(moff),
                                   segs[1], L.seg_cap);
            });
            level = 1;
            gcur = 1;
            K.run(kPhGate, [&] {
                launch(k_leaf_reset, dim3(1), dim3(256), 0, stream, Q, st, sig_spec, cond_h, cond_on ? 1 : 0, gcur);
            });
            ++Q.epoch;
            ++leaves_run;
            return;
        }
        init_launch();
        if (n > kInitLocalMax) global_pass();   // (its kernels exit at once when no segment is that long)
        leaf(sig_spec);
    };
    // The rest of the recursion on the device (graph path): a WHILE node whose
    // body runs two more levels (global pass + leaf launch at each parity) as
    // long as k_more finds work; the body's kernels exit at once when a level
    // has nothing to do.
    auto capture_device_loop = [&](cudaStream_t cs) {
        cudaStreamCaptureStatus cst_ = cudaStreamCaptureStatusNone;
        cudaGraph_t g = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t nd = 0;
        if (cudaStreamGetCaptureInfo(cs, &cst_, nullptr, &g, &deps, &nd) != cudaSuccess) {
            dloop_failed = true;
            return;
        }
        cudaGraphNodeParams np{};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = cond_h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t wn = nullptr;
        if (cudaGraphAddNode(&wn, g, deps, nd, &np) != cudaSuccess ||
            cudaStreamUpdateCaptureDependencies(cs, &wn, 1, cudaStreamSetCaptureDependencies) != cudaSuccess) {
            dloop_failed = true;
            return;
        }
        cudaGraph_t body = np.conditional.phGraph_out[0];
        cudaStream_t bs = body_stream();
        if (bs == nullptr || cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0,
                                                           cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            dloop_failed = true;
            return;
        }
        stream = bs;
        t_in_body = true;
        for (int half = 0; half < 2; ++half) {   // (each leaf launch's reset updates the condition)
            clear_ready();   // (this epoch value repeats each iteration)
            global_pass();
            leaf(hs_dev);
        }
        t_in_body = false;
        cudaGraph_t bg = body;
        if (cudaStreamEndCapture(bs, &bg) != cudaSuccess) {
            dloop_failed = true;
            cudaGetLastError();
        }
        stream = cs;
    };
    int launches_graph = 0;
    bool replayed = false;
    if (KS_GRAPH && !profile) {
        // the speculative schedule depends only on (buffers, sizes): replay it as one CUDA graph
        const GraphKey key{keys, d_off, ws, n, nseg0, ws_bytes, hs_dev};
        GraphEntry e{};
        bool seen = false;
        bool have = graph_lookup(key, &e, &seen);
        if (!have && seen) {
            cudaStream_t cs = capture_stream();
            if (cs == nullptr) return KS_CUDA_ERROR;
            e.key = key;
            stream = cs;
            KS_CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            int dev_ = 0;
            cudaGetDevice(&dev_);
            bool dloop = KS_DEVICE_LOOP && device_loop_ok() && (KS_DEVICE_LOOP == 2 || key_wants_loop(key, dev_));
            if (dloop) {
                cudaStreamCaptureStatus cst_ = cudaStreamCaptureStatusNone;
                cudaGraph_t g0 = nullptr;
                dloop = cudaStreamGetCaptureInfo(cs, &cst_, nullptr, &g0) == cudaSuccess &&
                        cudaGraphConditionalHandleCreate(&cond_h, g0, 0, 0) == cudaSuccess;   // (set by every reset)
                if (!dloop) {
                    cudaGetLastError();
                    dloop_failed = true;
                }
            }
            cond_on = dloop;
            spec();
            if (dloop) capture_device_loop(cs);
            cond_on = false;
            cudaGraph_t g = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(cs, &g);
            stream = user_stream;
            if (ce != cudaSuccess) {
                fprintf(stderr, "ksort: graph capture failed: %s\n", cudaGetErrorString(ce));
                cudaGetLastError();
                if (dloop) g_dloop_broken.store(1);
                return KS_CUDA_ERROR;
            }
            cudaGraphExec_t ge = nullptr;
            cudaError_t ie = dloop_failed ? cudaErrorNotSupported : cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
            if (ie != cudaSuccess && dloop) {
                // (the device loop could not be built here: this and later calls run the host loop)
                fprintf(stderr, "ksort: device loop unavailable (%s); using the host loop\n", cudaGetErrorString(ie));
                cudaGetLastError();
                g_dloop_broken.store(1);
                return fast_sort(keys, n, d_off, nseg0, ws, ws_bytes, user_stream, profile, res, h_out);
            }
            KS_CK(ie);
            e.exec = GraphExecPtr(ge, [](cudaGraphExec_t x) { cudaGraphExecDestroy(x); });
            e.level = level;
            e.gcur = gcur;
            e.leaves_run = leaves_run;
            e.epoch = Q.epoch;
            e.launches = K.total();
            e.has_loop = dloop && !dloop_failed;
            graph_store(e);
            have = true;
        }
        if (have) {
            KS_CK(cudaGraphLaunch(e.exec.get(), stream));
            level = e.level;
            gcur = e.gcur;
            leaves_run = e.leaves_run;
            Q.epoch = e.epoch;
            launches_graph = e.launches - K.total();   // (the capture's launches were counted by K)
            replayed = true;
        }
    }
    if (!replayed) spec();
    // host destination: copied behind the speculative schedule (an aborted sort
    // wrote nothing, so the copy returns the caller's own bytes)
    if (h_out != nullptr && n > 0) KS_CK(cudaMemcpyAsync(h_out, keys, 8ull * n, cudaMemcpyDeviceToHost, stream));
    int rc = sync_status();
    if (rc != KS_OK) return rc;
    // remaining work (rare): more global levels, or hand-backs queued for another leaf launch
    bool more = false;
    while (!aborted() && !h.done) {   // (the last reset's verdict: segments or hand-backs left)
        // (after a replay the epoch may repeat one of the device loop's; 4096 leaf
        // launches in one call wrap the tags' epoch field)
        if (replayed || (Q.epoch & ((1 << kTagEpBits) - 1)) == 0) clear_ready();
        if (h.nseg[gcur] > 0) global_pass();
        leaf(hs_dev);
        more = true;
        rc = sync_status();
        if (rc != KS_OK) return rc;
    }
    if (more && KS_GRAPH && !profile) {
        int dev_ = 0;
        cudaGetDevice(&dev_);
        key_mark_loop(GraphKey{keys, d_off, ws, n, nseg0, ws_bytes, hs_dev}, dev_);
    }
    if (more && h_out != nullptr) {
        KS_CK(cudaMemcpyAsync(h_out, keys, 8ull * n, cudaMemcpyDeviceToHost, stream));
        KS_CK(cudaStreamSynchronize(stream));
    }
    if (KS_CHECK && !aborted()) {   // self-check: same multiset, sorted per segment
        k_check_sum<<<sms * 4, 256, 0, stream>>>(keys, n, &cw->out_sum, &cw->out_xor);
        k_check_sorted<<<sms * 4, 256, 0, stream>>>(keys, n, d_off, nseg0, &cw->unsorted);
        CheckWords hc{};
        KS_CK(cudaMemcpyAsync(&hc, cw, sizeof(hc), cudaMemcpyDeviceToHost, stream));
        KS_CK(cudaStreamSynchronize(stream));
        if (hc.in_sum != hc.out_sum || hc.in_xor != hc.out_xor || hc.unsorted || hc.bad_tile) {
            fprintf(stderr, "ksort: self-check failed (n=%lld nseg=%lld): sum %s xor %s unsorted %llu bad_tile %llu\n",
                    n, nseg0, hc.in_sum == hc.out_sum ? "ok" : "DIFF", hc.in_xor == hc.out_xor ? "ok" : "DIFF",
                    hc.unsorted, hc.bad_tile);
            return KS_CUDA_ERROR;
        }
    }
    res->levels = h.npasses + h.nleaves;
    res->host_syncs = syncs;
    res->bad_index = h.bad_index == kNoIndex ? -1 : (long long)h.bad_index;
    res->mixed_zero = (h.pos_zero && h.neg_zero) ? 1 : 0;
    res->bad_arg = h.bad_arg ? 1 : 0;
    res->bytes_moved = h.bytes_moved;
    res->keys_partitioned = h.keys_partitioned;
    res->keys_leaf = h.keys_leaf;
    res->leaves = (long long)h.leaves;
    res->launches = K.total() + launches_graph;
    K.collect(res->phase_ms, res->phase_launches);
    for (int p = 0; p < 8; ++p) res->phase_bytes[p] = h.phase_bytes[p];
    return KS_OK;
}

}  // namespace ks

#ifdef KS_TRACE
extern "C" int ks_trace_read(unsigned long long *out, int n, int reset)
{
    unsigned long long h[32];
    cudaMemcpyFromSymbol(h, ks::g_trace, sizeof(h));
    for (int i = 0; i < n && i < 32; ++i) out[i] = h[i];
    if (reset) {
        unsigned long long z[32] = {0};
        cudaMemcpyToSymbol(ks::g_trace, z, sizeof(z));
    }
    return 0;
}
#endif
#ifdef KS_TIMELINE
namespace ks {
__global__ void k_tl_mark(int id)
{
    KS_TL_T0;
    KS_TL(id, 8, 0);
}
}  // namespace ks
extern "C" int ks_timeline_mark(void *stream, int id)
{
    ks::k_tl_mark<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(id);
    return (int)cudaGetLastError();
}
extern "C" int ks_timeline_read(unsigned long long *out, int max_records, int reset)
{
    unsigned n = 0;
    cudaMemcpyFromSymbol(&n, ks::g_tl_n, sizeof(n));
    if (n > (unsigned)ks::kTlCap) n = ks::kTlCap;
    if ((int)n > max_records) n = max_records;
    if (out && n) cudaMemcpyFromSymbol(out, ks::g_tl, 32ull * n);
    if (reset) {
        unsigned z = 0;
        cudaMemcpyToSymbol(ks::g_tl_n, &z, sizeof(z));
    }
    return (int)n;
}
#endif
