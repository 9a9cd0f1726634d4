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
// scatter -> plan -> finish.  No key crosses to the host; the host reads one
// small status block per pass to decide whether another pass is needed.
#include <cfloat>
#include <cstdio>
#include <vector>

#include "ks_host.h"
#include "ks_internal.cuh"
#include "ks_sortnet.cuh"

namespace ks {

constexpr int kScanBlock = 4096;   // count-matrix entries per scan CTA (512 thr x 8)
constexpr int kScanThreads = 512;

// ---------------------------------------------------------------------------
// finishing-pass work items
// ---------------------------------------------------------------------------
__device__ __forceinline__ Item make_item(long long start, long long len, int kind, int src)
{
    Item it{};
    it.start = start;
    it.len = (int)len;
    it.kind = kind;
    it.src = src;
    return it;
}

// single-lane append (init kernels); the plan kernel reserves ranges per CTA
__device__ __forceinline__ void push_big(DevStatus *st, Item *big, int cap, const Item &it)
{
    int i = atomicAdd(&st->nbig, 1);
    if (i >= cap) { st->overflow = 3; return; }
    big[i] = it;
}

// ---------------------------------------------------------------------------
// init / gate
// ---------------------------------------------------------------------------
__global__ void k_init_single(long long n, Seg *segs, Item *big, DevStatus *st, int cap)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (n > kLeafMax) {
        Seg g{};
        g.start = 0;
        g.len = n;
        segs[0] = g;
        st->nseg[0] = 1;
    } else if (n >= 2) {
        push_big(st, big, cap, make_item(0, n, kItemBig, 0));
        st->keys_leaf = (unsigned long long)n;
        st->leaves = 1;
        add_bytes(st, kPhGate, 8ull * (unsigned long long)n);    // finiteness gate read
        add_bytes(st, kPhLeaf, 16ull * (unsigned long long)n);   // on-chip sort read + write
    }
}

__global__ void k_init_segmented(const long long *off, long long nseg0, Seg *segs, Item *big, DevStatus *st,
                                 int seg_cap, int cap)
{
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nseg0;
         s += (long long)gridDim.x * blockDim.x) {
        long long a = off[s], b = off[s + 1];
        long long len = b - a;
        if (len > kLeafMax) {
            int i = atomicAdd(&st->nseg[0], 1);
            if (i >= seg_cap) { st->overflow = 1; continue; }
            Seg g{};
            g.start = a;
            g.len = len;
            segs[i] = g;
        } else if (len >= 2) {
            push_big(st, big, cap, make_item(a, len, kItemBig, 0));
            atomicAdd(&st->keys_leaf, (unsigned long long)len);
            atomicAdd(&st->leaves, 1ull);
            add_bytes(st, kPhLeaf, 16ull * (unsigned long long)len);
        }
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

// Finiteness gate (sort_core.py:50-59) for keys not covered by a level-0
// count pass: segments of length <= S (they go straight to the finishing pass).
__global__ void k_gate_segments(const double *keys, const long long *off, long long nseg0, long long n_single,
                                DevStatus *st)
{
    long long bad = LLONG_MAX;
    unsigned pz = 0, nz = 0;
    if (off == nullptr) {
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_single;
             i += (long long)gridDim.x * blockDim.x)
            gate_one(keys[i], i, bad, pz, nz);
    } else {
        long long checked = 0;
        for (long long s = blockIdx.x; s < nseg0; s += gridDim.x) {
            long long a = off[s], b = off[s + 1];
            if (b - a > kLeafMax) continue;  // covered by the level-0 count pass
            checked += b - a;
            for (long long i = a + threadIdx.x; i < b; i += blockDim.x) gate_one(keys[i], i, bad, pz, nz);
        }
        if (threadIdx.x == 0) add_bytes(st, kPhGate, 8ull * (unsigned long long)checked);
    }
    gate_flush(bad, pz, nz, st);
}

// ---------------------------------------------------------------------------
// per-pass segment bookkeeping
// ---------------------------------------------------------------------------
__global__ void k_seg_prep(Seg *segs, const int *nseg)
{
    int ns = *nseg;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
        Seg g = segs[s];
        long long P = cdiv(g.len, kKeysPerPivot);
        if (P > kPMax) P = kPMax;
        if (P < 1) P = 1;
        g.P = (int)P;
        g.rows = 2 * g.P + 1;
        g.nch = (int)cdiv(g.len, kChunk);
        g.T = g.P >= 2 ? next_pow2(4 * g.P) : 1;
        if (g.T > kLutMax) g.T = kLutMax;
        segs[s] = g;
    }
}

// One CTA: exclusive scans over segments for pool offsets and matrix layout.
__global__ void k_seg_offsets(Seg *segs, const int *nseg, DevStatus *st, long long mat_cap, int ch_cap,
                              int piv_cap, int lut_cap)
{
    __shared__ long long sh[33];
    int ns = *nseg;
    long long c_piv = 0, c_lut = 0, c_mat = 0, c_ch = 0;
    for (int base = 0; base < ns; base += blockDim.x) {
        int s = base + threadIdx.x;
        Seg g{};
        if (s < ns) g = segs[s];
        const bool in = s < ns;
        long long tp, tl, tm, tc;
        long long xp = block_exclusive_scan(in ? g.P + 1 : 0, sh, &tp);
        long long xl = block_exclusive_scan(in ? g.T : 0, sh, &tl);
        long long xm = block_exclusive_scan(in ? (long long)g.rows * g.nch : 0, sh, &tm);
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
        st->nchunks = (int)c_ch;
        st->mat_total = c_mat;
        add_bytes(st, kPhScan, 16ull * (unsigned long long)c_mat);   // reduce 4B + apply 4B in, 8B out
        add_bytes(st, kPhPivots, 8ull * (unsigned long long)c_piv);  // first P keys of each segment
        if (c_mat > mat_cap || c_ch > ch_cap || c_piv > piv_cap || c_lut > lut_cap) {
            st->overflow = 2;
            st->nchunks = 0;
            st->mat_total = 0;
        }
    }
}

// Pivots of each segment: the first P keys (the top of its K-sort tree),
// sorted and de-duplicated (NaN sentinel after them); plus the bucket LUT
// and the chunk -> segment map.
__global__ void __launch_bounds__(256) k_pivots(Seg *segs, const int *nseg, const double *src, double *piv_pool,
                                                int2 *lut_pool, int *chunk_seg)
{
    __shared__ double sp[kPMaxPow2];
    __shared__ double cp[kPMax + 1];
    __shared__ long long sh[33];
    __shared__ int sk;
    int ns = *nseg;
    for (int s = blockIdx.x; s < ns; s += gridDim.x) {
        __syncthreads();
        Seg g = segs[s];
        const int P = g.P, NP = next_pow2(P);
        for (int i = threadIdx.x; i < NP; i += blockDim.x) sp[i] = i < P ? src[g.start + i] : CUDART_INF;
        __syncthreads();
        for (int kk = 2; kk <= NP; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < NP / 2; i += blockDim.x) {
                    int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1)), hi = lo + j;
                    bool asc = (lo & kk) == 0;
                    double a = sp[lo], b = sp[hi];
                    if ((a > b) == asc) { sp[lo] = b; sp[hi] = a; }
                }
                __syncthreads();
            }
        }
        // de-duplicate (equal keys are one node of the tree: the fat pivot)
        long long carry = 0;
        for (int base = 0; base < P; base += blockDim.x) {
            int i = base + threadIdx.x;
            int keep = (i < P && (i == 0 || sp[i] != sp[i - 1])) ? 1 : 0;
            long long tot;
            long long pos = block_exclusive_scan(keep, sh, &tot);
            if (keep) cp[carry + pos] = sp[i];
            carry += tot;
        }
        if (threadIdx.x == 0) {
            sk = (int)carry;
            cp[carry] = CUDART_NAN;   // sentinel: compares false both ways, even with +/-inf keys
        }
        __syncthreads();
        const int k = sk;
        for (int i = threadIdx.x; i <= k; i += blockDim.x) piv_pool[g.piv_off + i] = cp[i];
        // LUT over the pivot range (monotone bucket map, ks_internal.cuh)
        int T = g.T;
        double lo = cp[0], hi = cp[k - 1], scale = 0.0;
        if (T > 1 && k >= 2 && hi > lo) {
            scale = (double)T / (hi - lo);
            if (!(scale > 0.0) || isinf(scale)) T = 1;
        } else {
            T = 1;
        }
        if (T == 1) scale = 0.0;
        for (int t = threadIdx.x; t < T; t += blockDim.x) {
            // lut[t] = (#{j : bucket(piv_j) < t}, #{j : bucket(piv_j) <= t})
            int a = 0, b = k;
            while (a < b) {
                int mid = (a + b) >> 1;
                if (lut_bucket(cp[mid], lo, scale, T) < t) a = mid + 1; else b = mid;
            }
            int a2 = a, b2 = k;
            while (a2 < b2) {
                int mid = (a2 + b2) >> 1;
                if (lut_bucket(cp[mid], lo, scale, T) <= t) a2 = mid + 1; else b2 = mid;
            }
            lut_pool[g.lut_off + t] = make_int2(a, a2);
        }
        for (int c = threadIdx.x; c < g.nch; c += blockDim.x) chunk_seg[g.ch_off + c] = s;
        if (threadIdx.x == 0) {
            segs[s].k = k;
            segs[s].T = T;
            segs[s].lo = lo;
            segs[s].scale = scale;
        }
    }
}

// ---------------------------------------------------------------------------
// count: per (segment, chunk) class histogram -> class-major count matrix
// (shared-memory atomics: measured ~0.03 SM-cycles/key on B200, far cheaper
// than ballot- or match-based peer aggregation; scripts/mb_hist.cu)
// ---------------------------------------------------------------------------
struct PassSmem {
    double piv[kPMax + 1];
    int2 lut[kLutMax];
};

__device__ __forceinline__ void load_seg(const Seg *segs, int s, const double *piv_pool, const int2 *lut_pool,
                                         Seg &sg, PassSmem &P)
{
    if (threadIdx.x == 0) sg = segs[s];
    __syncthreads();
    for (int i = threadIdx.x; i <= sg.k; i += blockDim.x) P.piv[i] = piv_pool[sg.piv_off + i];
    for (int i = threadIdx.x; i < sg.T; i += blockDim.x) P.lut[i] = lut_pool[sg.lut_off + i];
}

template <bool kGate>
__global__ void __launch_bounds__(kCountThreads) k_count(const Seg *segs, const int *chunk_seg, const DevStatus *cst,
                                                         const double *src, const double *piv_pool,
                                                         const int2 *lut_pool, unsigned *mat, DevStatus *st)
{
    constexpr int U = 8;   // keys in flight per lane
    __shared__ PassSmem P;
    __shared__ unsigned hist[kRowsMax];
    __shared__ Seg sg;
    int cached = -1;
    long long bad = LLONG_MAX;
    unsigned pz = 0, nz = 0;
    const int nchunks = cst->nchunks;
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
        const long long base = sg.start + (long long)j * kChunk;
        const int cnt = (int)min((long long)kChunk, sg.len - (long long)j * kChunk);
        const int T = sg.T;
        const double lo = sg.lo, scale = sg.scale;
        const double *in = src + base;
        for (int i0 = 0; i0 < cnt; i0 += U * kCountThreads) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kCountThreads + threadIdx.x;
                v[u] = i < cnt ? in[i] : 0.0;
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
        for (int c = threadIdx.x; c < sg.rows; c += blockDim.x) mat[sg.mat_off + (long long)c * sg.nch + j] = hist[c];
    }
    if (kGate) gate_flush(bad, pz, nz, st);
}

// ---------------------------------------------------------------------------
// flat exclusive scan of the count matrix -> absolute-within-level offsets
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const unsigned *mat, const DevStatus *st,
                                                              long long *bsum)
{
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

// start of class c inside segment g (relative), c in [0, rows]; rows -> len
__device__ __forceinline__ long long class_start(const Seg &g, const long long *moff, long long base_i, int c)
{
    return c < g.rows ? moff[g.mat_off + (long long)c * g.nch] - base_i : g.len;
}

// ---------------------------------------------------------------------------
// scatter: classify again, rank each key inside its tile (shared atomics),
// group the tile by class in shared memory, then write each class's run
// contiguously to its destination (coalesced runs).  Equality runs of at
// least kFillMin keys are not written: the finishing pass fills them.
// ---------------------------------------------------------------------------
struct ScatterSmem {
    double stage[kTile];
    long long cur[kRowsMax];
    PassSmem P;
    unsigned hist[kRowsMax + 1];
    unsigned off[kRowsMax + 1];
    unsigned short cls[kTile];
    unsigned char skip[kRowsMax + 1];
    long long sh[33];
    Seg sg;
};

__global__ void __launch_bounds__(kPassThreads) k_scatter(const Seg *segs, const int *chunk_seg, const DevStatus *cst,
                                                          const double *src, double *dst, const double *piv_pool,
                                                          const int2 *lut_pool, const long long *moff)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScatterSmem &S = *reinterpret_cast<ScatterSmem *>(smem_raw);
    constexpr int E = kTile / kPassThreads;   // keys per thread per tile (16)
    int cached = -1;
    const int nchunks = cst->nchunks;
    for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int s = chunk_seg[ch];
        __syncthreads();
        if (s != cached) {
            load_seg(segs, s, piv_pool, lut_pool, S.sg, S.P);
            cached = s;
        }
        const Seg &g = S.sg;
        const int j = ch - g.ch_off;
        const long long base = g.start + (long long)j * kChunk;
        const int cnt = (int)min((long long)kChunk, g.len - (long long)j * kChunk);
        const long long base_i = moff[g.mat_off];
        const int rows = g.rows, nch = g.nch, T = g.T;
        const double lo = g.lo, scale = g.scale;
        for (int c = threadIdx.x; c < rows; c += blockDim.x) {
            S.cur[c] = g.start + (moff[g.mat_off + (long long)c * nch + j] - base_i);
            const long long tot = class_start(g, moff, base_i, c + 1) - class_start(g, moff, base_i, c);
            S.skip[c] = ((c & 1) && tot >= kFillMin) ? 1 : 0;
        }
        const double *in = src + base;
        for (int t0 = 0; t0 < cnt; t0 += kTile) {
            const int tcnt = min(kTile, cnt - t0);
            for (int c = threadIdx.x; c < rows; c += blockDim.x) S.hist[c] = 0;
            __syncthreads();
            double v[E];
            unsigned cl[E], rk[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = e * kPassThreads + threadIdx.x;
                v[e] = i < tcnt ? in[t0 + i] : 0.0;
            }
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = e * kPassThreads + threadIdx.x;
                if (i < tcnt) {
                    cl[e] = (unsigned)classify(v[e], S.P.piv, S.P.lut, lo, scale, T);
                    rk[e] = atomicAdd(&S.hist[cl[e]], 1u);
                }
            }
            __syncthreads();
            {   // exclusive scan of the tile histogram: 2 classes per thread
                const int c0 = 2 * threadIdx.x;
                const unsigned h0 = c0 < rows ? S.hist[c0] : 0u;
                const unsigned h1 = c0 + 1 < rows ? S.hist[c0 + 1] : 0u;
                const long long ex = block_exclusive_scan((long long)h0 + h1, S.sh, nullptr);
                if (c0 < rows) S.off[c0] = (unsigned)ex;
                if (c0 + 1 < rows) S.off[c0 + 1] = (unsigned)ex + h0;
            }
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = e * kPassThreads + threadIdx.x;
                if (i < tcnt) {
                    const unsigned p = S.off[cl[e]] + rk[e];
                    S.stage[p] = v[e];
                    S.cls[p] = (unsigned short)cl[e];
                }
            }
            __syncthreads();
            for (int p = threadIdx.x; p < tcnt; p += blockDim.x) {
                const int c = S.cls[p];
                if (!S.skip[c]) dst[S.cur[c] + (p - (long long)S.off[c])] = S.stage[p];
            }
            __syncthreads();
            for (int c = threadIdx.x; c < rows; c += blockDim.x) S.cur[c] += S.hist[c];
        }
    }
}

// ---------------------------------------------------------------------------
// plan: turn class extents into next-pass segments and finishing work.
// Each thread owns one pivot j (<= 512 per segment): the gap below it (class
// 2j) and its equality run (class 2j+1).  A gap of <= kUnitMax keys plus its
// short equality run is one warp unit; longer equality runs are fills; gaps
// of kUnitMax+1..S keys are CTA "big" items; larger gaps become segments of
// the next pass.  Items are reserved per CTA with one atomic per list.
// ---------------------------------------------------------------------------
constexpr int kPlanThreads = 512;

__global__ void __launch_bounds__(kPlanThreads) k_plan(const Seg *segs, const int *nseg, const double *piv_pool,
                                                       const long long *moff, Seg *next, int *nnext, Item *units,
                                                       Item *big, DevStatus *st, int dst_id, int seg_cap,
                                                       int unit_cap, int big_cap)
{
    __shared__ long long sh[33];
    __shared__ long long sbase[3];
    static_assert(kPMax + 1 <= kPlanThreads, "one pivot pair per thread");
    const int ns = *nseg;
    for (int s = blockIdx.x; s < ns; s += gridDim.x) {
        __syncthreads();
        const Seg g = segs[s];
        const long long base_i = moff[g.mat_off];
        const int j = threadIdx.x;
        const bool have = j <= g.k;
        long long ag = 0, gl = 0, ae = 0, el = 0;
        if (have) {
            ag = class_start(g, moff, base_i, 2 * j);
            ae = class_start(g, moff, base_i, 2 * j + 1);
            gl = ae - ag;
            if (j < g.k) el = class_start(g, moff, base_i, 2 * j + 2) - ae;
        }
        const bool eq_written = el > 0 && el < kFillMin;   // the scatter wrote these keys
        // decide this pair's items
        int u_gap = 0, b_gap = 0, n_gap = 0, u_eq = 0, f_eq = 0;
        long long ulen_gap = gl;
        if (gl >= 2 || (gl == 1 && dst_id == 1)) {
            if (gl <= kUnitMax) {
                u_gap = 1;
                if (eq_written && gl + el <= kUnitMax) ulen_gap += el;
            } else if (gl <= kLeafMax) {
                b_gap = 1;
            } else {
                n_gap = 1;
            }
        }
        const bool eq_packed = u_gap && ulen_gap > gl;
        if (el >= kFillMin) f_eq = 1;
        else if (eq_written && !eq_packed && dst_id == 1) u_eq = 1;
        const int nu = u_gap + u_eq + f_eq;
        long long tu, tb, tn;
        const long long xu = block_exclusive_scan(nu, sh, &tu);
        const long long xb = block_exclusive_scan(b_gap, sh, &tb);
        const long long xn = block_exclusive_scan(n_gap, sh, &tn);
        if (threadIdx.x == 0) {
            sbase[0] = tu ? atomicAdd(&st->nunits, (int)tu) : 0;
            sbase[1] = tb ? atomicAdd(&st->nbig, (int)tb) : 0;
            sbase[2] = tn ? atomicAdd(nnext, (int)tn) : 0;
        }
        __syncthreads();
        long long ui = sbase[0] + xu;
        if (u_gap) {
            if (ui < unit_cap) units[ui] = make_item(g.start + ag, ulen_gap, kItemUnit, dst_id);
            else st->overflow = 3;
            ++ui;
        }
        if (u_eq) {
            if (ui < unit_cap) units[ui] = make_item(g.start + ae, el, kItemUnit, dst_id);
            else st->overflow = 3;
            ++ui;
        }
        if (f_eq) {
            Item it = make_item(g.start + ae, el, kItemFill, dst_id);
            it.value = piv_pool[g.piv_off + j];
            if (ui < unit_cap) units[ui] = it;
            else st->overflow = 3;
        }
        if (b_gap) {
            const long long bi = sbase[1] + xb;
            if (bi < big_cap) big[bi] = make_item(g.start + ag, gl, kItemBig, dst_id);
            else st->overflow = 5;
        }
        if (n_gap) {
            const long long ni = sbase[2] + xn;
            if (ni < seg_cap) {
                Seg n2{};
                n2.start = g.start + ag;
                n2.len = gl;
                next[ni] = n2;
            } else {
                st->overflow = 4;
            }
        }
        // algorithmic bytes (count reads 8B/key; scatter reads 8B/key and writes 8B
        // per key it places; units/big read+write 16B/key; fills write 8B/key)
        const long long fk = f_eq ? el : 0;
        const long long uk = (u_gap ? ulen_gap : 0) + (u_eq ? el : 0);
        const long long bk = b_gap ? gl : 0;
        long long t_fk, t_uk, t_bk;
        block_exclusive_scan(fk, sh, &t_fk);
        block_exclusive_scan(uk, sh, &t_uk);
        block_exclusive_scan(bk, sh, &t_bk);
        if (threadIdx.x == 0) {
            add_bytes(st, kPhCount, 8ull * g.len);
            add_bytes(st, kPhScatter, 8ull * g.len + 8ull * (g.len - t_fk));
            add_bytes(st, kPhLeaf, 16ull * (t_uk + t_bk) + 8ull * t_fk);
            atomicAdd(&st->keys_partitioned, (unsigned long long)g.len);
            atomicAdd(&st->keys_leaf, (unsigned long long)(t_uk + t_bk));
            atomicAdd(&st->leaves, (unsigned long long)(tu + tb));
        }
    }
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

__global__ void __launch_bounds__(kUnitWarps * 32, 3) k_finish_units(const Item *units, const DevStatus *cst,
                                                                     double *keys, const double *tmp)
{
    __shared__ double sm_all[kUnitWarps][sidx_size(kUnitMax)];
    if (abort_requested(cst)) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double *sm = sm_all[wid];
    const int n = cst->nunits;
    for (int d = blockIdx.x * kUnitWarps + wid; d < n; d += gridDim.x * kUnitWarps) {
        const Item it = units[d];
        double *out = keys + it.start;
        const int m = it.len;
        if (it.kind == kItemFill) {
            for (int i = lane; i < m; i += 32) out[i] = it.value;
            continue;
        }
        const double *in = (it.src ? tmp : keys) + it.start;
        if (m <= 2) {
            if (lane == 0) {
                double a = in[0];
                if (m == 2) {
                    double b = in[1];
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
}

// ---------------------------------------------------------------------------
// finish (big): one CTA per gap of kUnitMax+1 .. S keys: 16 warps sort runs of
// N/16 keys in registers, then four merge-path passes in shared memory.
// ---------------------------------------------------------------------------
struct BigSmem {
    double s[sidx_size(kLeafMax)];
};

template <int E>
__device__ __forceinline__ void warp_sort_smem(double *s, int off, int m)
{
    // sort s[off .. off+m) (sidx layout) in place with one warp, m <= 32*E
    const int lane = threadIdx.x & 31;
    double x[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int i = lane * E + r;
        x[r] = i < m ? s[sidx(off + i)] : CUDART_INF;
    }
    warp_bitonic_sort<E>(x);
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int i = lane * E + r;
        if (i < m) s[sidx(off + i)] = x[r];
    }
}

// block sort of s[0..N) (N = 512*E, padded with +inf): 16 warps x (32E-key runs), then merge passes
template <int E>
__device__ __forceinline__ void block_sort_smem(double *s)
{
    constexpr int N = 512 * E;
    const int wid = threadIdx.x >> 5;
    warp_sort_smem<E>(s, wid * 32 * E, 32 * E);
    __syncthreads();
#pragma unroll 1
    for (int size = 32 * E; size < N; size <<= 1) {
        const int o = threadIdx.x * E;
        const int g0 = o & ~(2 * size - 1);
        const int dg = o - g0;
        const int a = merge_path(s, g0, g0 + size, size, dg);
        double y[E];
        merge_serial<E>(s, g0, g0 + size, size, a, dg - a, y);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < E; ++r) s[sidx(o + r)] = y[r];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kBigThreads) k_finish_big(const Item *big, const DevStatus *cst, double *keys,
                                                            const double *tmp)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BigSmem &F = *reinterpret_cast<BigSmem *>(smem_raw);
    if (abort_requested(cst)) return;
    const int n = cst->nbig;
    for (int d = blockIdx.x; d < n; d += gridDim.x) {
        const Item it = big[d];
        const double *in = (it.src ? tmp : keys) + it.start;
        double *out = keys + it.start;
        const int m = it.len;
        __syncthreads();
        if (m <= kUnitMax) {   // initial small segments
            const int lane = threadIdx.x & 31;
            if (threadIdx.x < 32) {
                if (m <= 32) warp_unit_sort<1>(in, out, m, F.s);
                else if (m <= 64) warp_unit_sort<2>(in, out, m, F.s);
                else if (m <= 128) warp_unit_sort<4>(in, out, m, F.s);
                else if (m <= 256) warp_unit_sort<8>(in, out, m, F.s);
                else warp_unit_sort<16>(in, out, m, F.s);
            }
            (void)lane;
            continue;
        }
        const int N = next_pow2(m);
        for (int i = threadIdx.x; i < N; i += blockDim.x) F.s[sidx(i)] = i < m ? in[i] : CUDART_INF;
        __syncthreads();
        if (N <= 1024) block_sort_smem<2>(F.s);
        else if (N <= 2048) block_sort_smem<4>(F.s);
        else if (N <= 4096) block_sort_smem<8>(F.s);
        else block_sort_smem<16>(F.s);
        for (int i = threadIdx.x; i < m; i += blockDim.x) out[i] = F.s[sidx(i)];
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

FastLayout fast_layout(long long n, long long nseg0)
{
    FastLayout L{};
    L.n = n;
    L.seg_cap = (int)(n / (kLeafMax + 1) + 2);
    const long long psum = n / kKeysPerPivot + L.seg_cap + 1;    // sum of P_i  (P_i <= ceil(len/64))
    L.piv_cap = (int)(psum + L.seg_cap + 1);                     // + one NaN sentinel per segment
    L.lut_cap = (int)(8 * psum + kLutMax);                       // sum of T_i (T_i < 8 P_i)
    L.ch_cap = (int)(n / kChunk + L.seg_cap + 1);
    L.mat_cap = (2 * psum + L.seg_cap) + (long long)(2 * kPMax + 1) * (2 * (n / kChunk) + 2);
    L.unit_cap = (int)(2 * psum + 2 * L.seg_cap + 2);            // <= 2 items per pivot pair
    L.big_cap = (int)(n / (kUnitMax + 1) + nseg0 + 2);
    L.bsum_cap = cdiv(L.mat_cap, kScanBlock) + 1;
    size_t off = 0;
    L.o_status = off; off = align_up(off + sizeof(DevStatus));
    L.o_seg[0] = off; off = align_up(off + sizeof(Seg) * L.seg_cap);
    L.o_seg[1] = off; off = align_up(off + sizeof(Seg) * L.seg_cap);
    L.o_chunk = off; off = align_up(off + sizeof(int) * L.ch_cap);
    L.o_piv = off; off = align_up(off + sizeof(double) * L.piv_cap);
    L.o_lut = off; off = align_up(off + sizeof(int2) * L.lut_cap);
    L.o_mat = off; off = align_up(off + sizeof(unsigned) * L.mat_cap);
    L.o_moff = off; off = align_up(off + sizeof(long long) * L.mat_cap);
    L.o_bsum = off; off = align_up(off + sizeof(long long) * L.bsum_cap);
    L.o_units = off; off = align_up(off + sizeof(Item) * L.unit_cap);
    L.o_big = off; off = align_up(off + sizeof(Item) * L.big_cap);
    L.o_tmp = off; off = align_up(off + sizeof(double) * (size_t)n);
    L.total = off;
    return L;
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

int fast_sort(double *keys, long long n, const long long *d_off, long long nseg0, void *ws, size_t ws_bytes,
              cudaStream_t stream, bool profile, FastResult *res)
{
    FastLayout L = fast_layout(n, nseg0);
    if (ws_bytes < L.total) return KS_WORKSPACE_SMALL;
    char *w = static_cast<char *>(ws);
    DevStatus *st = reinterpret_cast<DevStatus *>(w + L.o_status);
    Seg *segs[2] = {reinterpret_cast<Seg *>(w + L.o_seg[0]), reinterpret_cast<Seg *>(w + L.o_seg[1])};
    int *chunk_seg = reinterpret_cast<int *>(w + L.o_chunk);
    double *piv = reinterpret_cast<double *>(w + L.o_piv);
    int2 *lut = reinterpret_cast<int2 *>(w + L.o_lut);
    unsigned *mat = reinterpret_cast<unsigned *>(w + L.o_mat);
    long long *moff = reinterpret_cast<long long *>(w + L.o_moff);
    long long *bsum = reinterpret_cast<long long *>(w + L.o_bsum);
    Item *units = reinterpret_cast<Item *>(w + L.o_units);
    Item *big = reinterpret_cast<Item *>(w + L.o_big);
    double *tmp = reinterpret_cast<double *>(w + L.o_tmp);

    KS_CK(cudaFuncSetAttribute(k_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ScatterSmem)));
    KS_CK(cudaFuncSetAttribute(k_finish_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BigSmem)));
    const int sms = sm_count();
    int occ_count = 1, occ_scatter = 1, occ_units = 1, occ_big = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_count, k_count<false>, kCountThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_scatter, k_scatter, kPassThreads, sizeof(ScatterSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_units, k_finish_units, kUnitWarps * 32, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_big, k_finish_big, kBigThreads, sizeof(BigSmem));
    const int g_count = sms * (occ_count > 0 ? occ_count : 1);
    const int g_scatter = sms * (occ_scatter > 0 ? occ_scatter : 1);
    const int g_units = sms * (occ_units > 0 ? occ_units : 1);
    const int g_big = sms * (occ_big > 0 ? occ_big : 1);
    const int g_scan = sms * 2;
    const int g_seg = sms * 4;
    Launcher K(stream, profile);

    DevStatus h{};
    KS_CK(cudaMemsetAsync(st, 0, sizeof(DevStatus), stream));
    KS_CK(cudaMemsetAsync(&st->bad_index, 0xff, sizeof(unsigned long long), stream));

    if (d_off == nullptr) {
        K.run(kPhGate, [&] { k_init_single<<<1, 32, 0, stream>>>(n, segs[0], big, st, L.big_cap); });
        if (n <= kLeafMax)
            K.run(kPhGate, [&] { k_gate_segments<<<sms, 256, 0, stream>>>(keys, nullptr, 0, n, st); });
    } else {
        K.run(kPhGate, [&] {
            k_init_segmented<<<sms, 256, 0, stream>>>(d_off, nseg0, segs[0], big, st, L.seg_cap, L.big_cap);
        });
        K.run(kPhGate, [&] { k_gate_segments<<<sms * 4, 256, 0, stream>>>(keys, d_off, nseg0, 0, st); });
    }
    KS_CK(cudaGetLastError());
    KS_CK(cudaMemcpyAsync(&h, st, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream));
    KS_CK(cudaStreamSynchronize(stream));
    if (h.overflow) return KS_CUDA_ERROR;

    int level = 0;
    int cur = 0;
    bool finished_once = false;
    while (h.nseg[cur] > 0) {
        const double *src = (level & 1) ? tmp : keys;
        double *dst = (level & 1) ? keys : tmp;
        const int dst_id = (level & 1) ? 0 : 1;
        int *nseg_cur = &st->nseg[cur];
        int *nseg_next = &st->nseg[cur ^ 1];
        K.run(kPhPivots, [&] { k_seg_prep<<<g_seg, 256, 0, stream>>>(segs[cur], nseg_cur); });
        K.run(kPhPivots, [&] {
            k_seg_offsets<<<1, 1024, 0, stream>>>(segs[cur], nseg_cur, st, L.mat_cap, L.ch_cap, L.piv_cap, L.lut_cap);
        });
        K.run(kPhPivots, [&] { k_pivots<<<g_seg, 256, 0, stream>>>(segs[cur], nseg_cur, src, piv, lut, chunk_seg); });
        if (level == 0)
            K.run(kPhCount, [&] {
                k_count<true><<<g_count, kCountThreads, 0, stream>>>(segs[cur], chunk_seg, st, src, piv, lut, mat, st);
            });
        else
            K.run(kPhCount, [&] {
                k_count<false><<<g_count, kCountThreads, 0, stream>>>(segs[cur], chunk_seg, st, src, piv, lut, mat, st);
            });
        K.run(kPhScan, [&] { k_scan_reduce<<<g_scan, kScanThreads, 0, stream>>>(mat, st, bsum); });
        K.run(kPhScan, [&] { k_scan_bsums<<<1, 1024, 0, stream>>>(bsum, st); });
        K.run(kPhScan, [&] { k_scan_apply<<<g_scan, kScanThreads, 0, stream>>>(mat, st, bsum, moff); });
        K.run(kPhScatter, [&] {
            k_scatter<<<g_scatter, kPassThreads, sizeof(ScatterSmem), stream>>>(segs[cur], chunk_seg, st, src, dst, piv,
                                                                               lut, moff);
        });
        KS_CK(cudaMemsetAsync(nseg_next, 0, sizeof(int), stream));
        K.run(kPhPlan, [&] {
            k_plan<<<g_seg, kPlanThreads, 0, stream>>>(segs[cur], nseg_cur, piv, moff, segs[cur ^ 1], nseg_next, units,
                                                       big, st, dst_id, L.seg_cap, L.unit_cap, L.big_cap);
        });
        K.run(kPhLeaf, [&] { k_finish_units<<<g_units, kUnitWarps * 32, 0, stream>>>(units, st, keys, tmp); });
        K.run(kPhLeaf, [&] {
            k_finish_big<<<g_big, kBigThreads, sizeof(BigSmem), stream>>>(big, st, keys, tmp);
        });
        finished_once = true;
        KS_CK(cudaMemsetAsync(&st->nunits, 0, 2 * sizeof(int), stream));   // nunits, nbig
        KS_CK(cudaGetLastError());
        KS_CK(cudaMemcpyAsync(&h, st, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream));
        KS_CK(cudaStreamSynchronize(stream));
        ++level;
        cur ^= 1;
        if (h.overflow) return KS_CUDA_ERROR;
        if (h.bad_index != kNoIndex || (h.pos_zero && h.neg_zero)) break;
    }
    if (!finished_once) {
        K.run(kPhLeaf, [&] {
            k_finish_big<<<g_big, kBigThreads, sizeof(BigSmem), stream>>>(big, st, keys, tmp);
        });
        KS_CK(cudaGetLastError());
        KS_CK(cudaMemcpyAsync(&h, st, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream));
        KS_CK(cudaStreamSynchronize(stream));
    }
    res->levels = level;
    res->bad_index = h.bad_index == kNoIndex ? -1 : (long long)h.bad_index;
    res->mixed_zero = (h.pos_zero && h.neg_zero) ? 1 : 0;
    res->bytes_moved = h.bytes_moved;
    res->keys_partitioned = h.keys_partitioned;
    res->keys_leaf = h.keys_leaf;
    res->leaves = (long long)h.leaves;
    res->launches = K.total();
    K.collect(res->phase_ms, res->phase_launches);
    for (int p = 0; p < 8; ++p) res->phase_bytes[p] = h.phase_bytes[p];
    return KS_OK;
}

}  // namespace ks
