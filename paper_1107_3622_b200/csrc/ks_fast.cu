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
//   leaf sorter, larger gaps become the next pass's segments.
//
// Kernels per pass: seg_prep -> seg_offsets -> pivots -> count -> scan (3) ->
// scatter -> plan -> leaf.  No data crosses to the host; the host reads one
// small status block per pass to decide whether another pass is needed.
#include <cfloat>
#include <cstdio>
#include <vector>

#include "ks_host.h"
#include "ks_internal.cuh"

namespace ks {

constexpr int kScanBlock = 4096;   // count-matrix entries per scan CTA (512 thr x 8)
constexpr int kScanThreads = 512;

// ---------------------------------------------------------------------------
// init / gate
// ---------------------------------------------------------------------------
__global__ void k_init_single(long long n, Seg *segs, Leaf *leaves, DevStatus *st)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (n > kLeafMax) {
        Seg g{};
        g.start = 0;
        g.len = n;
        segs[0] = g;
        st->nseg[0] = 1;
    } else if (n >= 2) {
        Leaf L{};
        L.start = 0;
        L.len = n;
        L.kind = kLeafSort;
        L.src = 0;
        leaves[0] = L;
        st->nleaf = 1;
        st->keys_leaf = (unsigned long long)n;
        st->leaves = 1;
        add_bytes(st, kPhGate, 8ull * (unsigned long long)n);    // finiteness gate read
        add_bytes(st, kPhLeaf, 16ull * (unsigned long long)n);   // leaf read + write
    }
}

__global__ void k_init_segmented(const long long *off, long long nseg0, Seg *segs, Leaf *leaves,
                                 DevStatus *st, int seg_cap, int leaf_cap)
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
            int i = atomicAdd(&st->nleaf, 1);
            if (i >= leaf_cap) { st->overflow = 1; continue; }
            Leaf L{};
            L.start = a;
            L.len = len;
            L.kind = kLeafSort;
            L.src = 0;
            leaves[i] = L;
            atomicAdd(&st->keys_leaf, (unsigned long long)len);
            atomicAdd(&st->leaves, 1ull);
            add_bytes(st, kPhLeaf, 16ull * (unsigned long long)len);
        }
    }
}

__device__ __forceinline__ void gate_one(double v, long long idx, long long &bad, unsigned &pz,
                                         unsigned &nz)
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
// count pass: segments of length <= S (they go straight to the leaf sorter).
__global__ void k_gate_segments(const double *keys, const long long *off, long long nseg0,
                                long long n_single, DevStatus *st)
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
        long long P = cdiv(g.len * kGapsPerLeaf, kLeafMax);
        if (P > kPMax) P = kPMax;
        if (P < 1) P = 1;
        g.P = (int)P;
        g.rows = 2 * g.P + 1;
        g.nch = (int)cdiv(g.len, kChunk);
        g.T = g.P >= 4 ? next_pow2(2 * g.P) : 1;
        if (g.T > kLutMax) g.T = kLutMax;
        segs[s] = g;
    }
}

// One CTA: exclusive scans over segments for pool offsets and matrix layout.
__global__ void k_seg_offsets(Seg *segs, const int *nseg, DevStatus *st, long long mat_cap,
                              int ch_cap, int piv_cap, int lut_cap)
{
    __shared__ long long sh[33];
    int ns = *nseg;
    long long c_piv = 0, c_lut = 0, c_mat = 0, c_ch = 0;
    for (int base = 0; base < ns; base += blockDim.x) {
        int s = base + threadIdx.x;
        Seg g{};
        if (s < ns) g = segs[s];
        long long tp, tl, tm, tc;
        long long xp = block_exclusive_scan(s < ns ? g.P : 0, sh, &tp);
        long long xl = block_exclusive_scan(s < ns ? g.T + 1 : 0, sh, &tl);
        long long xm = block_exclusive_scan(s < ns ? (long long)g.rows * g.nch : 0, sh, &tm);
        long long xc = block_exclusive_scan(s < ns ? g.nch : 0, sh, &tc);
        if (s < ns) {
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
// sorted and de-duplicated; plus the bucket LUT and the chunk -> segment map.
__global__ void __launch_bounds__(256) k_pivots(Seg *segs, const int *nseg, const double *src,
                                                double *piv_pool, int *lut_pool, int *chunk_seg)
{
    __shared__ double sp[kPMaxPow2];
    __shared__ double cp[kPMax];
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
                    int lo = 2 * j * (i / j) + (i % j), hi = lo + j;
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
        if (threadIdx.x == 0) sk = (int)carry;
        __syncthreads();
        const int k = sk;
        for (int i = threadIdx.x; i < k; i += blockDim.x) piv_pool[g.piv_off + i] = cp[i];
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
        for (int t = threadIdx.x; t <= T; t += blockDim.x) {
            // lut[t] = #{j : bucket(piv_j) < t}
            int a = 0, b = k;
            while (a < b) {
                int mid = (a + b) >> 1;
                if (lut_bucket(cp[mid], lo, scale, T) < t) a = mid + 1; else b = mid;
            }
            lut_pool[g.lut_off + t] = (t == T) ? k : a;
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
// ---------------------------------------------------------------------------
template <bool kGate>
__global__ void __launch_bounds__(kPassThreads) k_count(const Seg *segs, const int *chunk_seg,
                                                        const DevStatus *cst, const double *src,
                                                        const double *piv_pool, const int *lut_pool,
                                                        unsigned *mat, DevStatus *st)
{
    __shared__ double spiv[kPMax];
    __shared__ int slut[kLutMax + 1];
    __shared__ unsigned shist[kRowsMax];
    __shared__ Seg sg;
    int cached = -1;
    long long bad = LLONG_MAX;
    unsigned pz = 0, nz = 0;
    const int nchunks = cst->nchunks;
    for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int s = chunk_seg[ch];
        __syncthreads();
        if (s != cached) {
            if (threadIdx.x == 0) sg = segs[s];
            __syncthreads();
            for (int i = threadIdx.x; i < sg.k; i += blockDim.x) spiv[i] = piv_pool[sg.piv_off + i];
            for (int i = threadIdx.x; i <= sg.T; i += blockDim.x) slut[i] = lut_pool[sg.lut_off + i];
            cached = s;
        }
        for (int c = threadIdx.x; c < sg.rows; c += blockDim.x) shist[c] = 0;
        __syncthreads();
        const int j = ch - sg.ch_off;
        const long long base = sg.start + (long long)j * kChunk;
        const int cnt = (int)min((long long)kChunk, sg.len - (long long)j * kChunk);
        const int k = sg.k, T = sg.T;
        const double lo = sg.lo, scale = sg.scale;
#pragma unroll 4
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            double v = __ldg(src + base + i);
            if (kGate) gate_one(v, base + i, bad, pz, nz);
            int c = classify(v, spiv, k, slut, lo, scale, T);
            atomicAdd(&shist[c], 1u);
        }
        __syncthreads();
        for (int c = threadIdx.x; c < sg.rows; c += blockDim.x)
            mat[sg.mat_off + (long long)c * sg.nch + j] = shist[c];
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

// ---------------------------------------------------------------------------
// scatter: classify again, group each tile by class in shared memory, write
// each class's run contiguously to its destination (coalesced runs)
// ---------------------------------------------------------------------------
struct ScatterSmem {
    double stage[kTile];
    long long cur[kRowsMax];
    double piv[kPMax];
    int lut[kLutMax + 1];
    unsigned hist[kRowsMax];
    unsigned off[kRowsMax + 1];
    unsigned short cls[kTile];
    long long sh[33];
    Seg sg;
};

__global__ void __launch_bounds__(kPassThreads) k_scatter(const Seg *segs, const int *chunk_seg,
                                                          const DevStatus *cst, const double *src,
                                                          double *dst, const double *piv_pool,
                                                          const int *lut_pool, const long long *moff)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScatterSmem &S = *reinterpret_cast<ScatterSmem *>(smem_raw);
    constexpr int E = kTile / kPassThreads;
    int cached = -1;
    const int nchunks = cst->nchunks;
    for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int s = chunk_seg[ch];
        __syncthreads();
        if (s != cached) {
            if (threadIdx.x == 0) S.sg = segs[s];
            __syncthreads();
            for (int i = threadIdx.x; i < S.sg.k; i += blockDim.x) S.piv[i] = piv_pool[S.sg.piv_off + i];
            for (int i = threadIdx.x; i <= S.sg.T; i += blockDim.x) S.lut[i] = lut_pool[S.sg.lut_off + i];
            cached = s;
        }
        const Seg &g = S.sg;
        const int j = ch - g.ch_off;
        const long long base = g.start + (long long)j * kChunk;
        const int cnt = (int)min((long long)kChunk, g.len - (long long)j * kChunk);
        const long long base_i = moff[g.mat_off];
        const int rows = g.rows, nch = g.nch, k = g.k, T = g.T;
        const double lo = g.lo, scale = g.scale;
        for (int c = threadIdx.x; c < rows; c += blockDim.x)
            S.cur[c] = g.start + (moff[g.mat_off + (long long)c * nch + j] - base_i);
        for (int t0 = 0; t0 < cnt; t0 += kTile) {
            const int tcnt = min(kTile, cnt - t0);
            for (int c = threadIdx.x; c < rows; c += blockDim.x) S.hist[c] = 0;
            __syncthreads();
            double v[E];
            int cl[E];
            unsigned r[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = e * kPassThreads + threadIdx.x;
                if (i < tcnt) v[e] = __ldg(src + base + t0 + i);
            }
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = e * kPassThreads + threadIdx.x;
                if (i < tcnt) {
                    cl[e] = classify(v[e], S.piv, k, S.lut, lo, scale, T);
                    r[e] = atomicAdd(&S.hist[cl[e]], 1u);
                }
            }
            __syncthreads();
            {   // exclusive scan of the tile histogram: 2 classes per thread
                const int c0 = 2 * threadIdx.x;
                unsigned h0 = c0 < rows ? S.hist[c0] : 0u;
                unsigned h1 = c0 + 1 < rows ? S.hist[c0 + 1] : 0u;
                long long ex = block_exclusive_scan((long long)h0 + h1, S.sh, nullptr);
                if (c0 < rows) S.off[c0] = (unsigned)ex;
                if (c0 + 1 < rows) S.off[c0 + 1] = (unsigned)ex + h0;
            }
            __syncthreads();
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = e * kPassThreads + threadIdx.x;
                if (i < tcnt) {
                    const unsigned p = S.off[cl[e]] + r[e];
                    S.stage[p] = v[e];
                    S.cls[p] = (unsigned short)cl[e];
                }
            }
            __syncthreads();
            for (int p = threadIdx.x; p < tcnt; p += blockDim.x) {
                const int c = S.cls[p];
                if (!(c & 1)) dst[S.cur[c] + (p - (long long)S.off[c])] = S.stage[p];
            }
            __syncthreads();
            for (int c = threadIdx.x; c < rows; c += blockDim.x) S.cur[c] += S.hist[c];
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// plan: turn class extents into next-pass segments and leaf work
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_plan(const Seg *segs, const int *nseg, const double *piv_pool,
                                              const long long *moff, Seg *next, int *nnext, Leaf *leaves,
                                              DevStatus *st, int dst_id, int seg_cap, int leaf_cap)
{
    __shared__ long long sh[33];
    const int ns = *nseg;
    for (int s = blockIdx.x; s < ns; s += gridDim.x) {
        const Seg g = segs[s];
        const long long base_i = moff[g.mat_off];
        const int ncls = 2 * g.k + 1;
        long long eq = 0, leafk = 0, leafn = 0, fillk = 0, copyk = 0;
        for (int c = threadIdx.x; c < ncls; c += blockDim.x) {
            const long long a = moff[g.mat_off + (long long)c * g.nch] - base_i;
            const long long b = (c + 1 < g.rows) ? moff[g.mat_off + (long long)(c + 1) * g.nch] - base_i : g.len;
            const long long size = b - a, abs = g.start + a;
            if (size <= 0) continue;
            if (c & 1) {
                eq += size;
                fillk += size;
                int i = atomicAdd(&st->nleaf, 1);
                if (i >= leaf_cap) { st->overflow = 3; continue; }
                Leaf L{};
                L.start = abs;
                L.len = size;
                L.value = piv_pool[g.piv_off + (c >> 1)];
                L.kind = kLeafFill;
                L.src = dst_id;
                leaves[i] = L;
            } else if (size == 1) {
                if (dst_id == 1) {
                    copyk += 1;
                    int i = atomicAdd(&st->nleaf, 1);
                    if (i >= leaf_cap) { st->overflow = 3; continue; }
                    Leaf L{};
                    L.start = abs;
                    L.len = 1;
                    L.kind = kLeafCopy;
                    L.src = 1;
                    leaves[i] = L;
                }
            } else if (size <= kLeafMax) {
                leafk += size;
                leafn += 1;
                int i = atomicAdd(&st->nleaf, 1);
                if (i >= leaf_cap) { st->overflow = 3; continue; }
                Leaf L{};
                L.start = abs;
                L.len = size;
                L.kind = kLeafSort;
                L.src = dst_id;
                leaves[i] = L;
            } else {
                int i = atomicAdd(nnext, 1);
                if (i >= seg_cap) { st->overflow = 4; continue; }
                Seg n2{};
                n2.start = abs;
                n2.len = size;
                next[i] = n2;
            }
        }
        long long t_eq, t_lk, t_ln, t_fk, t_ck;
        block_exclusive_scan(eq, sh, &t_eq);
        block_exclusive_scan(leafk, sh, &t_lk);
        block_exclusive_scan(leafn, sh, &t_ln);
        block_exclusive_scan(fillk, sh, &t_fk);
        block_exclusive_scan(copyk, sh, &t_ck);
        if (threadIdx.x == 0) {
            // algorithmic bytes: count reads 8B/key; scatter reads 8B/key and
            // writes 8B per non-equal key; leaf sort 16B/key; fill 8B/key; copy 16B/key
            add_bytes(st, kPhCount, 8ull * g.len);
            add_bytes(st, kPhScatter, 8ull * g.len + 8ull * (g.len - t_eq));
            add_bytes(st, kPhLeaf, 16ull * t_lk + 8ull * t_fk + 16ull * t_ck);
            atomicAdd(&st->keys_partitioned, (unsigned long long)g.len);
            atomicAdd(&st->keys_leaf, (unsigned long long)t_lk);
            atomicAdd(&st->leaves, (unsigned long long)t_ln);
        }
    }
}

// ---------------------------------------------------------------------------
// leaf: finish segments <= S on chip, write final values into the user buffer
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kLeafThreads) k_leaf(const Leaf *leaves, const DevStatus *cst,
                                                       double *keys, const double *tmp)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *s = reinterpret_cast<double *>(smem_raw);
    if (abort_requested(cst)) return;
    const int nleaf = cst->nleaf;
    for (int d = blockIdx.x; d < nleaf; d += gridDim.x) {
        const Leaf L = leaves[d];
        const double *src = L.src ? tmp : keys;
        if (L.kind == kLeafFill) {
            for (long long i = threadIdx.x; i < L.len; i += blockDim.x) keys[L.start + i] = L.value;
            continue;
        }
        if (L.kind == kLeafCopy) {
            for (long long i = threadIdx.x; i < L.len; i += blockDim.x) keys[L.start + i] = src[L.start + i];
            continue;
        }
        const int m = (int)L.len, N = next_pow2(m);
        __syncthreads();
        for (int i = threadIdx.x; i < N; i += blockDim.x) s[i] = i < m ? src[L.start + i] : CUDART_INF;
        __syncthreads();
        for (int kk = 2; kk <= N; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
                    int lo = 2 * j * (i / j) + (i % j), hi = lo + j;
                    bool asc = (lo & kk) == 0;
                    double a = s[lo], b = s[hi];
                    if ((a > b) == asc) { s[lo] = b; s[hi] = a; }
                }
                __syncthreads();
            }
        }
        for (int i = threadIdx.x; i < m; i += blockDim.x) keys[L.start + i] = s[i];
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
    long long piv = 4 * n / kLeafMax + L.seg_cap + 1;           // sum of P_i
    L.piv_cap = (int)piv;
    L.lut_cap = (int)(4 * piv + L.seg_cap + 1);                  // sum of T_i + 1
    L.ch_cap = (int)(n / kChunk + L.seg_cap + 1);
    L.mat_cap = (2 * piv + L.seg_cap) + (long long)(2 * kPMax + 1) * (2 * (n / kChunk) + 2);
    L.leaf_cap = (int)(2 * piv + L.seg_cap + nseg0 + 1);
    L.bsum_cap = cdiv(L.mat_cap, kScanBlock) + 1;
    size_t off = 0;
    L.o_status = off; off = align_up(off + sizeof(DevStatus));
    L.o_seg[0] = off; off = align_up(off + sizeof(Seg) * L.seg_cap);
    L.o_seg[1] = off; off = align_up(off + sizeof(Seg) * L.seg_cap);
    L.o_chunk = off; off = align_up(off + sizeof(int) * L.ch_cap);
    L.o_piv = off; off = align_up(off + sizeof(double) * L.piv_cap);
    L.o_lut = off; off = align_up(off + sizeof(int) * L.lut_cap);
    L.o_mat = off; off = align_up(off + sizeof(unsigned) * L.mat_cap);
    L.o_moff = off; off = align_up(off + sizeof(long long) * L.mat_cap);
    L.o_bsum = off; off = align_up(off + sizeof(long long) * L.bsum_cap);
    L.o_leaf = off; off = align_up(off + sizeof(Leaf) * L.leaf_cap);
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

#define KS_CK(x)                                                            \
    do {                                                                    \
        cudaError_t e_ = (x);                                               \
        if (e_ != cudaSuccess) {                                            \
            fprintf(stderr, "ksort: %s failed: %s\n", #x, cudaGetErrorString(e_)); \
            return KS_CUDA_ERROR;                                           \
        }                                                                   \
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
    // after a stream sync
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

int fast_sort(double *keys, long long n, const long long *d_off, long long nseg0, void *ws,
              size_t ws_bytes, cudaStream_t stream, bool profile, FastResult *res)
{
    FastLayout L = fast_layout(n, nseg0);
    if (ws_bytes < L.total) return KS_WORKSPACE_SMALL;
    char *w = static_cast<char *>(ws);
    DevStatus *st = reinterpret_cast<DevStatus *>(w + L.o_status);
    Seg *segs[2] = {reinterpret_cast<Seg *>(w + L.o_seg[0]), reinterpret_cast<Seg *>(w + L.o_seg[1])};
    int *chunk_seg = reinterpret_cast<int *>(w + L.o_chunk);
    double *piv = reinterpret_cast<double *>(w + L.o_piv);
    int *lut = reinterpret_cast<int *>(w + L.o_lut);
    unsigned *mat = reinterpret_cast<unsigned *>(w + L.o_mat);
    long long *moff = reinterpret_cast<long long *>(w + L.o_moff);
    long long *bsum = reinterpret_cast<long long *>(w + L.o_bsum);
    Leaf *leaves = reinterpret_cast<Leaf *>(w + L.o_leaf);
    double *tmp = reinterpret_cast<double *>(w + L.o_tmp);

    KS_CK(cudaFuncSetAttribute(k_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ScatterSmem)));
    KS_CK(cudaFuncSetAttribute(k_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kLeafMax * sizeof(double))));
    const int sms = sm_count();
    int occ_count = 1, occ_scatter = 1, occ_leaf = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_count, k_count<false>, kPassThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_scatter, k_scatter, kPassThreads, sizeof(ScatterSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_leaf, k_leaf, kLeafThreads, kLeafMax * sizeof(double));
    const int g_count = sms * (occ_count > 0 ? occ_count : 1);
    const int g_scatter = sms * (occ_scatter > 0 ? occ_scatter : 1);
    const int g_leaf = sms * (occ_leaf > 0 ? occ_leaf : 1);
    const int g_scan = sms * 2;
    const int g_seg = sms * 4;
    Launcher K(stream, profile);

    DevStatus h{};
    KS_CK(cudaMemsetAsync(st, 0, sizeof(DevStatus), stream));
    KS_CK(cudaMemsetAsync(&st->bad_index, 0xff, sizeof(unsigned long long), stream));

    if (d_off == nullptr) {
        K.run(kPhGate, [&] { k_init_single<<<1, 32, 0, stream>>>(n, segs[0], leaves, st); });
        if (n <= kLeafMax)
            K.run(kPhGate, [&] { k_gate_segments<<<sms, 256, 0, stream>>>(keys, nullptr, 0, n, st); });
    } else {
        K.run(kPhGate, [&] {
            k_init_segmented<<<sms, 256, 0, stream>>>(d_off, nseg0, segs[0], leaves, st, L.seg_cap, L.leaf_cap);
        });
        K.run(kPhGate, [&] { k_gate_segments<<<sms * 4, 256, 0, stream>>>(keys, d_off, nseg0, 0, st); });
    }
    KS_CK(cudaGetLastError());
    KS_CK(cudaMemcpyAsync(&h, st, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream));
    KS_CK(cudaStreamSynchronize(stream));
    if (h.overflow) return KS_CUDA_ERROR;

    int level = 0;
    int cur = 0;
    bool leaf_done_once = false;
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
                k_count<true><<<g_count, kPassThreads, 0, stream>>>(segs[cur], chunk_seg, st, src, piv, lut, mat, st);
            });
        else
            K.run(kPhCount, [&] {
                k_count<false><<<g_count, kPassThreads, 0, stream>>>(segs[cur], chunk_seg, st, src, piv, lut, mat, st);
            });
        K.run(kPhScan, [&] { k_scan_reduce<<<g_scan, kScanThreads, 0, stream>>>(mat, st, bsum); });
        K.run(kPhScan, [&] { k_scan_bsums<<<1, 1024, 0, stream>>>(bsum, st); });
        K.run(kPhScan, [&] { k_scan_apply<<<g_scan, kScanThreads, 0, stream>>>(mat, st, bsum, moff); });
        K.run(kPhScatter, [&] {
            k_scatter<<<g_scatter, kPassThreads, sizeof(ScatterSmem), stream>>>(segs[cur], chunk_seg, st, src, dst,
                                                                               piv, lut, moff);
        });
        KS_CK(cudaMemsetAsync(nseg_next, 0, sizeof(int), stream));
        K.run(kPhPlan, [&] {
            k_plan<<<g_seg, 256, 0, stream>>>(segs[cur], nseg_cur, piv, moff, segs[cur ^ 1], nseg_next, leaves, st,
                                              dst_id, L.seg_cap, L.leaf_cap);
        });
        K.run(kPhLeaf, [&] {
            k_leaf<<<g_leaf, kLeafThreads, kLeafMax * sizeof(double), stream>>>(leaves, st, keys, tmp);
        });
        leaf_done_once = true;
        KS_CK(cudaMemsetAsync(&st->nleaf, 0, sizeof(int), stream));
        KS_CK(cudaGetLastError());
        KS_CK(cudaMemcpyAsync(&h, st, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream));
        KS_CK(cudaStreamSynchronize(stream));
        ++level;
        cur ^= 1;
        if (h.overflow) return KS_CUDA_ERROR;
        if (h.bad_index != kNoIndex || (h.pos_zero && h.neg_zero)) break;
    }
    if (!leaf_done_once) {
        K.run(kPhLeaf, [&] {
            k_leaf<<<g_leaf, kLeafThreads, kLeafMax * sizeof(double), stream>>>(leaves, st, keys, tmp);
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
