// ks_sortnet.cuh -- on-chip sorting primitives for the leaf sorter.
//
//  * warp_bitonic_sort<E>: 32*E keys held "blocked" in a warp's registers
//    (lane l holds elements l*E .. l*E+E-1) are sorted ascending by a bitonic
//    network: compare-exchange stages with partner distance j < E stay inside
//    a lane's registers, larger distances use warp shuffles (the warp-shuffle
//    merge of the north star).  FP64 min/max keep K-sort's `<=` order.
//  * merge-path block merge of sorted runs in shared memory.
//  * warp ranking by ballot (peer detection) for multisplit without atomics.
#pragma once

#include "ks_internal.cuh"

namespace ks {

// padded shared-memory index: one spare double every 16 keeps blocked
// (lane*16 + r) and strided (e*32 + lane) accesses at the 2-wavefront minimum
__device__ __forceinline__ int sidx(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int sidx_size(int n) { return n + (n >> 4) + 1; }

// compare-exchange a pair so that (a, b) is ascending iff asc
__device__ __forceinline__ void cas(double &a, double &b, bool asc)
{
    const bool sw = (b < a) == asc;   // one DSETP + four FSEL
    const double lo = sw ? b : a, hi = sw ? a : b;
    a = lo;
    b = hi;
}

// Stages whose partner distance is below E are unrolled (register indices
// must be compile-time); the five lane-level merge levels run as rolled
// loops so the code stays small -- the unrolled form of E=16 alone is ~3K
// instructions and warps sorting different sizes thrashed the I-cache
// (84% "no instruction" stalls in ncu).
template <int E>
__device__ __forceinline__ void warp_bitonic_sort(double (&x)[E])
{
    const int lane = threadIdx.x & 31;
    // k = 2 .. E: inside each lane (element i = lane*E + r)
#pragma unroll
    for (int k = 2; k <= E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int r = 0; r < E; ++r) {
                if ((r & j) == 0) {
                    const bool asc = (k < E) ? ((r & k) == 0) : ((lane & 1) == 0);
                    cas(x[r], x[r ^ j], asc);
                }
            }
        }
    }
    // k = 2E .. 32E: lane-distance stages by shuffle, then in-lane half-cleaners.
    // Small E (the common unit sizes) unroll completely -- rolled loops cost a
    // divergence check and loop bookkeeping per stage; large E stay rolled to
    // bound code size (I-cache).
#pragma unroll (E <= 4 ? 5 : 1)
    for (int kk = 2; kk <= 32; kk <<= 1) {          // k / E
        const bool asc = (lane & kk) == 0 || kk == 32;
#pragma unroll (E <= 4 ? 5 : 1)
        for (int lj = kk >> 1; lj > 0; lj >>= 1) {  // j / E
            const bool keep_min = ((lane & lj) == 0) == asc;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const double y = __shfl_xor_sync(0xffffffffu, x[r], lj);
                x[r] = ((y < x[r]) == keep_min) ? y : x[r];
            }
        }
#pragma unroll
        for (int j = E >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int r = 0; r < E; ++r) {
                if ((r & j) == 0) cas(x[r], x[r ^ j], asc);
            }
        }
    }
}

// Sort m <= 32*E keys of src[0..m) into dst[0..m) with one warp, staging
// through the warp's padded shared slice `sm` (sidx_size(32*E) doubles).
template <int E>
__device__ __forceinline__ void warp_sort_segment(const double *__restrict__ src, double *__restrict__ dst,
                                                  int m, double *sm)
{
    const int lane = threadIdx.x & 31;
    constexpr int N = 32 * E;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = e * 32 + lane;
        sm[sidx(i)] = i < m ? src[i] : CUDART_INF;
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
        if (i < m) dst[i] = sm[sidx(i)];
    }
    __syncwarp();
    (void)N;
}

// Merge path (first a in [lo,hi] with !(B[diag-1-a] < A[a]) false...): number of
// elements taken from A among the first `diag` outputs of merge(A, B), A first on ties.
__device__ __forceinline__ int merge_path(const double *s, int a0, int b0, int size, int diag)
{
    int lo = diag - size > 0 ? diag - size : 0;
    int hi = diag < size ? diag : size;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (!(s[sidx(b0 + diag - 1 - mid)] < s[sidx(a0 + mid)])) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Serially merge IPT outputs starting at (a, b) of runs A=[a0,a0+size), B=[b0,b0+size).
template <int IPT>
__device__ __forceinline__ void merge_serial(const double *s, int a0, int b0, int size, int a, int b,
                                             double (&out)[IPT])
{
    double va = a < size ? s[sidx(a0 + a)] : CUDART_INF;
    double vb = b < size ? s[sidx(b0 + b)] : CUDART_INF;
#pragma unroll
    for (int e = 0; e < IPT; ++e) {
        const bool takeA = !(vb < va);
        out[e] = takeA ? va : vb;
        if (takeA) ++a; else ++b;
        const bool ok = takeA ? (a < size) : (b < size);
        const int idx = takeA ? a0 + a : b0 + b;
        const double nx = ok ? s[sidx(idx)] : CUDART_INF;
        if (takeA) va = nx; else vb = nx;
    }
}

// Ballot peer detection: lanes of the warp holding the same NB-bit class.
template <int NB>
__device__ __forceinline__ unsigned warp_peers(unsigned c)
{
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const unsigned bit = (c >> b) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? m : ~m;
    }
    return peers;
}

__device__ __forceinline__ unsigned lanemask_lt()
{
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace ks
