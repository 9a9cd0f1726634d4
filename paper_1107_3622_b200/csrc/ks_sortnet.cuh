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

// Batcher odd-even merge sort of 16 keys in one thread's registers: 63
// compare-exchanges, all ascending (comparator list generated from the
// standard recursive construction; written out so every index is a
// compile-time register).
template <int N>
__device__ __forceinline__ void thread_sort(double (&x)[N]);

template <>
__device__ __forceinline__ void thread_sort<16>(double (&x)[16])
{
    cas(x[0], x[1], true);
    cas(x[2], x[3], true);
    cas(x[4], x[5], true);
    cas(x[6], x[7], true);
    cas(x[8], x[9], true);
    cas(x[10], x[11], true);
    cas(x[12], x[13], true);
    cas(x[14], x[15], true);
    cas(x[0], x[2], true);
    cas(x[1], x[3], true);
    cas(x[4], x[6], true);
    cas(x[5], x[7], true);
    cas(x[8], x[10], true);
    cas(x[9], x[11], true);
    cas(x[12], x[14], true);
    cas(x[13], x[15], true);
    cas(x[1], x[2], true);
    cas(x[5], x[6], true);
    cas(x[9], x[10], true);
    cas(x[13], x[14], true);
    cas(x[0], x[4], true);
    cas(x[1], x[5], true);
    cas(x[2], x[6], true);
    cas(x[3], x[7], true);
    cas(x[8], x[12], true);
    cas(x[9], x[13], true);
    cas(x[10], x[14], true);
    cas(x[11], x[15], true);
    cas(x[2], x[4], true);
    cas(x[3], x[5], true);
    cas(x[10], x[12], true);
    cas(x[11], x[13], true);
    cas(x[1], x[2], true);
    cas(x[3], x[4], true);
    cas(x[5], x[6], true);
    cas(x[9], x[10], true);
    cas(x[11], x[12], true);
    cas(x[13], x[14], true);
    cas(x[0], x[8], true);
    cas(x[1], x[9], true);
    cas(x[2], x[10], true);
    cas(x[3], x[11], true);
    cas(x[4], x[12], true);
    cas(x[5], x[13], true);
    cas(x[6], x[14], true);
    cas(x[7], x[15], true);
    cas(x[4], x[8], true);
    cas(x[5], x[9], true);
    cas(x[6], x[10], true);
    cas(x[7], x[11], true);
    cas(x[2], x[4], true);
    cas(x[3], x[5], true);
    cas(x[6], x[8], true);
    cas(x[7], x[9], true);
    cas(x[10], x[12], true);
    cas(x[11], x[13], true);
    cas(x[1], x[2], true);
    cas(x[3], x[4], true);
    cas(x[5], x[6], true);
    cas(x[7], x[8], true);
    cas(x[9], x[10], true);
    cas(x[11], x[12], true);
    cas(x[13], x[14], true);
}

// Merge path over runs A = s[a0, a0+aLen), B = s[b0, b0+bLen) (sidx layout):
// number of A elements among the first d outputs, A first on ties.
__device__ __forceinline__ int merge_path2(const double *s, int a0, int aLen, int b0, int bLen, int d)
{
    int lo = d - bLen > 0 ? d - bLen : 0;
    int hi = d < aLen ? d : aLen;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (!(s[sidx(b0 + d - 1 - mid)] < s[sidx(a0 + mid)])) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Warp merge sort of s[0..m) (sidx layout, m <= 32*IPT) in place: each lane
// sorts IPT consecutive keys in registers (Batcher network), then merge-path
// rounds double the sorted run length (runs of IPT, 2*IPT, ... < m).
template <int IPT>
__device__ __forceinline__ void warp_merge_sort(double *s, int m)
{
    const int lane = threadIdx.x & 31;
    const int o = lane * IPT;
    double x[IPT];
#pragma unroll
    for (int r = 0; r < IPT; ++r) x[r] = (o + r < m) ? s[sidx(o + r)] : CUDART_INF;
    thread_sort<IPT>(x);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < IPT; ++r)
        if (o + r < m) s[sidx(o + r)] = x[r];
    __syncwarp();
    for (int R = IPT; R < m; R <<= 1) {
        bool write = false;
        if (o < m) {
            const int g0 = o & ~(2 * R - 1);
            const int aLen = min(R, m - g0);
            const int b0 = g0 + R;
            const int bLen = min(R, m - b0);
            if (bLen > 0) {
                const int d = o - g0;
                int a = merge_path2(s, g0, aLen, b0, bLen, d);
                int b = d - a;
                double va = a < aLen ? s[sidx(g0 + a)] : CUDART_INF;
                double vb = b < bLen ? s[sidx(b0 + b)] : CUDART_INF;
#pragma unroll
                for (int r = 0; r < IPT; ++r) {
                    const bool takeA = !(vb < va);
                    x[r] = takeA ? va : vb;
                    if (takeA) {
                        ++a;
                        va = a < aLen ? s[sidx(g0 + a)] : CUDART_INF;
                    } else {
                        ++b;
                        vb = b < bLen ? s[sidx(b0 + b)] : CUDART_INF;
                    }
                }
                write = true;
            }
        }
        __syncwarp();
        if (write) {
#pragma unroll
            for (int r = 0; r < IPT; ++r)
                if (o + r < m) s[sidx(o + r)] = x[r];
        }
        __syncwarp();
    }
}

}  // namespace ks
