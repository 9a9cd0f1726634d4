// ks_heap.cu -- the reference's heap sort (sort_core.py:223-286) run exactly
// on the device by one sequential lane, with its op counts.
//
// Heap sort has no data-parallel form that preserves its permutation; this
// lane exists so heap_sort(a, counts) and inputs holding both signed zeros get
// the reference's exact bytes and tallies.  Everything else routes heap_sort
// to the K-sort engine (identical outputs).
#include <cstdio>

#include "ks_host.h"
#include "ks_internal.cuh"

namespace ks {

struct HeapStatus {
    unsigned long long bad;
    unsigned long long comparisons, moves;
};

__global__ void k_heap_gate(const double *a, long long n, HeapStatus *hs)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        if (!isfinite(a[i])) atomicMin(&hs->bad, (unsigned long long)i);
}

// sort_core.py:240-259 (_sift_down_counted; identical moves to _sift_down)
__device__ __forceinline__ void sift_down(double *a, long long root, long long end,
                                          unsigned long long &cmp, unsigned long long &mv)
{
    double val = a[root];
    mv += 1;
    for (;;) {
        long long child = 2 * root + 1;
        if (child > end) break;
        if (child + 1 <= end) {
            cmp += 1;
            if (a[child + 1] > a[child]) child += 1;
        }
        cmp += 1;
        if (a[child] > val) {
            a[root] = a[child];
            mv += 1;
            root = child;
        } else {
            break;
        }
    }
    a[root] = val;
    mv += 1;
}

__global__ void k_heap_sort(double *a, long long n, HeapStatus *hs)
{
    if (threadIdx.x || blockIdx.x) return;
    if (hs->bad != ~0ull || n < 2) return;   // sort_core.py:268-271
    unsigned long long cmp = 0, mv = 0;
    for (long long root = n / 2 - 1; root >= 0; --root) sift_down(a, root, n - 1, cmp, mv);
    for (long long end = n - 1; end > 0; --end) {
        double t = a[0];
        a[0] = a[end];
        a[end] = t;
        mv += 2;
        if (end > 1) sift_down(a, 0, end - 1, cmp, mv);
    }
    hs->comparisons = cmp;
    hs->moves = mv;
}

size_t heap_workspace_bytes() { return 256; }

int heap_sort_exact(double *keys, long long n, void *ws, size_t ws_bytes, cudaStream_t stream,
                    long long *bad_index, unsigned long long *comparisons, unsigned long long *moves)
{
    if (ws_bytes < sizeof(HeapStatus)) return KS_WORKSPACE_SMALL;
    HeapStatus *hs = static_cast<HeapStatus *>(ws);
    if (cudaMemsetAsync(hs, 0, sizeof(HeapStatus), stream) != cudaSuccess) return KS_CUDA_ERROR;
    if (cudaMemsetAsync(&hs->bad, 0xff, 8, stream) != cudaSuccess) return KS_CUDA_ERROR;
    if (n > 0) k_heap_gate<<<128, 256, 0, stream>>>(keys, n, hs);
    k_heap_sort<<<1, 32, 0, stream>>>(keys, n, hs);
    HeapStatus h{};
    if (cudaMemcpyAsync(&h, hs, sizeof(h), cudaMemcpyDeviceToHost, stream) != cudaSuccess) return KS_CUDA_ERROR;
    cudaError_t e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
        fprintf(stderr, "ksort(heap): %s\n", cudaGetErrorString(e));
        return KS_CUDA_ERROR;
    }
    *bad_index = h.bad == ~0ull ? -1 : (long long)h.bad;
    *comparisons = h.comparisons;
    *moves = h.moves;
    return KS_OK;
}

}  // namespace ks
