// ks_misc.cu -- device twins of the reference's workload generator
// (workload.py:43-78) and of sort_core.is_sorted (sort_core.py:62-67).
#include "ks_host.h"
#include "ks_internal.cuh"

namespace ks {

__device__ __forceinline__ unsigned long long mix64(unsigned long long x)
{
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// output t of the counter-based stream: mix64(seed + (t + 1) * gamma)
__global__ void k_generate(double *out, long long n, unsigned long long seed, int kind)
{
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        unsigned long long u = mix64(seed + (unsigned long long)(t + 1) * 0x9E3779B97F4A7C15ull);
        out[t] = kind == 1 ? (double)(u >> 56) * (1.0 / 256.0) : (double)(u >> 11) * 0x1p-53;
    }
}

__global__ void k_is_sorted(const double *a, long long n, int *flag)
{
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x + 1; t < n;
         t += (long long)gridDim.x * blockDim.x)
        if (a[t - 1] > a[t]) *flag = 0;
}

__global__ void k_gate_range(const double *a, long long n, unsigned long long *bad)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        if (!isfinite(a[i])) atomicMin(bad, (unsigned long long)i);
}

// first non-finite index of a[0..n) or -1 (sort_core.py:50-59); ws >= 8 bytes
int gate_range(const double *a, long long n, void *ws, cudaStream_t stream, long long *bad_index)
{
    unsigned long long *bad = static_cast<unsigned long long *>(ws);
    unsigned long long h = ~0ull;
    if (cudaMemsetAsync(bad, 0xff, 8, stream) != cudaSuccess) return KS_CUDA_ERROR;
    if (n > 0) k_gate_range<<<256, 256, 0, stream>>>(a, n, bad);
    if (cudaMemcpyAsync(&h, bad, 8, cudaMemcpyDeviceToHost, stream) != cudaSuccess) return KS_CUDA_ERROR;
    if (cudaStreamSynchronize(stream) != cudaSuccess) return KS_CUDA_ERROR;
    *bad_index = h == ~0ull ? -1 : (long long)h;
    return KS_OK;
}

int generate_f64(double *out, long long n, unsigned long long seed, int kind, cudaStream_t stream)
{
    if (n <= 0) return KS_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k_generate<<<sms * 8, 256, 0, stream>>>(out, n, seed, kind);
    return cudaGetLastError() == cudaSuccess ? KS_OK : KS_CUDA_ERROR;
}

int is_sorted_f64(const double *keys, long long n, void *ws, cudaStream_t stream, int *result)
{
    int *flag = static_cast<int *>(ws);
    int one = 1;
    if (cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return KS_CUDA_ERROR;
    if (n > 1) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        k_is_sorted<<<sms * 8, 256, 0, stream>>>(keys, n, flag);
    }
    if (cudaMemcpyAsync(result, flag, sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return KS_CUDA_ERROR;
    return cudaStreamSynchronize(stream) == cudaSuccess ? KS_OK : KS_CUDA_ERROR;
}

}  // namespace ks
