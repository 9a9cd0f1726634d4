// Microbenchmark: one-pass bucketed partition of 10M f64 keys into 2048
// over-provisioned buckets (per-tile shared histogram -> one global atomic per
// non-empty bucket -> scattered 8-byte stores), vs a count-only pass.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/mb_onepass.cu -o scripts/mb_onepass
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NB = 2048;
constexpr int TH = 512;

__device__ __forceinline__ unsigned long long mix(unsigned long long z)
{
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__global__ void k_gen(double *k, long long n)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        k[i] = (double)(mix(i * 0x9E3779B97F4A7C15ull + 1) >> 11) * 0x1.0p-53;
}

template <int E, int PF>
__global__ void __launch_bounds__(TH) k_one(const double *keys, long long n, double *bkt, int cap, unsigned *gcnt,
                                             int *ovf)
{
    __shared__ unsigned hist[NB];
    __shared__ unsigned base[NB];
    for (int c = threadIdx.x; c < NB; c += TH) hist[c] = 0;
    __syncthreads();
    const long long tile = (long long)TH * E;
    for (long long t0 = blockIdx.x * tile; t0 < n; t0 += (long long)gridDim.x * tile) {
        double v[E];
        unsigned cr[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const long long i = t0 + e * TH + threadIdx.x;
            v[e] = i < n ? __ldcs(keys + i) : -1.0;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (v[e] >= 0.0) {
                const int c = min((int)(v[e] * NB), NB - 1);
                cr[e] = ((unsigned)c << 20) | atomicAdd(&hist[c], 1u);
            }
        }
        __syncthreads();
        for (int c = threadIdx.x; c < NB; c += TH) {
            const unsigned h = hist[c];
            if (h) {
                const unsigned b = atomicAdd(&gcnt[c], h);
                base[c] = b;
                if (PF) {
                    const char *p0 = reinterpret_cast<const char *>(bkt + (long long)c * cap + b);
                    const char *p1 = reinterpret_cast<const char *>(bkt + (long long)c * cap + b + h);
                    for (unsigned long long a = reinterpret_cast<unsigned long long>(p0) & ~127ull;
                         a < reinterpret_cast<unsigned long long>(p1); a += 128)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(a) : "memory");
                }
                hist[c] = 0;
            }
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (v[e] >= 0.0) {
                const int c = cr[e] >> 20;
                const unsigned pos = base[c] + (cr[e] & 0xfffffu);
                if (pos < (unsigned)cap) bkt[(long long)c * cap + pos] = v[e]; else *ovf = 1;
            }
        }
        __syncthreads();
    }
}

template <int E>
__global__ void __launch_bounds__(TH) k_countonly(const double *keys, long long n, unsigned *mat)
{
    __shared__ unsigned hist[NB];
    for (int c = threadIdx.x; c < NB; c += TH) hist[c] = 0;
    __syncthreads();
    const long long chunk = (n + gridDim.x - 1) / gridDim.x;
    const long long a = blockIdx.x * chunk, b = min(n, a + chunk);
    for (long long t0 = a; t0 < b; t0 += (long long)TH * E) {
        double v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const long long i = t0 + e * TH + threadIdx.x;
            v[e] = i < b ? __ldcs(keys + i) : -1.0;
        }
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (v[e] >= 0.0) atomicAdd(&hist[min((int)(v[e] * NB), NB - 1)], 1u);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < NB; c += TH) mat[(long long)c * gridDim.x + blockIdx.x] = hist[c];
}

int main()
{
    const long long n = 10000000;
    const int cap = 16 * (int)(n / NB);
    double *keys, *bkt;
    unsigned *gcnt, *mat;
    int *ovf;
    char *flush;
    cudaMalloc(&keys, n * 8);
    cudaMalloc(&bkt, (size_t)NB * cap * 8);
    cudaMalloc(&gcnt, NB * 4);
    cudaMalloc(&mat, NB * 4096 * 4);
    cudaMalloc(&ovf, 4);
    cudaMalloc(&flush, 256 << 20);
    k_gen<<<1184, 256>>>(keys, n);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char *name, auto fn) {
        float best = 1e9, sum = 0;
        const int reps = 20;
        for (int r = 0; r < reps + 3; ++r) {
            cudaMemset(gcnt, 0, NB * 4);
            cudaMemset(flush, r, 256 << 20);
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) {
                best = ms < best ? ms : best;
                sum += ms;
            }
        }
        int h = 0;
        cudaMemcpy(&h, ovf, 4, cudaMemcpyDeviceToHost);
        printf("%-28s best %7.1f us  mean %7.1f us  ovf %d  %s\n", name, best * 1e3, sum / reps * 1e3, h,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int occ = 2; occ <= 3; ++occ) {
        char nm[64];
        snprintf(nm, 64, "one E=8 pf=0 occ=%d", occ);
        run(nm, [&] { k_one<8, 0><<<sms * occ, TH>>>(keys, n, bkt, cap, gcnt, ovf); });
        snprintf(nm, 64, "one E=8 pf=1 occ=%d", occ);
        run(nm, [&] { k_one<8, 1><<<sms * occ, TH>>>(keys, n, bkt, cap, gcnt, ovf); });
        snprintf(nm, 64, "one E=16 pf=0 occ=%d", occ);
        run(nm, [&] { k_one<16, 0><<<sms * occ, TH>>>(keys, n, bkt, cap, gcnt, ovf); });
        snprintf(nm, 64, "one E=16 pf=1 occ=%d", occ);
        run(nm, [&] { k_one<16, 1><<<sms * occ, TH>>>(keys, n, bkt, cap, gcnt, ovf); });
    }
    run("countonly E=8 3/SM", [&] { k_countonly<8><<<sms * 3, TH>>>(keys, n, mat); });
    return 0;
}
