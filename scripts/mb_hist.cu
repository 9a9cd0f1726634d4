// Microbenchmark: cost of building a shared-memory class histogram / in-warp
// rank for random 9-bit classes, three ways: ATOMS per key, ballot peer
// detection (9 ballots), MATCH.ANY.  Prints ns and cycles per key.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int C = 511;

__device__ __forceinline__ unsigned hash32(unsigned x)
{
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_hist(int iters, unsigned *out)
{
    __shared__ unsigned h[8][C + 1];
    for (int i = threadIdx.x; i < 8 * (C + 1); i += 256) (&h[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned seed = blockIdx.x * 256 + threadIdx.x;
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned c = hash32(seed + it * 7919u) % C;
        if (MODE == 0) {
            acc += atomicAdd(&h[0][c], 1u);
        } else if (MODE == 1) {
            unsigned peers = 0xffffffffu;
#pragma unroll
            for (int b = 0; b < 9; ++b) {
                unsigned bit = (c >> b) & 1u;
                unsigned m = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? m : ~m;
            }
            if (lane == __ffs(peers) - 1) h[wid][c] += __popc(peers);
            acc += peers;
        } else if (MODE == 2) {
            unsigned peers = __match_any_sync(0xffffffffu, c);
            if (lane == __ffs(peers) - 1) h[wid][c] += __popc(peers);
            acc += peers;
        } else {
            acc += c;   // baseline: hash only
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = acc + h[0][0] + h[wid][1];
}

int main()
{
    unsigned *out;
    cudaMalloc(&out, 1 << 20);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, iters = 4096;
    const char *names[4] = {"atoms", "ballot9", "match_any", "hash_only"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            if (mode == 0) k_hist<0><<<blocks, 256>>>(iters, out);
            if (mode == 1) k_hist<1><<<blocks, 256>>>(iters, out);
            if (mode == 2) k_hist<2><<<blocks, 256>>>(iters, out);
            if (mode == 3) k_hist<3><<<blocks, 256>>>(iters, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double keys = (double)blocks * 256 * iters;
            if (rep)
                printf("%-10s %.3f ms  %.4f ns/key  %.2f SM-cycles/key (at %d MHz)\n", names[mode], ms,
                       ms * 1e6 / keys, ms * 1e-3 * clk * 1e3 * sms / keys, clk / 1000);
        }
    }
    return 0;
}
