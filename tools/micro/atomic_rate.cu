// Microbenchmark: same-address atomicAdd throughput on one u64 counter, one atomic per warp
// iteration (the warp-level output reservation pattern), with `work` dependent ALU ops between.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(unsigned long long *ctr, unsigned long long *sink, int iters, int work, int spread)
{
    unsigned long long acc = threadIdx.x;
    const int lane = threadIdx.x & 31;
    unsigned long long *c = ctr + (spread > 1 ? ((blockIdx.x * 8 + (threadIdx.x >> 5)) % spread) * 32 : 0);
    for (int i = 0; i < iters; ++i) {
        for (int w = 0; w < work; ++w)
            acc = acc * 6364136223846793005ull + 1442695040888963407ull;
        unsigned long long b = 0;
        if (lane == 0)
            b = atomicAdd(c, 69ull);
        b = __shfl_sync(0xffffffffu, b, 0);
        acc ^= b;
    }
    if (acc == 42)
        *sink = acc;
}

int main()
{
    unsigned long long *ctr, *sink;
    cudaMalloc(&ctr, 1 << 20);
    cudaMalloc(&sink, 8);
    cudaMemset(ctr, 0, 1 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int spread : {1, 4, 16}) {
        for (int work : {0, 32, 128}) {
            const int blocks = sms * 4, iters = 2000;
            k<<<blocks, 256>>>(ctr, sink, 10, work, spread);
            cudaEventRecord(a);
            k<<<blocks, 256>>>(ctr, sink, iters, work, spread);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double n = (double)blocks * 8 * iters;
            printf("spread %2d work %3d: %.3f ms, %.3e warp-atomics/s\n", spread, work, ms, n / (ms * 1e-3));
        }
    }
    return 0;
}
