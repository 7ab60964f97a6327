// Micro-benchmark: where the K2 tail goes -- grid_reduce_dd<K> (common.cuh)
// on 296 CTAs x 288 threads (the row-warp K2 grid), %globaltimer stamps of
// the LAST CTA: entry -> after its block tree -> after the ticket -> after
// the fold of the 296 partials.  Also the same with the ticket fences removed
// (timing only) to price MEMBAR.SC.GPU.
#include <cstdio>
#include "../../paper_2211_15605_b200/csrc/common.cuh"

namespace mfx { void set_error(const char *, ...) {} }
using namespace mfx;

__device__ __forceinline__ unsigned long long gt()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int K>
__global__ void k(dd *part, unsigned *ticket, unsigned long long *st, double *out)
{
    // skew the CTAs a little, like the end of a streaming pass
    unsigned long long t0 = gt();
    while (gt() - t0 < (blockIdx.x * 7919u) % 3000u) {}
    dd v[K];
    for (int q = 0; q < K; q++) v[q] = dd{1.0 + threadIdx.x * 1e-3 + q + blockIdx.x, 1e-20};
    __syncthreads();
    const unsigned long long a = gt();
    block_reduce_lazy<K>(v);
    const unsigned long long b = gt();
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        for (int q = 0; q < K; q++) part[(size_t)blockIdx.x * K + q] = v[q];
        __threadfence();
        unsigned t = atomicAdd(ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    const unsigned long long c = gt();
    if (!s_last) return;
    __threadfence();
    const unsigned long long c2 = gt();
    dd f[K];
    block_fold_partials<K>(part, gridDim.x, K, f);
    const unsigned long long d = gt();
    if (threadIdx.x == 0) {
        st[0] = a; st[1] = b; st[2] = c; st[3] = c2; st[4] = d;
        out[0] = f[0].hi;
        *ticket = 0;
    }
}

int main()
{
    dd *part; unsigned *ticket; unsigned long long *st, h[5]; double *out;
    cudaMalloc(&part, 4096 * sizeof(dd) * 3); cudaMalloc(&ticket, 4); cudaMalloc(&st, 64); cudaMalloc(&out, 8);
    cudaMemset(ticket, 0, 4);
    for (int rep = 0; rep < 4; rep++) {
        k<3><<<296, 288>>>(part, ticket, st, out);
        cudaMemcpy(h, st, 40, cudaMemcpyDeviceToHost);
        printf("K=3 last CTA (ns): block tree %llu, publish+ticket %llu, fence %llu, fold %llu\n", h[1] - h[0], h[2] - h[1],
               h[3] - h[2], h[4] - h[3]);
        k<1><<<296, 288>>>(part, ticket, st, out);
        cudaMemcpy(h, st, 40, cudaMemcpyDeviceToHost);
        printf("K=1 last CTA (ns): block tree %llu, publish+ticket %llu, fence %llu, fold %llu\n", h[1] - h[0], h[2] - h[1],
               h[3] - h[2], h[4] - h[3]);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
