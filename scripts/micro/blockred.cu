// Micro-benchmark: cycles of block_reduce_dd<K> (common.cuh) for K = 1, 2, 3 in a
// 288-thread block (the row-warp kernels' shape): first (cold instruction cache)
// call and the average of 16 warm calls.
#include <cstdio>
#include "../../paper_2211_15605_b200/csrc/common.cuh"

namespace mfx { void set_error(const char *, ...) {} }
using namespace mfx;

template <int K>
__global__ void k(double *out, long long *cyc)
{
    __shared__ dd sh[9 * 3];
    dd v[K];
    for (int q = 0; q < K; q++) v[q] = dd{1.0 + threadIdx.x * 1e-3 + q, 1e-20};
    __syncthreads();
    long long t0 = clock64();
    block_reduce_dd<K>(v, sh);
    long long t1 = clock64();
    for (int r = 0; r < 16; r++) block_reduce_dd<K>(v, sh);
    long long t2 = clock64();
    if (threadIdx.x == 0) { cyc[2 * K] = t1 - t0; cyc[2 * K + 1] = (t2 - t1) / 16; out[K] = v[0].hi; }
}

int main()
{
    double *o; long long *c, h[8];
    cudaMalloc(&o, 64); cudaMalloc(&c, 64);
    k<1><<<1, 288>>>(o, c); k<2><<<1, 288>>>(o, c); k<3><<<1, 288>>>(o, c);
    cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("block_reduce_dd cycles: cold first call / warm average: K=1 %lld / %lld  K=2 %lld / %lld  K=3 %lld / %lld\n",
           h[2], h[3], h[4], h[5], h[6], h[7]);
    return 0;
}
