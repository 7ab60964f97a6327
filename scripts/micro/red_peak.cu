// red_peak.cu -- measured ceiling for the PIC deposits:
// fp64 global reductions (RED.E.ADD.F64) per second on this B200, for
// (a) random addresses spread over an L2-resident 32 MiB region,
// (b) random addresses over 256 MiB (L2 misses), (c) warp-contiguous runs.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o red_peak red_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash32(unsigned x)
{
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void k_red(double *buf, unsigned mask, int per_thread)
{
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int q = 0; q < per_thread; q++) {
        unsigned idx;
        if (MODE == 0) idx = hash32(t * 131u + q) & mask;
        else idx = ((hash32((t >> 5) * 977u + q) & mask) & ~31u) + (threadIdx.x & 31);
        atomicAdd(buf + idx, 1.0);
    }
}

int main()
{
    double *buf;
    const size_t big = 256ull << 20;
    cudaMalloc(&buf, big);
    cudaMemset(buf, 0, big);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = 148 * 8, threads = 256, per = 64;
    struct { const char *name; unsigned mask; int mode; } cases[] = {
        {"random_32MiB_L2", (32u << 20) / 8 - 1, 0},
        {"random_256MiB", (256u << 20) / 8 - 1, 0},
        {"warp_contiguous_32MiB", (32u << 20) / 8 - 1, 1},
    };
    for (auto &c : cases) {
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(a);
            if (c.mode == 0) k_red<0><<<blocks, threads>>>(buf, c.mask, per);
            else k_red<1><<<blocks, threads>>>(buf, c.mask, per);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2)
                printf("{\"case\": \"%s\", \"reductions_per_s\": %.4g, \"ms\": %.4f}\n", c.name,
                       (double)blocks * threads * per / (ms * 1e-3), ms);
        }
    }
    return 0;
}
