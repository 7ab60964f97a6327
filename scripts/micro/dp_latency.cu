// Micro-benchmark: dependent FP64 add / fma, SHFL of a double, FP32 add latency
// on sm_100a (clock64 around 16x-unrolled dependent chains).
#include <cstdio>
#include <cuda_runtime.h>

#define R16(s) s s s s s s s s s s s s s s s s
__global__ void k(double *out, long long *cyc, double a, double b)
{
    double x = a;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; i++) { R16(x = x + b;) }
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; i++) { R16(x = fma(x, a, b);) }
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; i++) { R16(x = __shfl_xor_sync(0xffffffffu, x, 1);) }
    long long t3 = clock64();
    float f = (float)x, fb = (float)b;
#pragma unroll 1
    for (int i = 0; i < 256; i++) { R16(f = f + fb;) }
    long long t4 = clock64();
    out[threadIdx.x] = x + f;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}

int main()
{
    double *o; long long *c, h[4];
    cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
    for (int rep = 0; rep < 2; rep++) {
        k<<<1, 32>>>(o, c, 1.0000001, 1e-9);
        cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    }
    printf("DADD dependent latency %.1f cycles\n", h[0] / 4096.0);
    printf("DFMA dependent latency %.1f cycles\n", h[1] / 4096.0);
    printf("SHFL of a double (2 x SHFL.BFLY) %.1f cycles\n", h[2] / 4096.0);
    printf("FADD dependent latency %.1f cycles\n", h[3] / 4096.0);
    return 0;
}
