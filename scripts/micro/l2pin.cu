// Micro-benchmark: can a 64 MB read-only vector (BiCGSTAB's r^ at c2) stay
// L2-resident on B200 while ~600 MB per pass streams past it?  A K3-like
// kernel reads A + 5 streaming arrays and writes 2 (8 x 64 MB per pass);
// modes: 0 plain loads; 1 A with an L2::evict_last policy, streams
// evict_first; 2 = 1 + a persisting-L2 carve-out and an access-policy window
// on A; 3 = window only (plain loads).  Times per pass (CUDA events).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 ld_pol(const double *p, unsigned long long pol)
{
    double2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ld_plain(const double *p) { return __ldg((const double2 *)p); }

template <int MODE>
__global__ void k(long long n, const double *A, const double *B0, const double *B1, const double *B2,
                  const double *B3, const double *B4, double *W0, double *W1, double *out)
{
    unsigned long long pl = 0, pf = 0;
    if (MODE == 1 || MODE == 2) {
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
    }
    double acc = 0.0;
    for (long long i = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x); i < n; i += 2LL * gridDim.x * blockDim.x) {
        double2 a, b0, b1, b2, b3, b4;
        if (MODE == 1 || MODE == 2) {
            a = ld_pol(A + i, pl);
            b0 = ld_pol(B0 + i, pf); b1 = ld_pol(B1 + i, pf); b2 = ld_pol(B2 + i, pf);
            b3 = ld_pol(B3 + i, pf); b4 = ld_pol(B4 + i, pf);
        } else {
            a = ld_plain(A + i);
            b0 = ld_plain(B0 + i); b1 = ld_plain(B1 + i); b2 = ld_plain(B2 + i); b3 = ld_plain(B3 + i); b4 = ld_plain(B4 + i);
        }
        double2 w0 = make_double2(b0.x + b1.x * b2.x, b0.y + b1.y * b2.y);
        double2 w1 = make_double2(b3.x - b4.x * a.x, b3.y - b4.y * a.y);
        *(double2 *)(W0 + i) = w0;
        *(double2 *)(W1 + i) = w1;
        acc += a.x * w1.x + a.y * w1.y;
    }
    if (acc == 12345.0) out[0] = acc;
}

int main()
{
    const long long n = 8LL << 20;   // 8M doubles = 64 MiB
    double *buf;
    cudaMalloc(&buf, 8 * n * 8 + 64);
    cudaMemset(buf, 0, 8 * n * 8);
    double *A = buf, *B[5], *W[2];
    for (int q = 0; q < 5; q++) B[q] = buf + (1 + q) * n;
    W[0] = buf + 6 * n; W[1] = buf + 7 * n;
    double *out = buf + 8 * n;
    int dev = 0, maxp = 0, l2 = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    printf("L2 %d MB, max persisting %d MB\n", l2 >> 20, maxp >> 20);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int grid = 148 * 8, block = 256;
    for (int mode = 0; mode < 4; mode++) {
        if (mode >= 2) {
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp);
            cudaStreamAttrValue at = {};
            at.accessPolicyWindow.base_ptr = A;
            at.accessPolicyWindow.num_bytes = n * 8;
            at.accessPolicyWindow.hitRatio = (float)((double)maxp / (n * 8) < 1.0 ? (double)maxp / (n * 8) : 1.0);
            at.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            at.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &at);
        }
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0, s);
            for (int it = 0; it < 20; it++) {
                if (mode == 0 || mode == 3) k<0><<<grid, block, 0, s>>>(n, A, B[0], B[1], B[2], B[3], B[4], W[0], W[1], out);
                else k<1><<<grid, block, 0, s>>>(n, A, B[0], B[1], B[2], B[3], B[4], W[0], W[1], out);
            }
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("mode %d rep %d: %.1f us per pass (%.0f GB/s over 8 x 64 MiB)\n", mode, rep, ms * 1e3 / 20,
                   8.0 * n * 8 / (ms * 1e-3 / 20) / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
