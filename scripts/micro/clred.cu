// Micro-benchmark: cost of the pieces of the single-cluster solver's push
// reduction (bicg_cluster.cu) on a 16-CTA x 512-thread cluster, K = 1..3:
// lane butterfly only / + CTA fold / + push + wait / full (+ final fold),
// cycles per reduction averaged over 64 back-to-back reductions (CTA 0).
#include <cstdio>
#include "../../paper_2211_15605_b200/csrc/common.cuh"
#include "../../paper_2211_15605_b200/csrc/tma.cuh"

namespace mfx { void set_error(const char *, ...) {} }
using namespace mfx;

constexpr int CT = 512, NW = 16, CL = 16;

template <int K, int VAR>
__global__ void __launch_bounds__(CT) k(double *out, long long *cyc)
{
    __shared__ __align__(16) dd wpart[3][NW];
    __shared__ __align__(16) dd red[2][3][CL];
    __shared__ __align__(8) uint64_t mb[2];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int rank = (int)cl_rank();
    if (tid == 0) { mbar_init(&mb[0], 1); mbar_init(&mb[1], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    cluster_sync_full();
    uint32_t dst = mapa_u32(smem_u32(&red[0][0][rank]), lane & (CL - 1));
    uint32_t bar0 = mapa_u32(smem_u32(&mb[0]), lane & (CL - 1)), bar1 = bar0 + 8;
    uint32_t ph0 = 0, ph1 = 0;
    int buf = 0;
    dd v[K];
    for (int q = 0; q < K; q++) v[q] = dd{1.0 + tid * 1e-3 + q + rank, 1e-20};
    double acc = 0.0;
    cluster_sync_full();
    long long t0 = clock64();
    for (int r = 0; r < 64; r++) {
        if (VAR >= 2 && tid == 0) mbar_arrive_expect_tx(&mb[buf], (uint32_t)(CL * K * 16));
        dd x[K];
        for (int q = 0; q < K; q++) x[q] = v[q];
        butterfly_k<K, 32>(x);
        if (VAR >= 1) {
            if (lane == 0) for (int q = 0; q < K; q++) wpart[q][wid] = x[q];
            __syncthreads();
            if (wid == 0) {
                dd y[K];
                for (int q = 0; q < K; q++) y[q] = wpart[q][lane & (NW - 1)];
                butterfly_k<K, NW>(y);
                if (VAR >= 2 && lane < CL)
                    for (int q = 0; q < K; q++)
                        push_f64x2(dst + (uint32_t)((buf * 3 + q) * CL * 16), y[q].hi, y[q].lo, buf ? bar1 : bar0);
                x[0] = y[0];
            }
            if (VAR == 1) __syncthreads();
        }
        if (VAR >= 2) {
            if (buf) { mbar_wait(&mb[1], ph1); ph1 ^= 1u; } else { mbar_wait(&mb[0], ph0); ph0 ^= 1u; }
            dd y[K];
            for (int q = 0; q < K; q++) y[q] = red[buf][q][lane & (CL - 1)];
            if (VAR >= 3) butterfly_k<K, CL>(y);
            x[0] = y[0];
            buf ^= 1;
        }
        acc += x[0].hi;
        v[0].lo = acc * 1e-30;   // carry a dependence into the next round
    }
    long long t1 = clock64();
    out[blockIdx.x * CT + tid] = acc;
    if (tid == 0 && rank == 0) cyc[VAR * 4 + K] = (t1 - t0) / 64;
    cluster_sync_full();
}

__global__ void lat(double *out, long long *cyc, double a, double b)
{
    double x = a;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) x = x + b;
    }
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) x = __shfl_xor_sync(0xffffffffu, x, 1);
    }
    long long t2 = clock64();
    dd d{x, 0.0};
#pragma unroll 1
    for (int i = 0; i < 64; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) d = dd_add_fast(d, dd{b, 1e-20});
    }
    long long t3 = clock64();
    out[threadIdx.x] = d.hi + d.lo;
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 1024; cyc[1] = (t2 - t1) / 1024; cyc[2] = (t3 - t2) / 1024; }
}

template <int K, int VAR>
void run(double *o, long long *c)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL); cfg.blockDim = dim3(CT); cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(k<K, VAR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k<K, VAR>, o, c);
    if (e != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(e));
}

int main()
{
    double *o; long long *c, h[32];
    cudaMalloc(&o, CL * CT * 8); cudaMalloc(&c, 32 * 8); cudaMemset(c, 0, 32 * 8);
    lat<<<1, 32>>>(o, c, 1.0, 1e-9);
    cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("latency cycles: DADD %lld  SHFL.f64 %lld  dd_add_fast %lld\n", h[0], h[1], h[2]);
    cudaMemset(c, 0, 32 * 8);
    for (int w = 0; w < 2; w++) {
        run<1, 0>(o, c); run<2, 0>(o, c); run<3, 0>(o, c);
        run<1, 1>(o, c); run<2, 1>(o, c); run<3, 1>(o, c);
        run<1, 2>(o, c); run<2, 2>(o, c); run<3, 2>(o, c);
        run<1, 3>(o, c); run<2, 3>(o, c); run<3, 3>(o, c);
    }
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, c, 32 * 8, cudaMemcpyDeviceToHost);
    printf("sync: %s\n", cudaGetErrorString(e));
    const char *nm[4] = {"lane butterfly", "+ CTA fold", "+ push/wait", "full"};
    for (int v = 0; v < 4; v++) printf("%-16s K=1 %lld  K=2 %lld  K=3 %lld cycles\n", nm[v], h[v * 4 + 1], h[v * 4 + 2], h[v * 4 + 3]);
    return 0;
}
