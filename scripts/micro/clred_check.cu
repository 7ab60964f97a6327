// Correctness stress of the push reduction (bicg_cluster.cu ClusterRed): each
// round every thread contributes an integer-valued double; CTAs are skewed by
// pseudo-random spins; every CTA checks the folded value against the exact sum.
#include <cstdio>
#include "../../paper_2211_15605_b200/csrc/common.cuh"
#include "../../paper_2211_15605_b200/csrc/tma.cuh"

namespace mfx { void set_error(const char *, ...) {} }
using namespace mfx;

constexpr int CT = 512, NW = 16;

template <int CL, int SKEW>
__global__ void __launch_bounds__(CT) k(unsigned *bad, int rounds)
{
    __shared__ __align__(16) dd wpart[3][NW];
    __shared__ __align__(16) dd red[2][3][CL];
    __shared__ __align__(8) uint64_t mb[2];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int rank = (int)cl_rank();
    if (tid == 0) {
        mbar_init(&mb[0], 1); mbar_init(&mb[1], 1);
        mbar_arrive_expect_tx(&mb[0], CL * 3 * 16); mbar_arrive_expect_tx(&mb[1], CL * 3 * 16);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync_full();
    uint32_t dst = mapa_u32(smem_u32(&red[0][0][rank]), lane & (CL - 1));
    uint32_t bar0 = mapa_u32(smem_u32(&mb[0]), lane & (CL - 1)), bar1 = mapa_u32(smem_u32(&mb[1]), lane & (CL - 1));
    uint32_t ph0 = 0, ph1 = 0;
    int buf = 0;
    unsigned nb = 0;
    for (int r = 0; r < rounds; r++) {
        if (SKEW) {
            unsigned h = (unsigned)(r * 2654435761u) ^ (unsigned)(rank * 40503u) ^ (unsigned)(tid * 97u);
            long long t0 = clock64();
            while (clock64() - t0 < (long long)(h % 2000)) {}
        }
        const int K = 1 + r % 3;
        dd v[3];
        for (int q = 0; q < 3; q++) v[q] = dd{(double)((r + 1) * (q + 1)) * (double)(tid + 1 + rank * 1000), 0.0};
        butterfly_k<3, 32>(v);
        if (lane == 0) for (int q = 0; q < 3; q++) wpart[q][wid] = v[q];
        __syncthreads();
        if (wid == 0) {
            dd y[3];
            for (int q = 0; q < 3; q++) y[q] = wpart[q][lane & (NW - 1)];
            butterfly_k<3, NW>(y);
            if (lane < CL)
                for (int q = 0; q < 3; q++)
                    push_f64x2(dst + (uint32_t)((buf * 3 + q) * CL * 16), q < K ? y[q].hi : 0.0, q < K ? y[q].lo : 0.0,
                               buf ? bar1 : bar0);
        }
        if (buf) { mbar_wait_cluster(&mb[1], ph1); ph1 ^= 1u; } else { mbar_wait_cluster(&mb[0], ph0); ph0 ^= 1u; }
        if (tid == 0) mbar_arrive_expect_tx(&mb[buf], CL * 3 * 16);
        dd y[3];
        for (int q = 0; q < 3; q++) y[q] = red[buf][q][lane & (CL - 1)];
        butterfly_k<3, CL>(y);
        // exact: sum over ranks, tids of (r+1)(q+1)(tid+1+1000 rank)
        for (int q = 0; q < K; q++) {
            double S = 0;
            // sum_{rank} sum_{t=1..CT} (t + 1000 rank) = CL*CT(CT+1)/2 + 1000*CT*CL(CL-1)/2
            S = (double)CL * CT * (CT + 1) / 2 + 1000.0 * CT * CL * (CL - 1) / 2;
            S *= (double)((r + 1) * (q + 1));
            if (y[q].hi + y[q].lo != S) nb++;
        }
        buf ^= 1;
    }
    if (nb) atomicAdd(bad, nb);
    cluster_sync_full();
}

template <int CL, int SKEW>
void run(unsigned *b, int rounds)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL); cfg.blockDim = dim3(CT); cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(k<CL, SKEW>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaMemset(b, 0, 4);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k<CL, SKEW>, b, rounds);
    unsigned h = 0;
    cudaError_t e2 = cudaDeviceSynchronize();
    cudaMemcpy(&h, b, 4, cudaMemcpyDeviceToHost);
    printf("CL %d skew %d rounds %d: launch %s sync %s, bad %u\n", CL, SKEW, rounds, cudaGetErrorString(e), cudaGetErrorString(e2), h);
}

int main()
{
    unsigned *b; cudaMalloc(&b, 4);
    run<8, 0>(b, 3000); run<16, 0>(b, 3000); run<8, 1>(b, 3000); run<16, 1>(b, 3000);
    return 0;
}
