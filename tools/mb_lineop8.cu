// DMMA experiment for k_axis8's line operator (VERDICT r01 "next round" item 3; north_star: FP64 DMMA "only if
// ncu shows the small dense contractions actually gain"). Not part of libdg.
//
// Both kernels apply the 8x8 line operator B^ to the 64 lines (8 contiguous doubles each, the 128B-swizzled
// layout of k_axis8's TMA planes) of shared-memory cell blocks, one warp per cell, and write the 64 output lines
// back to shared memory — the per-line work of one k_axis8 pass without the neighbour couplings:
//   eo   : k_axis8's even/odd form (2 lines per lane: 4 x LDS.128, 8 + 8 adds, 2 x 4x4 DFMA blocks, 4 x STS.128)
//   dmma : mma.sync.m8n8k4.f64, Y (8 x 64) = B^ (8 x 8) X (8 x 64): per 8-line tile 2 k-chunks, the B^ fragment
//          in 2 registers per lane (vs ~32 table doubles of the even/odd form), X fragments by LDS.64
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_lineop8 tools/mb_lineop8.cu
#include <cstdio>
#include <cuda_runtime.h>

struct Tab {
    double Ee[4][4], Oo[4][4];
    double B[8][8];
};

__device__ __forceinline__ unsigned swz(unsigned off) { return off ^ (((off >> 7) & 7u) << 4); }
__device__ __forceinline__ double lds(unsigned a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void lds2(unsigned a, double& x, double& y)
{
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ void sts(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ void sts2(unsigned a, double x, double y)
{
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y));
}

constexpr int CELLS = 8;          // per CTA (one per warp), X and Y buffers: 2 x 32 KB
constexpr int CB = 512 * 8;       // bytes per cell

template <int MB>
__global__ void __launch_bounds__(256, MB) k_eo(double* out, int iters, const Tab T)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    const unsigned base = ((unsigned)__cvta_generic_to_shared(sm) + 1023u) & ~1023u;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < CELLS * 512; i += 256) sts(base + 8 * i, 1e-3 * (i % 97));
    __syncthreads();
    const unsigned X = base + warp * CB, Y = base + CELLS * CB + warp * CB;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int L = lane + 32 * q;
            double v[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) lds2(X + swz(8 * (8 * L + 2 * k)), v[2 * k], v[2 * k + 1]);
            double xe[4], xo[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) { xe[j] = v[j] + v[7 - j]; xo[j] = v[j] - v[7 - j]; }
            double y[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                double e = 0.0, o = 0.0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    e = fma(T.Ee[i][j], xe[j], e);
                    o = fma(T.Oo[i][j], xo[j], o);
                }
                y[i] = e + o;
                y[7 - i] = e - o;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) sts2(Y + swz(8 * (8 * L + 2 * k)), y[2 * k], y[2 * k + 1]);
        }
        __syncwarp();
    }
    if (lane == 0 && warp == 0) out[blockIdx.x] = lds(Y);
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int MB>
__global__ void __launch_bounds__(256, MB) k_dmma(double* out, int iters, const Tab T)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    const unsigned base = ((unsigned)__cvta_generic_to_shared(sm) + 1023u) & ~1023u;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < CELLS * 512; i += 256) sts(base + 8 * i, 1e-3 * (i % 97));
    __syncthreads();
    const unsigned X = base + warp * CB, Y = base + CELLS * CB + warp * CB;
    const int g = lane >> 2, k = lane & 3;
    // A fragment (row-major 8x4): lane holds A[g][k] of each k-chunk
    const double a0 = T.B[g][k], a1 = T.B[g][4 + k];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            // B fragment (col-major 4x8): lane holds B[k][n = g] = X of line 8t + g, component k (+4)
            const int line = 8 * t + g;
            const double b0 = lds(X + swz(8 * (8 * line + k)));
            const double b1 = lds(X + swz(8 * (8 * line + 4 + k)));
            double c0 = 0.0, c1 = 0.0;
            dmma(c0, c1, a0, b0);
            dmma(c0, c1, a1, b1);
            // C (8x8): lane holds C[g][2k], C[g][2k+1] = Y component g of lines 8t + 2k, 8t + 2k + 1
            sts(Y + swz(8 * (8 * (8 * t + 2 * k) + g)), c0);
            sts(Y + swz(8 * (8 * (8 * t + 2 * k + 1) + g)), c1);
        }
        __syncwarp();
    }
    if (lane == 0 && warp == 0) out[blockIdx.x] = lds(Y);
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    Tab T;
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) T.B[i][j] = (i == j ? 0.5 : 0.0) + 0.01 * (i - j);
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            T.Ee[i][j] = 0.5 * (T.B[i][j] + T.B[i][7 - j]);
            T.Oo[i][j] = 0.5 * (T.B[i][j] - T.B[i][7 - j]);
        }
    double* out;
    cudaMalloc(&out, sizeof(double) * sms * 64);
    const int smem = 2 * CELLS * CB + 1024;
    cudaFuncSetAttribute(k_eo<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_dmma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_eo<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_dmma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000;
    auto run = [&](const char* name, auto kern, int ctas_per_sm) {
        const int grid = sms * ctas_per_sm;
        kern<<<grid, 256, smem>>>(out, 10, T);
        cudaEventRecord(e0);
        kern<<<grid, 256, smem>>>(out, iters, T);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double cells = (double)grid * CELLS * iters;
        // useful line-operator FMAs: 64 lines x 64 per cell (the dense 8x8 product)
        printf("%-10s %d CTA/SM: %.3f ms  %.2f Gcells/s  dense-equivalent %.2f TFLOP/s\n", name, ctas_per_sm, ms,
               cells / ms / 1e6, cells * 64 * 64 * 2 / ms / 1e9);
    };
    run("eo", k_eo<2>, 2);
    run("dmma", k_dmma<2>, 2);
    run("eo", k_eo<3>, 3);
    run("dmma", k_dmma<3>, 3);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
