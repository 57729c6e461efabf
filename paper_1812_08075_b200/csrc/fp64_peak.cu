// FP64 DFMA throughput microbenchmark: the measured denominator for the
// "alu" roofline next to the nominal SMs x 64 DFMA/clk x 2 x clock figure.
// Every thread runs 8 independent DFMA chains (enough ILP to cover the DFMA latency with
// 8 warps per SM sub-partition); the grid is a multiple of the SM count.
#include "../../include/dg.h"

#include <cuda_runtime.h>

namespace {

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b)
{
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = fma(v[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
    if (s == 1.2345) out[blockIdx.x] = s; // never true; keeps the chains live
}

} // namespace

extern "C" int dg_bench_fp64(int device, int iters, double* tflops, double* ms)
{
    if (!tflops || !ms || iters < 1) return DG_ERR_INVALID;
    if (cudaSetDevice(device) != cudaSuccess) return DG_ERR_CUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double) * sms * 8) != cudaSuccess) return DG_ERR_OOM;
    const int grid = sms * 8, block = 256; // 64 warps per SM
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<grid, block>>>(out, iters / 4 + 1, 0.999999, 1e-7); // warm-up
    cudaEventRecord(e0);
    k_dfma<<<grid, block>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return DG_ERR_CUDA;
    const double flops = 2.0 * 8 * 16 * (double)iters * grid * block;
    *ms = t;
    *tflops = flops / (t * 1e-3) / 1e12;
    return DG_OK;
}
