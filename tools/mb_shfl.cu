// Microbenchmark (development): do warp shuffles compete with shared-memory loads for the LSU data pipe?
// Kernels: L (8-byte conflict-free shared loads), S (64-bit shuffles), LS (both in one loop); independent chains.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double lds(unsigned a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(512) k(double* out, int iters)
{
    __shared__ double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double a0 = lane, a1 = 1, a2 = 2, a3 = 3, b0 = 4, b1 = 5, b2 = 6, b3 = 7;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(s) + 8u * (((threadIdx.x & ~31) * 4 + lane) & 4095);
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 2) {
            const unsigned o = sb + 8u * ((it * 32) & 1023);
            a0 += lds(o);
            a1 += lds(o + 2048);
            a2 += lds(o + 4096);
            a3 += lds(o + 6144);
        }
        if (MODE == 1 || MODE == 2) {
            b0 = __shfl_sync(0xffffffffu, b0, (lane + 1) & 31) + 1.0;
            b1 = __shfl_sync(0xffffffffu, b1, (lane + 3) & 31) + 1.0;
            b2 = __shfl_sync(0xffffffffu, b2, (lane + 5) & 31) + 1.0;
            b3 = __shfl_sync(0xffffffffu, b3, (lane + 7) & 31) + 1.0;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + b0 + b1 + b2 + b3;
}

int main()
{
    double* out;
    cudaMalloc(&out, sizeof(double) * 148 * 4 * 512);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    auto run = [&](auto kern, const char* name) {
        kern<<<148 * 4, 512>>>(out, 100);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        kern<<<148 * 4, 512>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warp_ops = 148.0 * 4 * 16 * iters * 4; // 4 ops of each kind per iteration per warp
        printf("%-3s %8.3f ms  %.3f warp-ops(each kind) / clk / SM (at 1.9 GHz)\n", name, ms,
               warp_ops / 148 / (ms * 1e-3 * 1.9e9));
    };
    run(k<0>, "L");
    run(k<1>, "S");
    run(k<2>, "LS");
    return 0;
}
