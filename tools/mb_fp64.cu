// Microbenchmarks that decide the general kernel's design (not part of libdg):
//   dfma  : vector DFMA throughput
//   dmma  : FP64 tensor-core mma.sync m8n8k4 throughput (register operands only)
//   mix   : DMMA and DFMA interleaved in the same warps (do they share the FP64 datapath?)
//   lds   : LDS.64 throughput (conflict-free), doubles per clock per SM
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_fp64 tools/mb_fp64.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b)
{
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = fma(v[i], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
    if (s == 1.2345) out[blockIdx.x] = s;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int CH>
__global__ void __launch_bounds__(256) k_dmma(double* out, int iters, double a, double b)
{
    double c[CH][2];
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_mix(double* out, int iters, double a, double b)
{
    double c[4][2], v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma(c[i][0], c[i][1], a, b);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = fma(v[i], a, b);
        }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
    if (s == 1.2345) out[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_lds(double* out, int iters)
{
    __shared__ double sm[256 * 8];
    for (int i = threadIdx.x; i < 256 * 8; i += 256) sm[i] = i;
    __syncthreads();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + 8u * threadIdx.x;
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double v;
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + 2048u * u));
            s[u] += v;
        }
    }
    double t = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) t += s[u];
    if (t == 1.2345) out[blockIdx.x] = t;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * sms * 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * 8, block = 256;
    auto timeit = [&](auto launch) {
        launch();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t;
        cudaEventElapsedTime(&t, e0, e1);
        return (double)t;
    };
    const int it = 4000;
    double t = timeit([&] { k_dfma<<<grid, block>>>(out, it, 0.999999, 1e-7); });
    double fl = 2.0 * 8 * 16 * it * (double)grid * block;
    printf("dfma: %.2f TFLOP/s  (%.3f ms)\n", fl / t / 1e9, t);
    t = timeit([&] { k_dmma<4><<<grid, block>>>(out, it, 0.999999, 1e-7); });
    fl = 2.0 * 256 * 4 * 16 * it * (double)grid * block / 32;
    printf("dmma m8n8k4 (4 chains): %.2f TFLOP/s  (%.3f ms)\n", fl / t / 1e9, t);
    t = timeit([&] { k_dmma<8><<<grid, block>>>(out, it, 0.999999, 1e-7); });
    fl = 2.0 * 256 * 8 * 16 * it * (double)grid * block / 32;
    printf("dmma m8n8k4 (8 chains): %.2f TFLOP/s  (%.3f ms)\n", fl / t / 1e9, t);
    t = timeit([&] { k_mix<<<grid, block>>>(out, it, 0.999999, 1e-7); });
    double fl_mma = 2.0 * 256 * 4 * 16 * it * (double)grid * block / 32, fl_fma = 2.0 * 8 * 16 * it * (double)grid * block;
    printf("mix: dmma part %.2f + dfma part %.2f = %.2f TFLOP/s (%.3f ms)\n", fl_mma / t / 1e9, fl_fma / t / 1e9,
           (fl_mma + fl_fma) / t / 1e9, t);
    const int it2 = 20000;
    t = timeit([&] { k_lds<<<grid, block>>>(out, it2); });
    double lds = 8.0 * it2 * (double)grid * block;
    printf("lds.64: %.1f Gdoubles/s = %.2f doubles/clk/SM at %d MHz\n", lds / t / 1e6, lds / (t * 1e-3) / sms / (clk * 1e3),
           clk / 1000);
    cudaError_t e = cudaGetLastError();
    printf("err: %s\n", cudaGetErrorString(e));
    return 0;
}
