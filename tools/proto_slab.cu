// Prototype (development, not part of libdg): the VOLUME part of the affine c(x) operator (stage 1 -> 2 -> 3 of Alg.
// assembly, collocation, n = 5) in a slab-owner layout, to measure whether keeping a whole j0-slab of a cell in one
// thread's registers (stage-1 / 3 contractions along j1 and j2 in registers, only j0 transposed through shared memory)
// beats k_gen's line-owner layout. Random tables; checked against a direct per-DOF reference kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/proto_slab tools/proto_slab.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <cmath>

constexpr int N = 5, N2 = 25, N3 = 125;
struct Tab {
    double D[N * N];
    double w[N];
};
constexpr int CX = 2 * 3 * (N + 1); // complex entries per cell: [k][b][q]

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity)
{
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     s32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(s32(b)) : "memory");
}

// ---------------------------------------------------------------- reference: one thread per output DOF
__device__ double cval(const double2* cx, int p0, int p1, int p2)
{
    // z_k = E_k0(p0) E_k1(p1) E_k2(p2); c = 1 + 0.5 Im(z_0) Re(z_1)
    double zr[2], zi[2];
    for (int k = 0; k < 2; ++k) {
        double2 a = cx[(k * 3 + 0) * (N + 1) + p0], b = cx[(k * 3 + 1) * (N + 1) + p1], c = cx[(k * 3 + 2) * (N + 1) + p2];
        double r1 = a.x * b.x - a.y * b.y, i1 = a.x * b.y + a.y * b.x;
        zr[k] = r1 * c.x - i1 * c.y;
        zi[k] = r1 * c.y + i1 * c.x;
    }
    return 1.0 + 0.5 * zi[0] * zr[1];
}
__global__ void k_ref(const double* x, double* r, const double* gt, const double2* cxt, long long ncell, Tab T)
{
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncell * N3) return;
    long long c = t / N3;
    int J = (int)(t % N3), j[3] = {J % N, (J / N) % N, J / N2};
    const double* X = x + c * N3;
    const double* g = gt + c * 6;
    const double2* cx = reinterpret_cast<const double2*>(cxt) + c * CX;
    double acc = 0;
    for (int d = 0; d < 3; ++d)
        for (int q = 0; q < N; ++q) {
            int p[3] = {j[0], j[1], j[2]};
            p[d] = q;
            double G[3];
            for (int e = 0; e < 3; ++e) {
                double s = 0;
                for (int k = 0; k < N; ++k) {
                    int pp[3] = {p[0], p[1], p[2]};
                    pp[e] = k;
                    s += T.D[p[e] * N + k] * X[pp[0] + N * pp[1] + N2 * pp[2]];
                }
                G[e] = s;
            }
            double cw = T.w[p[0]] * T.w[p[1]] * T.w[p[2]] * cval(cx, p[0], p[1], p[2]);
            double Q[3] = {g[0] * G[0] + g[3] * G[1] + g[4] * G[2], g[3] * G[0] + g[1] * G[1] + g[5] * G[2],
                           g[4] * G[0] + g[5] * G[1] + g[2] * G[2]};
            acc += T.D[q * N + j[d]] * cw * Q[d];
        }
    r[t] = acc;
}

// ---------------------------------------------------------------- slab-owner volume kernel
// tile T1 x T2 cells in (i1, i2), marching along i0 over chunk planes; thread (cell mc, a): the slab j0 = a of its
// cell (registers) and the d0 lines (., a, c), c < N (DR role). Shared: X own planes (2 buffers), W (G0 -> Q0 -> R0),
// geometry G~ (6) and c(x) factors per cell (2 buffers).
template <int T1, int T2>
struct Lay {
    static constexpr int NC = T1 * T2, NT = NC * N;
    static constexpr int XS = 0, W = XS + 2 * NC * N3, GT = W + NC * N3, CXS = GT + 2 * NC * 6;
    static constexpr int END = CXS + 2 * NC * CX * 2;
    static constexpr int BYTES = END * 8 + 16;
};

template <int T1, int T2>
__global__ void __launch_bounds__(Lay<T1, T2>::NT) k_slab(const double* __restrict__ x, double* __restrict__ r,
                                                         const double* __restrict__ gt, const double* __restrict__ cxt,
                                                         int N1, int N2c, int L, int chunk, Tab T)
{
    using Y = Lay<T1, T2>;
    constexpr int NC = Y::NC, NT = Y::NT;
    extern __shared__ __align__(16) double sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + Y::END);
    double* W = sm + Y::W;
    const int tid = threadIdx.x;
    const int nt2 = N2c / T2, ntiles = (N1 / T1) * nt2;
    const int ch = blockIdx.x / ntiles, tile = blockIdx.x % ntiles, ti1 = tile / nt2, ti2 = tile % nt2;
    const int p0 = ch * chunk, p1 = min(L, p0 + chunk);
    const long long PC = (long long)N1 * N2c;
    const int mc = tid / N, a = tid % N;
    __shared__ double sD[N * N], sW[N];
    if (tid < N * N) sD[tid] = T.D[tid];
    if (tid < N) sW[tid] = T.w[tid];
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int lp, int buf) {
        mbar_expect_tx(bar, NC * (N3 + 6 + 2 * CX) * 8);
        for (int c1 = 0; c1 < T1; ++c1) {
            const long long cell = lp * PC + (long long)(ti1 * T1 + c1) * N2c + ti2 * T2;
            bulk(sm + Y::XS + buf * NC * N3 + c1 * T2 * N3, x + cell * N3, T2 * N3 * 8, bar);
            bulk(sm + Y::GT + buf * NC * 6 + c1 * T2 * 6, gt + cell * 6, T2 * 6 * 8, bar);
            bulk(sm + Y::CXS + buf * NC * CX * 2 + c1 * T2 * CX * 2, cxt + cell * CX * 2, T2 * CX * 2 * 8, bar);
        }
    };
    if (tid == 0) issue(p0, 0);
    for (int lp = p0, s = 0; lp < p1; ++lp, ++s) {
        const int buf = s & 1;
        mbar_wait(bar, s & 1);
        __syncthreads();
        if (tid == 0 && lp + 1 < p1) issue(lp + 1, buf ^ 1);
        const double* X = sm + Y::XS + buf * NC * N3 + mc * N3;
        double* Wc = W + mc * N3;
        // ---- P1: d0 lines (., a, c) -> G0 into W; the slab S[b][c] = X(a, b, c) into registers
#pragma unroll
        for (int c = 0; c < N; ++c) {
            double v[N];
#pragma unroll
            for (int j = 0; j < N; ++j) v[j] = X[j + N * a + N2 * c];
#pragma unroll
            for (int q = 0; q < N; ++q) {
                double s = 0;
#pragma unroll
                for (int k = 0; k < N; ++k) s = fma(sD[q * N + k], v[k], s);
                Wc[q + N * a + N2 * c] = s;
            }
        }
        double S[N][N];
#pragma unroll
        for (int b = 0; b < N; ++b)
#pragma unroll
            for (int c = 0; c < N; ++c) S[b][c] = X[a + N * b + N2 * c];
        __syncthreads();
        // ---- P2: stage 2 at the slab's points; Q1 / Q2 contracted in registers into R; Q0 into W (in place)
        const double* g = sm + Y::GT + buf * NC * 6 + mc * 6;
        const double g0 = g[0], g1 = g[1], g2 = g[2], g3 = g[3], g4 = g[4], g5 = g[5];
        const double2* cx = reinterpret_cast<const double2*>(sm + Y::CXS + buf * NC * CX * 2) + mc * CX;
        const double2 e00 = cx[(0 * 3 + 0) * (N + 1) + a], e10 = cx[(1 * 3 + 0) * (N + 1) + a];
        double R[N][N];
#pragma unroll
        for (int b = 0; b < N; ++b)
#pragma unroll
            for (int c = 0; c < N; ++c) R[b][c] = 0;
#pragma unroll
        for (int c = 0; c < N; ++c) {
            const double2 e02 = cx[(0 * 3 + 2) * (N + 1) + c], e12 = cx[(1 * 3 + 2) * (N + 1) + c];
            const double zr0 = e00.x * e02.x - e00.y * e02.y, zi0 = e00.x * e02.y + e00.y * e02.x;
            const double zr1 = e10.x * e12.x - e10.y * e12.y, zi1 = e10.x * e12.y + e10.y * e12.x;
            double G1c[N], Q1c[N];
#pragma unroll
            for (int b = 0; b < N; ++b) { // G1 along j1 (column c of the slab)
                double s = 0;
#pragma unroll
                for (int k = 0; k < N; ++k) s = fma(sD[b * N + k], S[k][c], s);
                G1c[b] = s;
            }
#pragma unroll
            for (int b = 0; b < N; ++b) {
                double G2 = 0;
#pragma unroll
                for (int k = 0; k < N; ++k) G2 = fma(sD[c * N + k], S[b][k], G2);
                const double G0 = Wc[a + N * b + N2 * c];
                const double2 e01 = cx[(0 * 3 + 1) * (N + 1) + b], e11 = cx[(1 * 3 + 1) * (N + 1) + b];
                const double im0 = zr0 * e01.y + zi0 * e01.x;
                const double re1 = zr1 * e11.x - zi1 * e11.y;
                const double cw = sW[a] * sW[b] * sW[c] * fma(0.5 * im0, re1, 1.0);
                const double G1 = G1c[b];
                const double q0 = cw * fma(g0, G0, fma(g3, G1, g4 * G2));
                Q1c[b] = cw * fma(g3, G0, fma(g1, G1, g5 * G2));
                const double q2 = cw * fma(g4, G0, fma(g5, G1, g2 * G2));
                Wc[a + N * b + N2 * c] = q0;
#pragma unroll
                for (int k = 0; k < N; ++k) R[b][k] = fma(sD[c * N + k], q2, R[b][k]); // D^T along j2
            }
#pragma unroll
            for (int k = 0; k < N; ++k) { // D^T along j1 of the column
                double s = R[k][c];
#pragma unroll
                for (int b = 0; b < N; ++b) s = fma(sD[b * N + k], Q1c[b], s);
                R[k][c] = s;
            }
        }
        __syncthreads();
        // ---- P3: D^T along j0 of the d0 lines (., a, c) in W (in place)
#pragma unroll
        for (int c = 0; c < N; ++c) {
            double v[N];
#pragma unroll
            for (int j = 0; j < N; ++j) v[j] = Wc[j + N * a + N2 * c];
#pragma unroll
            for (int k = 0; k < N; ++k) {
                double s = 0;
#pragma unroll
                for (int q = 0; q < N; ++q) s = fma(sD[q * N + k], v[q], s);
                Wc[k + N * a + N2 * c] = s;
            }
        }
        __syncthreads();
        // ---- P4: sum and write r once (the slab's points)
        const long long cell = lp * PC + (long long)(ti1 * T1 + mc / T2) * N2c + ti2 * T2 + mc % T2;
        double* dst = r + cell * N3;
#pragma unroll
        for (int b = 0; b < N; ++b)
#pragma unroll
            for (int c = 0; c < N; ++c) dst[a + N * b + N2 * c] = R[b][c] + Wc[a + N * b + N2 * c];
    }
}

int main(int argc, char** argv)
{
    const int NN = argc > 1 ? atoi(argv[1]) : 128;
    const long long ncell = (long long)NN * NN * NN;
    Tab T;
    srand(1);
    for (int i = 0; i < N * N; ++i) T.D[i] = (rand() / (double)RAND_MAX) - 0.5;
    for (int i = 0; i < N; ++i) T.w[i] = 0.1 + rand() / (double)RAND_MAX;
    double *x, *r, *rr, *gt, *cx;
    cudaMalloc(&x, ncell * N3 * 8);
    cudaMalloc(&r, ncell * N3 * 8);
    cudaMalloc(&rr, ncell * N3 * 8);
    cudaMalloc(&gt, ncell * 6 * 8);
    cudaMalloc(&cx, ncell * CX * 2 * 8);
    {
        std::vector<double> h(ncell * CX * 2);
        for (auto& v : h) v = rand() / (double)RAND_MAX - 0.5;
        cudaMemcpy(cx, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        std::vector<double> hg(ncell * 6);
        for (auto& v : hg) v = rand() / (double)RAND_MAX;
        cudaMemcpy(gt, hg.data(), hg.size() * 8, cudaMemcpyHostToDevice);
        std::vector<double> hx(ncell * N3);
        for (auto& v : hx) v = rand() / (double)RAND_MAX - 0.5;
        cudaMemcpy(x, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice);
    }
    auto run = [&](auto kern, int T1, int T2, int NT, int bytes, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        const int chunk = 16;
        const int grid = (NN / T1) * (NN / T2) * ((NN + chunk - 1) / chunk);
        kern<<<grid, NT, bytes>>>(x, r, gt, cx, NN, NN, NN, chunk, T);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        const int R = 10;
        for (int i = 0; i < R; ++i) kern<<<grid, NT, bytes>>>(x, r, gt, cx, NN, NN, NN, chunk, T);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s %dx%d: %.4f ms per apply (%lld cells, %.1f GDOF/s)\n", name, T1, T2, ms / R, ncell, ncell * N3 / (ms / R * 1e-3) / 1e9);
    };
    run(k_slab<4, 8>, 4, 8, Lay<4, 8>::NT, Lay<4, 8>::BYTES, "slab");
    run(k_slab<4, 4>, 4, 4, Lay<4, 4>::NT, Lay<4, 4>::BYTES, "slab");
    run(k_slab<2, 8>, 2, 8, Lay<2, 8>::NT, Lay<2, 8>::BYTES, "slab");
    if (NN <= 32) { // check against the direct reference
        k_ref<<<(unsigned)((ncell * N3 + 255) / 256), 256>>>(x, rr, gt, reinterpret_cast<const double2*>(cx), ncell, T);
        k_slab<4, 8><<<(NN / 4) * (NN / 8) * ((NN + 15) / 16), Lay<4, 8>::NT, Lay<4, 8>::BYTES>>>(x, r, gt, cx, NN, NN, NN, 16, T);
        cudaDeviceSynchronize();
        std::vector<double> a(ncell * N3), b(ncell * N3);
        cudaMemcpy(a.data(), r, a.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(b.data(), rr, b.size() * 8, cudaMemcpyDeviceToHost);
        double md = 0, mx = 0;
        for (size_t i = 0; i < a.size(); ++i) { md = fmax(md, fabs(a[i] - b[i])); mx = fmax(mx, fabs(b[i])); }
        printf("check: max|slab - ref| / max|ref| = %.3e\n", md / mx);
    }
    return 0;
}
