// K_axis8: axis-aligned Poisson (c = 1), n = 8 (Q7, cfg3) — the benchmark kernel.
//
// Algebra (exact reordering of Alg. assembly, for J = diag(h), c = 1):
// with collocation (A = I) the flux of stage 2 is diagonal, so stage 1 -> 2 -> 3 along one
// direction d collapses into the 1D stiffness  (1/h_d) D^T W D  applied to every line of the
// cell along d, scaled by the tangential weights w_a w_b h_t1 h_t2. The face terms of
// Eq. diffreac_weak (theta = -1) on faces normal to d only touch the same lines
// (tangential basis functions are nodal at the face quadrature points), so per line
//
//   r_line += S_ab [ B^ x_line + a^_L u_L + b^_L g_L + a^_R u_R + b^_R g_R ],  S_ab = w_a w_b h_t1 h_t2 / h_d
//   B^   = D^T W D + 1/2 (e0 d0^T + d0 e0^T - e1 d1^T - d1 e1^T) + P (e0 e0^T + e1 e1^T),  P = penalty_scale k(k+1)
//   u_L = e1.x_L, g_L = d1.x_L  (traces of the lower neighbour along d; 1-point tables)
//   u_R = e0.x_R, g_R = d0.x_R  (upper neighbour),  a^_L = -d0/2 - P e0, b^_L = e0/2, a^_R = d1/2 - P e1, b^_R = -e1/2.
// This is the sum-factorised operator with the face contraction done first in the normal
// direction. B^ is centro-symmetric (symmetric Gauss nodes), so every line product
// runs in even/odd form: 2 (4x4) products instead of one 8x8.
//
// Mapping (B200): one CTA (256 threads, 1 per SM, 192 KB smem) owns a 4x4 tile of cells in
// (i1, i2) and MARCHES along i0 through the planes [p_begin, p_end):
//   * each plane's 16 blocks (64 KB) arrive by TMA (cp.async.bulk.tensor, 128B swizzle) into a
//     double buffer one plane ahead of use;
//   * pass d=1 and pass d=2: a thread owns one line position across the 4 cells of a tile row,
//     so neighbour traces inside the tile stay in registers; the ring cells outside the tile are
//     read from L2 (their owner CTAs stream them concurrently);
//   * pass d=0 (the marching direction): the lower neighbour's traces are carried in registers
//     from the previous plane, the upper neighbour's come from the prefetched next plane;
//   * partial sums of the three passes meet in a swizzled smem buffer; the d=0 pass adds them
//     and writes r straight to global memory, once, with 64-byte coalesced rows.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace dg {

struct AxisTab8 {
    double Ee[4][4], Oo[4][4];           // even/odd halves of B^ (with the 1/2)
    double te[4], to[4], qe[4], qo[4];   // e0 and d0 in even/odd form
    double aue[4], age[4], auo[4], ago[4]; // neighbour-trace coefficients in even/odd form
    double e0[8], d0[8];
    double w[8];
    double c[3];                         // h_t1 h_t2 / h_d
};

namespace ax8 {

constexpr int N = 8, T = 4, NT = 256;
constexpr int CELL_BYTES = N * N * N * 8;        // 4096
constexpr int BUF_BYTES = T * T * CELL_BYTES;    // 65536
constexpr int SMEM_BYTES = 3 * BUF_BYTES + 1024; // X0, X1, R (+ barriers, alignment slack)

__device__ __forceinline__ uint32_t swz(uint32_t off) { return off ^ (((off >> 7) & 7u) << 4); }

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// Even/odd line kernel: given xe, xo (4 each) and neighbour traces, return ye, yo.
__device__ __forceinline__ void line_eo(const AxisTab8& A, const double xe[4], const double xo[4], double uL, double gL,
                                        double uR, double gR, double ye[4], double yo[4])
{
    const double su = uL + uR, du = uL - uR, sg = gL + gR, dg = gL - gR;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        double e = fma(A.aue[i], su, A.age[i] * dg);
        double o = fma(A.auo[i], du, A.ago[i] * sg);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            e = fma(A.Ee[i][j], xe[j], e);
            o = fma(A.Oo[i][j], xo[j], o);
        }
        ye[i] = e;
        yo[i] = o;
    }
}

// traces of a line in even/odd form: u0 = e0.x, u1 = e1.x, g0 = d0.x, g1 = d1.x
__device__ __forceinline__ void traces_eo(const AxisTab8& A, const double xe[4], const double xo[4], double& u0,
                                          double& u1, double& g0, double& g1)
{
    double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        a = fma(A.te[j], xe[j], a);
        b = fma(A.to[j], xo[j], b);
        c = fma(A.qe[j], xe[j], c);
        d = fma(A.qo[j], xo[j], d);
    }
    u0 = a + b;
    u1 = a - b;
    g0 = c + d;
    g1 = d - c;
}

} // namespace ax8

// grid: (N1/4) * (N2/4) CTAs, block 256, dynamic smem ax8::SMEM_BYTES
__global__ void __launch_bounds__(ax8::NT, 1)
k_axis8(const __grid_constant__ CUtensorMap tmx, const double* __restrict__ x, const double* __restrict__ xb,
        const double* __restrict__ xa, double* __restrict__ r, int p_begin, int p_end, const AxisTab8 A,
        const MeshArgs M)
{
    using namespace ax8;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* bufX[2] = {smem, smem + BUF_BYTES};
    unsigned char* bufR = smem + 2 * BUF_BYTES;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 3 * BUF_BYTES);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ntile2 = M.N2 / T;
    const int ti1 = blockIdx.x / ntile2, ti2 = blockIdx.x % ntile2;
    const int PC = M.plane_cells;
    const int nsteps = p_end - p_begin;
    if (nsteps <= 0) return;

    auto cell_index = [&](int lp, int i1, int i2) -> long long { return (long long)lp * PC + (long long)i1 * M.N2 + i2; };

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int step) {
        // TMA the 16 blocks of plane p_begin + step into buffer (step & 1): one 16 KB box per tile row
        const int lp = p_begin + step;
        uint64_t* b = &bar[step & 1];
        mbar_expect_tx(b, BUF_BYTES);
#pragma unroll
        for (int c1 = 0; c1 < T; ++c1) {
            const long long cell = cell_index(lp, ti1 * T + c1, ti2 * T);
            tma_load_2d(bufX[step & 1] + c1 * T * CELL_BYTES, &tmx, 0, (int)(cell * (CELL_BYTES / 128)), b);
        }
    };
    if (tid == 0) {
        issue(0);
        if (nsteps > 1) issue(1);
    }

    // ---- d=0 mapping: warp w owns cells 2w, 2w+1 (buffer order c1*4+c2); lanes own lines L, L+32
    const int dcell0 = 2 * warp;
    double prevU[4], prevG[4]; // traces e1.x, d1.x of the lower x0-neighbour for the thread's 4 lines
    {
        // prologue: lower neighbour plane p_begin - 1 (halo x_below if p_begin == 0)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int cb = dcell0 + (q >> 1), L = lane + 32 * (q & 1);
            const int c1 = cb >> 2, c2 = cb & 3;
            const long long inplane = (long long)(ti1 * T + c1) * M.N2 + ti2 * T + c2;
            const double* src = (p_begin == 0) ? xb + inplane * 512 : x + (cell_index(p_begin - 1, 0, 0) + inplane) * 512;
            const double2* s2 = reinterpret_cast<const double2*>(src + 8 * L);
            double v[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                double2 t = __ldg(s2 + k);
                v[2 * k] = t.x;
                v[2 * k + 1] = t.y;
            }
            double xe[4], xo[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) { xe[j] = v[j] + v[7 - j]; xo[j] = v[j] - v[7 - j]; }
            double u0, u1, g0, g1;
            ax8::traces_eo(A, xe, xo, u0, u1, g0, g1);
            prevU[q] = u1;
            prevG[q] = g1;
        }
    }

    for (int s = 0; s < nsteps; ++s) {
        const int lp = p_begin + s;
        const unsigned char* X = bufX[s & 1];
        mbar_wait(&bar[s & 1], (s >> 1) & 1);

        // ================= pass d = 1 (lines along j1; neighbours along i1) =================
        {
            const int j0 = lane & 7, j2 = (lane >> 3) + 4 * (warp & 1), c2 = warp >> 1;
            const int i2 = ti2 * T + c2;
            const int i1L = (ti1 * T - 1 + M.N1) % M.N1, i1R = (ti1 * T + T) % M.N1;
            const double* gl = x + cell_index(lp, i1L, i2) * 512 + j0 + 64 * j2;
            const double* gr = x + cell_index(lp, i1R, i2) * 512 + j0 + 64 * j2;
            double rl[8], rr[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) { rl[j] = __ldg(gl + 8 * j); rr[j] = __ldg(gr + 8 * j); }
            double xe[T][4], xo[T][4], u0[T], u1[T], g0[T], g1[T];
#pragma unroll
            for (int c1 = 0; c1 < T; ++c1) {
                const unsigned char* cb = X + (c1 * T + c2) * CELL_BYTES;
                double v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = *reinterpret_cast<const double*>(cb + swz(8 * (j0 + 8 * j + 64 * j2)));
#pragma unroll
                for (int j = 0; j < 4; ++j) { xe[c1][j] = v[j] + v[7 - j]; xo[c1][j] = v[j] - v[7 - j]; }
                ax8::traces_eo(A, xe[c1], xo[c1], u0[c1], u1[c1], g0[c1], g1[c1]);
            }
            double uLr, gLr, uRr, gRr;
            {
                double a = 0, b = 0, c = 0, d = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    a = fma(A.e0[7 - j], rl[j], a);  // e1.x_L (e1_j = e0_{7-j})
                    b = fma(-A.d0[7 - j], rl[j], b); // d1.x_L (d1_j = -d0_{7-j})
                    c = fma(A.e0[j], rr[j], c);
                    d = fma(A.d0[j], rr[j], d);
                }
                uLr = a; gLr = b; uRr = c; gRr = d;
            }
            const double S = A.w[j0] * A.w[j2] * A.c[1];
#pragma unroll
            for (int c1 = 0; c1 < T; ++c1) {
                const double uL = c1 > 0 ? u1[c1 - 1] : uLr, gL = c1 > 0 ? g1[c1 - 1] : gLr;
                const double uR = c1 < T - 1 ? u0[c1 + 1] : uRr, gR = c1 < T - 1 ? g0[c1 + 1] : gRr;
                double ye[4], yo[4];
                ax8::line_eo(A, xe[c1], xo[c1], uL, gL, uR, gR, ye, yo);
                unsigned char* rb = bufR + (c1 * T + c2) * CELL_BYTES;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    *reinterpret_cast<double*>(rb + swz(8 * (j0 + 8 * i + 64 * j2))) = S * (ye[i] + yo[i]);
                    *reinterpret_cast<double*>(rb + swz(8 * (j0 + 8 * (7 - i) + 64 * j2))) = S * (ye[i] - yo[i]);
                }
            }
        }
        __syncthreads();

        // ================= pass d = 2 (lines along j2; neighbours along i2) =================
        {
            const int j0 = lane & 7, j1 = (lane >> 3) + 4 * (warp & 1), c1 = warp >> 1;
            const int i1 = ti1 * T + c1;
            const int i2L = (ti2 * T - 1 + M.N2) % M.N2, i2R = (ti2 * T + T) % M.N2;
            const double* gl = x + cell_index(lp, i1, i2L) * 512 + j0 + 8 * j1;
            const double* gr = x + cell_index(lp, i1, i2R) * 512 + j0 + 8 * j1;
            double rl[8], rr[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) { rl[j] = __ldg(gl + 64 * j); rr[j] = __ldg(gr + 64 * j); }
            double xe[T][4], xo[T][4], u0[T], u1[T], g0[T], g1[T];
#pragma unroll
            for (int c2 = 0; c2 < T; ++c2) {
                const unsigned char* cb = X + (c1 * T + c2) * CELL_BYTES;
                double v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = *reinterpret_cast<const double*>(cb + swz(8 * (j0 + 8 * j1 + 64 * j)));
#pragma unroll
                for (int j = 0; j < 4; ++j) { xe[c2][j] = v[j] + v[7 - j]; xo[c2][j] = v[j] - v[7 - j]; }
                ax8::traces_eo(A, xe[c2], xo[c2], u0[c2], u1[c2], g0[c2], g1[c2]);
            }
            double uLr, gLr, uRr, gRr;
            {
                double a = 0, b = 0, c = 0, d = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    a = fma(A.e0[7 - j], rl[j], a);
                    b = fma(-A.d0[7 - j], rl[j], b);
                    c = fma(A.e0[j], rr[j], c);
                    d = fma(A.d0[j], rr[j], d);
                }
                uLr = a; gLr = b; uRr = c; gRr = d;
            }
            const double S = A.w[j0] * A.w[j1] * A.c[2];
#pragma unroll
            for (int c2 = 0; c2 < T; ++c2) {
                const double uL = c2 > 0 ? u1[c2 - 1] : uLr, gL = c2 > 0 ? g1[c2 - 1] : gLr;
                const double uR = c2 < T - 1 ? u0[c2 + 1] : uRr, gR = c2 < T - 1 ? g0[c2 + 1] : gRr;
                double ye[4], yo[4];
                ax8::line_eo(A, xe[c2], xo[c2], uL, gL, uR, gR, ye, yo);
                unsigned char* rb = bufR + (c1 * T + c2) * CELL_BYTES;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    double* p0 = reinterpret_cast<double*>(rb + swz(8 * (j0 + 8 * j1 + 64 * i)));
                    double* p1 = reinterpret_cast<double*>(rb + swz(8 * (j0 + 8 * j1 + 64 * (7 - i))));
                    *p0 = fma(S, ye[i] + yo[i], *p0);
                    *p1 = fma(S, ye[i] - yo[i], *p1);
                }
            }
        }
        __syncthreads();

        // ================= pass d = 0 (lines along j0; neighbours along i0: marching) =================
        {
            const bool last = (s == nsteps - 1);
            if (!last) mbar_wait(&bar[(s + 1) & 1], ((s + 1) >> 1) & 1);
            const unsigned char* XN = bufX[(s + 1) & 1];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int cb = dcell0 + (q >> 1), L = lane + 32 * (q & 1);
                const int c1 = cb >> 2, c2 = cb & 3;
                const long long inplane = (long long)(ti1 * T + c1) * M.N2 + ti2 * T + c2;
                // upper neighbour's traces e0.x, d0.x
                double uR = 0.0, gR = 0.0;
                {
                    double v[8];
                    if (!last) {
                        const unsigned char* nb = XN + cb * CELL_BYTES;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            double2 t = *reinterpret_cast<const double2*>(nb + swz(8 * (8 * L + 2 * k)));
                            v[2 * k] = t.x;
                            v[2 * k + 1] = t.y;
                        }
                    } else {
                        const double* src = (p_end == M.L) ? xa + inplane * 512 : x + (cell_index(p_end, 0, 0) + inplane) * 512;
                        const double2* s2 = reinterpret_cast<const double2*>(src + 8 * L);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            double2 t = __ldg(s2 + k);
                            v[2 * k] = t.x;
                            v[2 * k + 1] = t.y;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        uR = fma(A.e0[j], v[j], uR);
                        gR = fma(A.d0[j], v[j], gR);
                    }
                }
                // own line
                double v[8];
                const unsigned char* xcb = X + cb * CELL_BYTES;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    double2 t = *reinterpret_cast<const double2*>(xcb + swz(8 * (8 * L + 2 * k)));
                    v[2 * k] = t.x;
                    v[2 * k + 1] = t.y;
                }
                double xe[4], xo[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) { xe[j] = v[j] + v[7 - j]; xo[j] = v[j] - v[7 - j]; }
                double u0, u1, g0, g1;
                ax8::traces_eo(A, xe, xo, u0, u1, g0, g1);
                double ye[4], yo[4];
                ax8::line_eo(A, xe, xo, prevU[q], prevG[q], uR, gR, ye, yo);
                prevU[q] = u1;
                prevG[q] = g1;
                const double S = A.w[L & 7] * A.w[L >> 3] * A.c[0];
                // partial sums of passes 1, 2
                const unsigned char* rb = bufR + cb * CELL_BYTES;
                double o[8];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    double2 t = *reinterpret_cast<const double2*>(rb + swz(8 * (8 * L + 2 * k)));
                    o[2 * k] = t.x;
                    o[2 * k + 1] = t.y;
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    o[i] = fma(S, ye[i] + yo[i], o[i]);
                    o[7 - i] = fma(S, ye[i] - yo[i], o[7 - i]);
                }
                double2* dst = reinterpret_cast<double2*>(r + (cell_index(lp, 0, 0) + inplane) * 512 + 8 * L);
#pragma unroll
                for (int k = 0; k < 4; ++k) dst[k] = make_double2(o[2 * k], o[2 * k + 1]);
            }
        }
        __syncthreads();
        if (tid == 0 && s + 2 < nsteps) issue(s + 2);
    }
}

} // namespace dg
