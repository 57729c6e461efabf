// Per-cell geometry records (k_geom, once at setup) and the TMA / mbarrier helpers shared by the
// marching-tile kernels.
//
// Geometry (reading R11): for the affine map x = o_T + J_T xi of cell T,
//   G~ = |det J| J^{-1} J^{-T}                       (stage 2 of Alg. assembly)
// and for each upper face d of T (T = T-, T+ = T + e_d):
//   nu = J_-^{-T} e_d, n_F = nu / |nu|, dS = |det J_-| |nu|   (Nanson; face geometry from T-)
//   a- = J_-^{-1} n_F, a+ = J_+^{-1} n_F                      (grad u . n_F = a . grad_hat u on each side)
#pragma once

#include "common.cuh"

namespace dg {


// ----------------------------------------------------------------------------- geometry record
constexpr int GREC = 36; // doubles per cell
// [0..5]   G~ (00, 11, 22, 01, 02, 12)
// [6..11]  J00 J01 J02 J10 J11 J12
// [12 + 8 d .. 19 + 8 d]  upper face d: a-_t1, a+_t1, a-_t2, a+_t2, a-_d, a+_d, dS, 0  (a- = J_-^{-1} n_F,
//                         a+ = J_+^{-1} n_F in (normal, tangential 1, tangential 2) order; 16-B pairs
//                         grouped by the face pass that reads them)

// One thread per cell of the L+2 planes plane_begin-1 .. plane_begin+L (same layout as jac).
__global__ void k_geom(const double* __restrict__ jac, double* __restrict__ geo, long long ncell, int plane_cells,
                       int N1, int N2, int nplanes_total)
{
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const int pl = (int)(c / plane_cells), rem = (int)(c % plane_cells);
    const int i1 = rem / N2, i2 = rem % N2;
    double J[9], Ji[9];
    for (int i = 0; i < 9; ++i) J[i] = jac[c * 9 + i];
    const double adet = fabs(inv3(J, Ji));
    double* g = geo + c * GREC;
    auto gg = [&](int a, int b) { return adet * (Ji[3 * a] * Ji[3 * b] + Ji[3 * a + 1] * Ji[3 * b + 1] + Ji[3 * a + 2] * Ji[3 * b + 2]); };
    g[0] = gg(0, 0); g[1] = gg(1, 1); g[2] = gg(2, 2); g[3] = gg(0, 1); g[4] = gg(0, 2); g[5] = gg(1, 2);
    for (int i = 0; i < 6; ++i) g[6 + i] = J[i];
    for (int d = 0; d < 3; ++d) {
        double* f = g + 12 + 8 * d;
        f[7] = 0.0;
        long long nb;
        if (d == 0) {
            if (pl + 1 >= nplanes_total) { for (int i = 0; i < 7; ++i) f[i] = 0.0; continue; }
            nb = c + plane_cells;
        } else if (d == 1) {
            nb = (long long)pl * plane_cells + (long long)((i1 + 1) % N1) * N2 + i2;
        } else {
            nb = (long long)pl * plane_cells + (long long)i1 * N2 + (i2 + 1) % N2;
        }
        double Jn[9], Jni[9];
        for (int i = 0; i < 9; ++i) Jn[i] = jac[nb * 9 + i];
        inv3(Jn, Jni);
        // nu = J_-^{-T} e_d = row d of J_-^{-1}; n_F = nu/|nu|; dS = |det J_-| |nu| (Nanson)
        const double nu0 = Ji[3 * d], nu1 = Ji[3 * d + 1], nu2 = Ji[3 * d + 2];
        const double nn = sqrt(nu0 * nu0 + nu1 * nu1 + nu2 * nu2);
        const double n0 = nu0 / nn, n1 = nu1 / nn, n2 = nu2 / nn;
        double am[3], ap[3];
        for (int e = 0; e < 3; ++e) {
            am[e] = Ji[3 * e] * n0 + Ji[3 * e + 1] * n1 + Ji[3 * e + 2] * n2;   // a- = J_-^{-1} n_F
            ap[e] = Jni[3 * e] * n0 + Jni[3 * e + 1] * n1 + Jni[3 * e + 2] * n2; // a+ = J_+^{-1} n_F
        }
        const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
        f[0] = am[t1];
        f[1] = ap[t1];
        f[2] = am[t2];
        f[3] = ap[t2];
        f[4] = am[d];
        f[5] = ap[d];
        f[6] = adet * nn; // dS = |det J_-| |J_-^{-T} e_d| (Nanson)
    }
}

namespace tl {

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
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
                     s32(b)),
                 "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(s32(b))
                 : "memory");
}

} // namespace tl
} // namespace dg
