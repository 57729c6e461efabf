// libdg C-ABI (include/dg.h): context setup, kernel dispatch, slab / host-pipelined apply.
#include "../../include/dg.h"
#include "common.cuh"
#include "kernel_axis8.cuh"
#include "kernel_cell.cuh"
#include "kernel_gen.cuh"
#include "kernel_line.cuh"
#include "kernel_quad.cuh"
#include "kernel_stokes.cuh"
#include "tables.h"

#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h> // types only: the library is dlopen'ed (a process may already hold torch's libnccl.so.2)

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

// k_axis8 variants (DG_AX8_TILE=<T1>x<T2>m<minBlocks>; default = the first): ID, T1, T2, threads, min CTAs/SM
#define AX8_VARIANTS(X) \
    X(0, 2, 4, 256, 2)  \
    X(1, 2, 4, 256, 1)  \
    X(2, 4, 4, 512, 1)  \
    X(3, 2, 2, 256, 3)  \
    X(4, 2, 2, 256, 2)  \
    X(5, 4, 2, 256, 2)

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail(e_ == cudaErrorMemoryAllocation ? DG_ERR_OOM : DG_ERR_CUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                          \
    } while (0)

using LaunchFn = cudaError_t (*)(const void* tab, const dg::MeshArgs& M, const double* x, const double* xb,
                                 const double* xa, double* r, long long c0, long long c1, cudaStream_t st,
                                 const double* geo);

template <int N, bool AFF, bool COEF>
cudaError_t launch_cell(const void* tab, const dg::MeshArgs& M, const double* x, const double* xb, const double* xa,
                        double* r, long long c0, long long c1, cudaStream_t st, const double*)
{
    constexpr int CPB = dg::CellCfg<N>::CPB;
    const long long ncell = c1 - c0;
    if (ncell <= 0) return cudaSuccess;
    const long long grid = (ncell + CPB - 1) / CPB;
    dg::k_cell_general<N, AFF, COEF><<<(unsigned)grid, dg::CellCfg<N>::THREADS, 0, st>>>(
        x, xb, xa, r, c0, c1, *static_cast<const dg::Tab<N>*>(tab), M);
    return cudaGetLastError();
}

template <int N>
LaunchFn pick_cell(bool aff, bool coef)
{
    if (aff) return coef ? launch_cell<N, true, true> : launch_cell<N, true, false>;
    return coef ? launch_cell<N, false, true> : launch_cell<N, false, false>;
}

LaunchFn pick(int n, bool aff, bool coef)
{
    switch (n) {
    case 2: return pick_cell<2>(aff, coef);
    case 3: return pick_cell<3>(aff, coef);
    case 4: return pick_cell<4>(aff, coef);
    case 5: return pick_cell<5>(aff, coef);
    case 6: return pick_cell<6>(aff, coef);
    case 7: return pick_cell<7>(aff, coef);
    case 8: return pick_cell<8>(aff, coef);
    default: return nullptr;
    }
}

// ---- marching-tile general kernel v2 (k_gen): tile per degree (T1, T2 even for odd n: 16-B bulk rows)
template <int N> struct GenShape;
template <> struct GenShape<2> { static constexpr int T1 = 4, T2 = 4, MINB = 4; };
template <> struct GenShape<3> { static constexpr int T1 = 2, T2 = 4, MINB = 4; };

// (T1, T2, min CTAs/SM) for n = 4, 5, 6; overridable at build time for tuning sweeps
#ifndef GEN4_T1
#define GEN4_T1 2
#define GEN4_T2 4
#define GEN4_MB 4
#endif
#ifndef GEN5_T1
#define GEN5_T1 2
#define GEN5_T2 4
#define GEN5_MB 2
#endif
#ifndef GEN6_T1
#define GEN6_T1 2
#define GEN6_T2 2
#define GEN6_MB 2
#endif
template <int a, int b, int c> struct GenS { static constexpr int T1 = a, T2 = b, MINB = c; };
template <> struct GenShape<4> : GenS<GEN4_T1, GEN4_T2, GEN4_MB> {};
template <> struct GenShape<5> : GenS<GEN5_T1, GEN5_T2, GEN5_MB> {};
template <> struct GenShape<6> : GenS<GEN6_T1, GEN6_T2, GEN6_MB> {};
template <> struct GenShape<7> { static constexpr int T1 = 2, T2 = 2, MINB = 1; };
template <> struct GenShape<8> { static constexpr int T1 = 2, T2 = 2, MINB = 1; };

using GenFn = cudaError_t (*)(const void* eot, const dg::MeshArgs& M, const double* x, const double* xb, const double* xa,
                              double* r, int p0, int p1, int chunk, int halo_tr, cudaStream_t st, const double* geo,
                              const double* ctab, const double* cface);

template <int N, bool AFF, bool COEF>
cudaError_t launch_gen(const void* eot, const dg::MeshArgs& M, const double* x, const double* xb, const double* xa,
                       double* r, int p0, int p1, int chunk, int halo_tr, cudaStream_t st, const double* geo,
                       const double* ctab, const double* cface)
{
    constexpr int T1 = GenShape<N>::T1, T2 = GenShape<N>::T2, MB = GenShape<N>::MINB;
    using Y = dg::gn::Lay<N, AFF, COEF, T1, T2>;
    if (p1 <= p0) return cudaSuccess;
    const int np = p1 - p0;
    const int CL = chunk > 0 && chunk < np ? chunk : np;
    const unsigned grid = (unsigned)((M.N1 / T1) * (M.N2 / T2) * ((np + CL - 1) / CL));
    dg::k_gen<N, AFF, COEF, T1, T2, MB><<<grid, Y::NT, Y::BYTES, st>>>(
        x, xb, xa, r, p0, p1, CL, halo_tr, *static_cast<const dg::EOTab<N>*>(eot), M, geo, ctab, cface);
    return cudaGetLastError();
}

template <int N, bool AFF, bool COEF>
cudaError_t attr_gen()
{
    constexpr int T1 = GenShape<N>::T1, T2 = GenShape<N>::T2, MB = GenShape<N>::MINB;
    return cudaFuncSetAttribute(dg::k_gen<N, AFF, COEF, T1, T2, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                dg::gn::Lay<N, AFF, COEF, T1, T2>::BYTES);
}

struct GenInfo {
    GenFn fn;
    int T1, T2, smem;
    cudaError_t (*attr)();
};

template <int N>
GenInfo gen_info(bool aff, bool coef)
{
    GenInfo g;
    g.T1 = GenShape<N>::T1;
    g.T2 = GenShape<N>::T2;
    if (aff) {
        g.fn = coef ? launch_gen<N, true, true> : launch_gen<N, true, false>;
        g.attr = coef ? attr_gen<N, true, true> : attr_gen<N, true, false>;
        g.smem = coef ? dg::gn::Lay<N, true, true, GenShape<N>::T1, GenShape<N>::T2>::BYTES
                      : dg::gn::Lay<N, true, false, GenShape<N>::T1, GenShape<N>::T2>::BYTES;
    } else {
        g.fn = coef ? launch_gen<N, false, true> : launch_gen<N, false, false>;
        g.attr = coef ? attr_gen<N, false, true> : attr_gen<N, false, false>;
        g.smem = coef ? dg::gn::Lay<N, false, true, GenShape<N>::T1, GenShape<N>::T2>::BYTES
                      : dg::gn::Lay<N, false, false, GenShape<N>::T1, GenShape<N>::T2>::BYTES;
    }
    return g;
}

GenInfo pick_gen(int n, bool aff, bool coef)
{
    switch (n) {
    case 2: return gen_info<2>(aff, coef);
    case 3: return gen_info<3>(aff, coef);
    case 4: return gen_info<4>(aff, coef);
    case 5: return gen_info<5>(aff, coef);
    case 6: return gen_info<6>(aff, coef);
    case 7: return gen_info<7>(aff, coef);
    default: return gen_info<8>(aff, coef);
    }
}

// even/odd tables (kernel_gen.cuh, EOTab): D is centro-antisymmetric and e1, d1 are the mirrored
// e0, -d0 on the symmetric Gauss nodes; the halves fold the factor 1/2 in.
template <int N>
void fill_eotab(const dg::HostTables& Ht, double P, const double h[3], void* out)
{
    dg::EOTab<N>* E = static_cast<dg::EOTab<N>*>(out);
    constexpr int H = N / 2;
    auto D = [&](int q, int j) { return Ht.D[q * N + j]; };
    for (int q = 0; q < H; ++q) {
        for (int j = 0; j < H; ++j) {
            E->Fm[q][j] = 0.5 * (D(q, j) - D(q, N - 1 - j));
            E->Fp[q][j] = 0.5 * (D(q, j) + D(q, N - 1 - j));
        }
        if (N & 1) {
            E->Fp[q][H] = D(q, H);
            E->Fmid[q] = D(H, q);
        } else {
            E->Fmid[q] = 0.0;
        }
    }
    for (int j = 0; j < H; ++j) {
        E->Es[j] = 0.5 * (Ht.e0[j] + Ht.e0[N - 1 - j]);
        E->Ea[j] = 0.5 * (Ht.e0[j] - Ht.e0[N - 1 - j]);
        E->Ds[j] = 0.5 * (Ht.d0[j] + Ht.d0[N - 1 - j]);
        E->Da[j] = 0.5 * (Ht.d0[j] - Ht.d0[N - 1 - j]);
    }
    if (N & 1) {
        E->Es[H] = Ht.e0[H];
        E->Ds[H] = Ht.d0[H];
    }
    for (int i = 0; i < N * N; ++i) E->D[i] = Ht.D[i];
    for (int i = 0; i < N; ++i) {
        E->w[i] = Ht.w[i];
        E->xi[i] = Ht.xi[i];
    }
    // line operator B^ (kernel_axis8.cuh) and its neighbour couplings aL = -d0/2 - P e0, bL = e0/2
    // (aR_i = aL_{n-1-i}, bR_i = -bL_{n-1-i} by the mirror symmetry)
    double B[N][N], aL[N], bL[N];
    for (int i = 0; i < N; ++i) {
        for (int j = 0; j < N; ++j) {
            double s = 0.0;
            for (int q = 0; q < N; ++q) s += Ht.D[q * N + i] * Ht.w[q] * Ht.D[q * N + j];
            s += 0.5 * (Ht.e0[i] * Ht.d0[j] + Ht.d0[i] * Ht.e0[j] - Ht.e1[i] * Ht.d1[j] - Ht.d1[i] * Ht.e1[j]);
            s += P * (Ht.e0[i] * Ht.e0[j] + Ht.e1[i] * Ht.e1[j]);
            B[i][j] = s;
        }
        aL[i] = -0.5 * Ht.d0[i] - P * Ht.e0[i];
        bL[i] = 0.5 * Ht.e0[i];
    }
    for (int i = 0; i < H; ++i) {
        for (int j = 0; j < H; ++j) {
            E->Lp[i][j] = 0.5 * (B[i][j] + B[i][N - 1 - j]);
            E->Lm[i][j] = 0.5 * (B[i][j] - B[i][N - 1 - j]);
        }
        if (N & 1) E->Lp[i][H] = B[i][H];
        E->Ae[i] = 0.5 * (aL[i] + aL[N - 1 - i]);
        E->Be[i] = 0.5 * (bL[i] + bL[N - 1 - i]);
        E->Ao[i] = 0.5 * (aL[i] - aL[N - 1 - i]);
        E->Bo[i] = 0.5 * (bL[i] - bL[N - 1 - i]);
    }
    if (N & 1) {
        for (int j = 0; j < H; ++j) E->Lmid[j] = B[H][j];
        E->Lmid[H] = B[H][H];
        E->Ae[H] = aL[H];
        E->Be[H] = bL[H];
    }
    E->Sc[0] = h[1] * h[2] / h[0];
    E->Sc[1] = h[0] * h[2] / h[1];
    E->Sc[2] = h[0] * h[1] / h[2];
}

// ---- general quadrature (M = n + MQ Gauss points per direction, MQ = 1 or 2; MQ = 0 with the Gauss-Lobatto basis;
//      SURVEY §8(f2)): k_quad
template <int N, bool AFF, bool COEF, int PR = 0, int MQ = 1>
cudaError_t launch_quad(const void* qt, const dg::MeshArgs& M, const double* x, const double* xb, const double* xa,
                        double* r, long long c0, long long c1, cudaStream_t st, const double* u0)
{
    if (c1 <= c0) return cudaSuccess;
    using L = dg::qd::QLay<N, N + MQ, PR == 3>;
    const long long grid = (c1 - c0 + L::CPB - 1) / L::CPB;
    dg::k_quad<N, N + MQ, AFF, COEF, PR><<<(unsigned)grid, L::NT, L::BYTES, st>>>(
        x, xb, xa, r, c0, c1, *static_cast<const dg::QTab<N, N + MQ>*>(qt), M, u0);
    return cudaGetLastError();
}
template <int N, bool AFF, bool COEF, int PR = 0, int MQ = 1>
cudaError_t attr_quad()
{
    if (dg::qd::QLay<N, N + MQ, PR == 3>::BYTES > 227 * 1024) return cudaErrorInvalidValue; // does not fit an SM
    return cudaFuncSetAttribute(dg::k_quad<N, N + MQ, AFF, COEF, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                dg::qd::QLay<N, N + MQ, PR == 3>::BYTES);
}
// pr: the problem mode of k_quad (0 periodic, 1 diffusion-reaction, 2 its nonlinear variant, 3 the Jacobian
// action of the nonlinear variant); mq = m - n (2: the periodic problem only)
template <int N>
LaunchFn pick_quad_n(bool aff, bool coef, cudaError_t* err, int pr = 0, int mq = 1)
{
    if (pr == 1) { *err = attr_quad<N, false, false, 1>(); return launch_quad<N, false, false, 1>; }
    if (pr == 2) { *err = attr_quad<N, false, false, 2>(); return launch_quad<N, false, false, 2>; }
    if (pr == 3) { *err = attr_quad<N, false, false, 3>(); return launch_quad<N, false, false, 3>; }
    if (mq == 0) { // the Gauss-Lobatto basis with m = n Gauss points (A != I)
        if (aff) {
            *err = coef ? attr_quad<N, true, true, 0, 0>() : attr_quad<N, true, false, 0, 0>();
            return coef ? launch_quad<N, true, true, 0, 0> : launch_quad<N, true, false, 0, 0>;
        }
        *err = coef ? attr_quad<N, false, true, 0, 0>() : attr_quad<N, false, false, 0, 0>();
        return coef ? launch_quad<N, false, true, 0, 0> : launch_quad<N, false, false, 0, 0>;
    }
    if constexpr (N <= 7) {
        if (mq == 2) {
            if (aff) {
                *err = coef ? attr_quad<N, true, true, 0, 2>() : attr_quad<N, true, false, 0, 2>();
                return coef ? launch_quad<N, true, true, 0, 2> : launch_quad<N, true, false, 0, 2>;
            }
            *err = coef ? attr_quad<N, false, true, 0, 2>() : attr_quad<N, false, false, 0, 2>();
            return coef ? launch_quad<N, false, true, 0, 2> : launch_quad<N, false, false, 0, 2>;
        }
    }
    if (aff) {
        *err = coef ? attr_quad<N, true, true>() : attr_quad<N, true, false>();
        return coef ? launch_quad<N, true, true> : launch_quad<N, true, false>;
    }
    *err = coef ? attr_quad<N, false, true>() : attr_quad<N, false, false>();
    return coef ? launch_quad<N, false, true> : launch_quad<N, false, false>;
}
LaunchFn pick_quad(int n, bool aff, bool coef, cudaError_t* err, int pr = 0, int mq = 1)
{
    switch (n) {
    case 2: return pick_quad_n<2>(aff, coef, err, pr, mq);
    case 3: return pick_quad_n<3>(aff, coef, err, pr, mq);
    case 4: return pick_quad_n<4>(aff, coef, err, pr, mq);
    case 5: return pick_quad_n<5>(aff, coef, err, pr, mq);
    case 6: return pick_quad_n<6>(aff, coef, err, pr, mq);
    case 7: return pick_quad_n<7>(aff, coef, err, pr, mq);
    default: return pick_quad_n<8>(aff, coef, err, pr, mq);
    }
}
// ---- the paper's Stokes problem: k_stokes, one cell per CTA
template <int N>
cudaError_t launch_stokes(const void* st_, const dg::MeshArgs& M, const double* x, const double* xb, const double* xa,
                          double* r, long long c0, long long c1, cudaStream_t st, const double*)
{
    if (c1 <= c0) return cudaSuccess;
    using L = dg::sk::SLay<N>;
    dg::k_stokes<N><<<(unsigned)(c1 - c0), L::NT, L::BYTES, st>>>(x, xb, xa, r, c0, c1,
                                                                   *static_cast<const dg::STab<N>*>(st_), M);
    return cudaGetLastError();
}
template <int N>
LaunchFn pick_stokes_n(cudaError_t* err)
{
    *err = cudaFuncSetAttribute(dg::k_stokes<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, dg::sk::SLay<N>::BYTES);
    return launch_stokes<N>;
}
LaunchFn pick_stokes(int n, cudaError_t* err)
{
    switch (n) {
    case 2: return pick_stokes_n<2>(err);
    case 3: return pick_stokes_n<3>(err);
    case 4: return pick_stokes_n<4>(err);
    case 5: return pick_stokes_n<5>(err);
    case 6: return pick_stokes_n<6>(err);
    case 7: return pick_stokes_n<7>(err);
    default: return pick_stokes_n<8>(err);
    }
}
// velocity tables (collocated: D at the n Gauss points) and the pressure basis (n-1 Gauss nodes) at the
// velocity nodes (long double product formulas, as fill_qtab)
// even/odd form of an LO x LIN row-major table (kernel_quad.cuh, EOMat); tr: read the table transposed (T[j][q])
template <int LO, int LIN, int S>
void fill_eomat(const double* T, bool tr, dg::EOMat<LO, LIN, S>* E)
{
    constexpr int HO = LO / 2, HI = LIN / 2;
    auto t = [&](int q, int j) { return tr ? T[j * LO + q] : T[q * LIN + j]; };
    for (int q = 0; q < HO; ++q) {
        for (int j = 0; j < HI; ++j) {
            E->Pe[q][j] = 0.5 * (t(q, j) + t(q, LIN - 1 - j));
            E->Po[q][j] = 0.5 * (t(q, j) - t(q, LIN - 1 - j));
        }
        if (LIN & 1) E->Pe[q][HI] = t(q, HI);
    }
    if (LO & 1) {
        for (int j = 0; j < HI; ++j) E->Pm[j] = t(HO, j);
        if (LIN & 1) E->Pm[HI] = S > 0 ? t(HO, HI) : 0.0;
    }
}

template <int N>
void fill_stab(const dg::HostTables& H, const dg::HostTables& Hp, void* out)
{
    constexpr int NP = N - 1;
    dg::STab<N>* S = static_cast<dg::STab<N>*>(out);
    for (int i = 0; i < N * N; ++i) S->D[i] = H.D[i];
    for (int q = 0; q < N; ++q) {
        const long double s = H.xi[q];
        for (int j = 0; j < NP; ++j) {
            long double v = 1.0L;
            for (int a = 0; a < NP; ++a)
                if (a != j) v *= (s - Hp.xi[a]) / ((long double)Hp.xi[j] - Hp.xi[a]);
            S->AP[q * NP + j] = (double)v;
        }
        S->w[q] = H.w[q];
        S->xi[q] = H.xi[q];
        S->e0[q] = H.e0[q];
        S->e1[q] = H.e1[q];
        S->d0[q] = H.d0[q];
        S->d1[q] = H.d1[q];
    }
    for (int j = 0; j < NP; ++j) {
        S->ep0[j] = Hp.e0[j];
        S->ep1[j] = Hp.e1[j];
    }
    fill_eomat(S->D, false, &S->eD);
    fill_eomat(S->D, true, &S->eDt);
    fill_eomat(S->AP, false, &S->eAP);
    fill_eomat(S->AP, true, &S->eAPt);
}

// interpolation / derivative of the n-node Lagrange basis at the m = n + MQ Gauss points (long double
// product formulas, no division by (s - x_a): robust when a quadrature point is close to a node)
template <int N, int MQ = 1>
void fill_qtab(const dg::HostTables& Hn, const dg::HostTables& Hm, void* out)
{
    constexpr int M = N + MQ;
    dg::QTab<N, M>* Q = static_cast<dg::QTab<N, M>*>(out);
    for (int q = 0; q < M; ++q) {
        const long double s = Hm.xi[q];
        for (int j = 0; j < N; ++j) {
            long double v = 1.0L, dv = 0.0L;
            for (int a = 0; a < N; ++a) {
                if (a == j) continue;
                const long double den = (long double)Hn.xi[j] - Hn.xi[a];
                dv = dv * ((s - Hn.xi[a]) / den) + v / den; // product rule, accumulated
                v *= (s - Hn.xi[a]) / den;
            }
            Q->A[q * N + j] = (double)v;
            Q->Dq[q * N + j] = (double)dv;
        }
        Q->wq[q] = Hm.w[q];
        Q->xq[q] = Hm.xi[q];
    }
    for (int j = 0; j < N; ++j) {
        Q->e0[j] = Hn.e0[j];
        Q->e1[j] = Hn.e1[j];
        Q->d0[j] = Hn.d0[j];
        Q->d1[j] = Hn.d1[j];
    }
    fill_eomat(Q->A, false, &Q->eA);
    fill_eomat(Q->Dq, false, &Q->eD);
    fill_eomat(Q->A, true, &Q->eAt);
    fill_eomat(Q->Dq, true, &Q->eDt);
}

template <int N>
void fill_tab(const dg::HostTables& H, void* out)
{
    dg::Tab<N>* T = static_cast<dg::Tab<N>*>(out);
    for (int i = 0; i < N * N; ++i) T->D[i] = H.D[i];
    for (int i = 0; i < N; ++i) {
        T->w[i] = H.w[i];
        T->xi[i] = H.xi[i];
        T->e0[i] = H.e0[i];
        T->e1[i] = H.e1[i];
        T->d0[i] = H.d0[i];
        T->d1[i] = H.d1[i];
    }
}

// B^ = D^T W D + 1/2 (e0 d0^T + d0 e0^T - e1 d1^T - d1 e1^T) + P (e0 e0^T + e1 e1^T)  (see kernel_axis8.cuh)
void build_axis8(const dg::HostTables& H, double P, const double h[3], dg::AxisTab8* A)
{
    // K = D^T W D (the volume stiffness of one line) in even/odd halves, symmetrised (the kernel reads the upper
    // triangle); the face terms of B^ and the neighbour couplings are formed in the kernel from the trace vectors
    const int n = 8, m = 4;
    double K[8][8];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int q = 0; q < n; ++q) s += H.D[q * n + i] * H.w[q] * H.D[q * n + j];
            K[i][j] = s;
        }
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
            const double ke = 0.5 * (K[i][j] + K[i][n - 1 - j]), ke_t = 0.5 * (K[j][i] + K[j][n - 1 - i]);
            const double ko = 0.5 * (K[i][j] - K[i][n - 1 - j]), ko_t = 0.5 * (K[j][i] - K[j][n - 1 - i]);
            A->Ke[i][j] = 0.5 * (ke + ke_t);
            A->Ko[i][j] = 0.5 * (ko + ko_t);
        }
    for (int i = 0; i < m; ++i) {
        A->te[i] = 0.5 * (H.e0[i] + H.e0[n - 1 - i]);
        A->to[i] = 0.5 * (H.e0[i] - H.e0[n - 1 - i]);
        A->qe[i] = 0.5 * (H.d0[i] + H.d0[n - 1 - i]);
        A->qo[i] = 0.5 * (H.d0[i] - H.d0[n - 1 - i]);
    }
    A->P = P;
    for (int i = 0; i < n; ++i) A->w[i] = H.w[i];
    A->c[0] = h[1] * h[2] / h[0];
    A->c[1] = h[0] * h[2] / h[1];
    A->c[2] = h[0] * h[1] / h[2];
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

} // namespace

struct dg_ctx {
    dg_mesh mesh;
    int k, n;
    int device;
    cudaStream_t stream;
    dg::MeshArgs M;
    alignas(16) unsigned char tab[sizeof(dg::Tab<dg::kMaxN>)];
    LaunchFn launch;
    LaunchFn launch_jac; // DG_PROBLEM_NLREAC: the Jacobian action (k_quad mode 3)
    const char* kname;
    // axis-aligned n = 8 fast path (k_axis8)
    bool ax8;
    bool gen;
    bool line; // k_line: axis-aligned c = 1, L2-resident vectors
    GenInfo ginfo;
    int m;     // Gauss points per direction
    bool quad; // m = n + 1: k_quad
    alignas(16) unsigned char qtab[sizeof(dg::QTab<dg::kMaxN, dg::kMaxN + 1>)];
    bool stokes; // DG_PROBLEM_STOKES: k_stokes
    alignas(16) unsigned char stab[sizeof(dg::STab<8>)];
    int gen_chunk;
    alignas(16) unsigned char eotab[sizeof(dg::EOTab<dg::kMaxN>)];
    int ax8_tile, ax8_T1, ax8_T2, ax8_chunk;
    dg::AxisTab8 atab;
    CUtensorMap tmap;
    const double* tmap_ptr;
    long long* dbg; // DG_TRACE: device buffer of per-phase clock64 stamps (k_axis8)
    double* d_jac;
    double* d_geo;  // k_gen geometry records (affine)
    double* d_ctab;  // k_gen c(x) factor tables (coefficient c(x))
    double* d_cface; // k_gen c(x) at the upper-face points of every cell
    // host-pipeline state (dg_apply_host)
    double* hx_d;
    double* hr_d;
    cudaStream_t s_h2d, s_d2h, s_cmp;
    cudaEvent_t ev_in[32], ev_cmp[32]; // created with the streams, destroyed by dg_destroy (no per-call events)
    // collective form (dg_setup_dist / dg_apply_dist): library-owned NCCL communicator and halo state
    ncclComm_t comm;
    int rank, nranks;
    bool dist_tr;                  // trace halos (k_gen, k_axis8, k_line) or full boundary planes
    int64_t halo_n;                // doubles per halo message
    double *d_hb, *d_ha, *d_tlo, *d_thi;
    cudaStream_t s_comm;
    cudaEvent_t ev_x, ev_halo;
    int64_t plane_dofs, local_dofs;
};

static cudaError_t launch_planes(dg_ctx* c, const double* x, const double* xb, const double* xa, double* r, int p0,
                                 int p1, cudaStream_t st, const double* u0 = nullptr, int halo_tr = 0)
{
    if (p1 <= p0) return cudaSuccess;
    if (u0) { // the Jacobian action of the nonlinear variant (dg_apply_jacobian*)
        const long long pcq = c->M.plane_cells;
        return c->launch_jac(c->qtab, c->M, x, xb, xa, r, (long long)p0 * pcq, (long long)p1 * pcq, st, u0);
    }
    if (c->ax8) {
        if (c->tmap_ptr != x) {
            cuuint64_t dims[2] = {16, (cuuint64_t)(c->local_dofs / 16)};
            cuuint64_t strides[1] = {128};
            cuuint32_t box[2] = {16, (cuuint32_t)(c->ax8_T2 * 32)};
            cuuint32_t estr[2] = {1, 1};
            CUresult rc = get_encode()(&c->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)x, dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (rc != CUDA_SUCCESS) return cudaErrorInvalidValue;
            c->tmap_ptr = x;
        }
        const int ntiles = (c->M.N1 / c->ax8_T1) * (c->M.N2 / c->ax8_T2);
        const int np = p1 - p0;
        const int CL = c->ax8_chunk > 0 ? (c->ax8_chunk < np ? c->ax8_chunk : np) : np;
        const unsigned grid = (unsigned)(ntiles * ((np + CL - 1) / CL));
        switch (c->ax8_tile) {
#define AX8_LAUNCH(ID, T1, T2, NT, MB)                                                                               \
    case ID:                                                                                                         \
        dg::k_axis8<T1, T2, NT, MB><<<grid, NT, dg::ax8::Cfg<T1, T2, NT>::SMEM_BYTES, st>>>(c->tmap, x, xb, xa, r, p0, p1, \
                                                                                          CL, halo_tr, c->atab, c->M, c->dbg); \
        break;
            AX8_VARIANTS(AX8_LAUNCH)
#undef AX8_LAUNCH
        }
        return cudaGetLastError();
    }
    if (c->stokes) {
        const long long pcs = c->M.plane_cells;
        return c->launch(c->stab, c->M, x, xb, xa, r, (long long)p0 * pcs, (long long)p1 * pcs, st, nullptr);
    }
    if (c->quad) {
        const long long pcq = c->M.plane_cells;
        return c->launch(c->qtab, c->M, x, xb, xa, r, (long long)p0 * pcq, (long long)p1 * pcq, st, nullptr);
    }
    if (c->line) {
        const long long ncell = (long long)(p1 - p0) * c->M.plane_cells;
        switch (c->n) {
#define LINE_CASE(NN)                                                                                                  \
    case NN: {                                                                                                         \
        const unsigned grid = (unsigned)((ncell + dg::LineCfg<NN>::CPB - 1) / dg::LineCfg<NN>::CPB);                   \
        dg::k_line<NN><<<grid, dg::LineCfg<NN>::NT, 0, st>>>(x, xb, xa, r, p0, p1, halo_tr,                            \
                                                            *reinterpret_cast<const dg::EOTab<NN>*>(c->eotab), c->M); \
        break;                                                                                                         \
    }
            LINE_CASE(2) LINE_CASE(3) LINE_CASE(4) LINE_CASE(5) LINE_CASE(6) LINE_CASE(7) LINE_CASE(8)
#undef LINE_CASE
        }
        return cudaGetLastError();
    }
    if (c->gen)
        return c->ginfo.fn(c->eotab, c->M, x, xb, xa, r, p0, p1, c->gen_chunk, halo_tr, st, c->d_geo, c->d_ctab, c->d_cface);
    const long long pc = c->M.plane_cells;
    return c->launch(c->tab, c->M, x, xb, xa, r, (long long)p0 * pc, (long long)p1 * pc, st, nullptr);
}

namespace {
template <int N>
int host_line_ops(const dg::HostTables& Ht, double P, const double* x, const double* nb, double* out)
{
    alignas(16) unsigned char buf[sizeof(dg::EOTab<N>)];
    const double h[3] = {1.0, 1.0, 1.0};
    fill_eotab<N>(Ht, P, h, buf);
    const dg::EOTab<N>& E = *reinterpret_cast<const dg::EOTab<N>*>(buf);
    double v[N], xe[dg::EOTab<N>::HE], xo[dg::EOTab<N>::H], y[N];
    for (int j = 0; j < N; ++j) v[j] = x[j];
    dg::gn::split<N>(v, xe, xo);
    dg::gn::sweep<N, false, false>(E, xe, xo, y);
    for (int j = 0; j < N; ++j) out[j] = y[j];
    dg::gn::sweep<N, true, true>(E, xe, xo, y, nb[0], nb[1], nb[2], nb[3]);
    for (int j = 0; j < N; ++j) out[N + j] = y[j];
    dg::gn::lineop<N>(E, xe, xo, y, nb[0], nb[1], nb[2], nb[3]);
    for (int j = 0; j < N; ++j) out[2 * N + j] = y[j];
    dg::gn::traces<N>(E, xe, xo, out[3 * N], out[3 * N + 1], out[3 * N + 2], out[3 * N + 3]);
    return DG_OK;
}
} // namespace

// ---- NCCL, loaded at run time (dlopen of libnccl.so.2: the process's already-loaded instance, e.g. torch's, or the
// system one); only the collective entry points need it
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
};
static const NcclApi* nccl_api()
{
    static NcclApi api;
    static int state = 0; // 0 untried, 1 ok, -1 unavailable
    if (state == 0) {
        state = -1;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (h) {
            api.GetUniqueId = (ncclResult_t(*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
            api.CommInitRank = (ncclResult_t(*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(h, "ncclCommInitRank");
            api.CommDestroy = (ncclResult_t(*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
            api.Send = (ncclResult_t(*)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclSend");
            api.Recv = (ncclResult_t(*)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclRecv");
            api.GroupStart = (ncclResult_t(*)())dlsym(h, "ncclGroupStart");
            api.GroupEnd = (ncclResult_t(*)())dlsym(h, "ncclGroupEnd");
            api.GetErrorString = (const char* (*)(ncclResult_t))dlsym(h, "ncclGetErrorString");
            if (api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
                api.GroupEnd && api.GetErrorString)
                state = 1;
        }
    }
    return state == 1 ? &api : nullptr;
}

static void dist_release(dg_ctx* c)
{
    if (c->comm) {
        if (const NcclApi* N = nccl_api()) N->CommDestroy(c->comm);
        c->comm = nullptr;
    }
    if (c->d_hb) cudaFree(c->d_hb);
    if (c->d_ha) cudaFree(c->d_ha);
    if (c->d_tlo) cudaFree(c->d_tlo);
    if (c->d_thi) cudaFree(c->d_thi);
    if (c->s_comm) cudaStreamDestroy(c->s_comm);
    if (c->ev_x) cudaEventDestroy(c->ev_x);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    c->d_hb = c->d_ha = c->d_tlo = c->d_thi = nullptr;
    c->s_comm = nullptr;
    c->ev_x = c->ev_halo = nullptr;
}

// release a partially built context and report the failure (dg_setup never leaks on an error path)
static int setup_fail(dg_ctx* c, int code, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    dg_destroy(c);
    g_err = buf;
    return code;
}

extern "C" {

const char* dg_last_error(void) { return g_err.c_str(); }

int dg_setup(const dg_mesh* mesh, int k, int quad, dg_ctx** out)
{
    g_err.clear();
    if (!mesh || !out) return fail(DG_ERR_INVALID, "dg_setup: NULL argument");
    *out = nullptr;
    if (k < 1 || k > 7) return fail(DG_ERR_INVALID, "dg_setup: k=%d outside [1,7]", k);
    if (quad != k + 1 && quad != k + 2 && !(quad == k + 3 && k <= 6 && mesh->problem == DG_PROBLEM_PERIODIC))
        return fail(DG_ERR_UNSUPPORTED,
                    "dg_setup: quad=%d (supported: k+1 collocation, k+2 overintegration, k+3 for the periodic problem "
                    "with k <= 6)", quad);
    for (int d = 0; d < 3; ++d)
        if (mesh->N[d] < 2) return fail(DG_ERR_INVALID, "dg_setup: N[%d]=%d < 2", d, mesh->N[d]);
    if (mesh->plane_begin < 0 || mesh->plane_begin >= mesh->N[0] || mesh->nplanes < 1 || mesh->nplanes > mesh->N[0])
        return fail(DG_ERR_INVALID, "dg_setup: bad slab [%d, +%d) for N0=%d", mesh->plane_begin, mesh->nplanes,
                    mesh->N[0]);
    if (mesh->geom_kind != DG_GEOM_AXIS && mesh->geom_kind != DG_GEOM_AFFINE)
        return fail(DG_ERR_INVALID, "dg_setup: geom_kind=%d", mesh->geom_kind);
    if ((mesh->geom_kind == DG_GEOM_AFFINE) != (mesh->jac != nullptr))
        return fail(DG_ERR_INVALID, "dg_setup: jac must be given iff geom_kind == DG_GEOM_AFFINE");
    if (mesh->coeff_kind != DG_COEFF_ONE && mesh->coeff_kind != DG_COEFF_SINCOS)
        return fail(DG_ERR_INVALID, "dg_setup: coeff_kind=%d", mesh->coeff_kind);
    if (!(mesh->penalty_scale > 0.0)) return fail(DG_ERR_INVALID, "dg_setup: penalty_scale must be > 0");
    if (mesh->problem != DG_PROBLEM_PERIODIC && mesh->problem != DG_PROBLEM_DIFFREAC && mesh->problem != DG_PROBLEM_NLREAC &&
        mesh->problem != DG_PROBLEM_STOKES)
        return fail(DG_ERR_INVALID, "dg_setup: problem=%d", mesh->problem);
    if (mesh->basis != DG_BASIS_GAUSS && mesh->basis != DG_BASIS_LOBATTO && mesh->basis != DG_BASIS_EQUIDISTANT)
        return fail(DG_ERR_INVALID, "dg_setup: basis=%d", mesh->basis);
    if (mesh->basis != DG_BASIS_GAUSS && mesh->problem != DG_PROBLEM_PERIODIC)
        return fail(DG_ERR_UNSUPPORTED, "dg_setup: the non-Gauss bases are built for DG_PROBLEM_PERIODIC only");
    if (mesh->problem == DG_PROBLEM_STOKES &&
        (mesh->geom_kind != DG_GEOM_AXIS || mesh->coeff_kind != DG_COEFF_ONE || quad != k + 1))
        return fail(DG_ERR_UNSUPPORTED, "dg_setup: the Stokes problem needs DG_GEOM_AXIS, DG_COEFF_ONE and quad = k+1");
    const bool dr = mesh->problem == DG_PROBLEM_DIFFREAC || mesh->problem == DG_PROBLEM_NLREAC;
    if (dr && (mesh->geom_kind != DG_GEOM_AXIS || mesh->coeff_kind != DG_COEFF_ONE || quad != k + 2))
        return fail(DG_ERR_UNSUPPORTED, "dg_setup: the diffusion-reaction problems need DG_GEOM_AXIS, DG_COEFF_ONE and quad = k+2");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(DG_ERR_CUDA, "dg_setup: no CUDA device (libdg has no CPU path)");
    if (mesh->device < 0 || mesh->device >= ndev) return fail(DG_ERR_INVALID, "dg_setup: device %d", mesh->device);
    CU(cudaSetDevice(mesh->device));

    dg_ctx* c = (dg_ctx*)calloc(1, sizeof(dg_ctx));
    if (!c) return fail(DG_ERR_OOM, "dg_setup: host allocation");
    c->mesh = *mesh;
    c->mesh.jac = nullptr;
    c->k = k;
    c->n = k + 1;
    c->device = mesh->device;
    c->stream = (cudaStream_t)mesh->stream;
    const int n = c->n;

    dg::HostTables H;
    if (dg::build_tables(n, &H)) { free(c); return fail(DG_ERR_INVALID, "tables n=%d", n); }
    switch (n) {
    case 2: fill_tab<2>(H, c->tab); break;
    case 3: fill_tab<3>(H, c->tab); break;
    case 4: fill_tab<4>(H, c->tab); break;
    case 5: fill_tab<5>(H, c->tab); break;
    case 6: fill_tab<6>(H, c->tab); break;
    case 7: fill_tab<7>(H, c->tab); break;
    case 8: fill_tab<8>(H, c->tab); break;
    }

    dg::MeshArgs& M = c->M;
    M.N0 = mesh->N[0]; M.N1 = mesh->N[1]; M.N2 = mesh->N[2];
    M.plane_begin = mesh->plane_begin;
    M.L = mesh->nplanes;
    M.plane_cells = mesh->N[1] * mesh->N[2];
    for (int d = 0; d < 3; ++d) {
        M.h[d] = 1.0 / mesh->N[d];
        M.gamma[d] = mesh->penalty_scale * k * (k + 1) * (double)mesh->N[d];
        // the paper's problem: gamma_F = alpha k (k+d-1) |F| / |T| = alpha k (k+2) / h_d
        if (dr || mesh->problem == DG_PROBLEM_STOKES) M.gamma[d] = mesh->penalty_scale * k * (k + 2) * (double)mesh->N[d];
    }
    M.jac = nullptr;
    const int64_t n3 = (int64_t)n * n * n;
    // DOFs per cell: n^3, Stokes 3 n^3 + k^3 ([u_0 | u_1 | u_2 | p])
    const int64_t blk = mesh->problem == DG_PROBLEM_STOKES ? 3 * n3 + (int64_t)k * k * k : n3;
    c->plane_dofs = (int64_t)M.plane_cells * blk;
    c->local_dofs = c->plane_dofs * M.L;

    if (mesh->geom_kind == DG_GEOM_AFFINE) {
        const size_t bytes = sizeof(double) * 9 * (size_t)M.plane_cells * (size_t)(M.L + 2);
        cudaError_t e = cudaMalloc(&c->d_jac, bytes);
        if (e != cudaSuccess) { free(c); return fail(DG_ERR_OOM, "dg_setup: jac alloc %zu B: %s", bytes, cudaGetErrorString(e)); }
        e = cudaMemcpy(c->d_jac, mesh->jac, bytes, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) { cudaFree(c->d_jac); free(c); return fail(DG_ERR_CUDA, "dg_setup: jac copy: %s", cudaGetErrorString(e)); }
        M.jac = c->d_jac;
    }
    c->launch = pick(n, mesh->geom_kind == DG_GEOM_AFFINE, mesh->coeff_kind == DG_COEFF_SINCOS);
    c->kname = "k_cell_general";
    c->m = quad;
    c->quad = quad >= k + 2 || mesh->basis != DG_BASIS_GAUSS;
    if (c->quad) {
        // overintegration: m = n + 1 or n + 2 Gauss points, interpolation A != I -> k_quad
        dg::HostTables Hm;
        if (dg::build_tables(quad, &Hm)) {
            return setup_fail(c, DG_ERR_INVALID, "tables m=%d", quad);
        }
        const int mq = quad - k - 1;
        // the basis: Gauss-Legendre (collocated only at m = n, which does not come here) or Gauss-Lobatto nodes
        dg::HostTables Hb;
        if (mesh->basis == DG_BASIS_LOBATTO) {
            if (dg::build_tables_lobatto(n, &Hb)) return setup_fail(c, DG_ERR_INVALID, "Gauss-Lobatto tables n=%d", n);
        } else if (mesh->basis == DG_BASIS_EQUIDISTANT) {
            if (dg::build_tables_equidistant(n, &Hb)) return setup_fail(c, DG_ERR_INVALID, "equidistant tables n=%d", n);
        } else {
            Hb = H;
        }
        switch (n) {
#define QTAB_CASE(NN)                                                                                                  \
    case NN:                                                                                                           \
        if (mq == 2) fill_qtab<NN, (NN <= 7 ? 2 : 1)>(Hb, Hm, c->qtab);                                                \
        else if (mq == 0) fill_qtab<NN, 0>(Hb, Hm, c->qtab);                                                           \
        else fill_qtab<NN>(Hb, Hm, c->qtab);                                                                           \
        break;
            QTAB_CASE(2) QTAB_CASE(3) QTAB_CASE(4) QTAB_CASE(5) QTAB_CASE(6) QTAB_CASE(7) QTAB_CASE(8)
#undef QTAB_CASE
        }
        cudaError_t e = cudaSuccess;
        const int pr = mesh->problem == DG_PROBLEM_DIFFREAC ? 1 : (mesh->problem == DG_PROBLEM_NLREAC ? 2 : 0);
        c->launch = pick_quad(n, mesh->geom_kind == DG_GEOM_AFFINE, mesh->coeff_kind == DG_COEFF_SINCOS, &e, pr, mq);
        if (e == cudaSuccess && pr == 2) c->launch_jac = pick_quad(n, false, false, &e, 3);
        if (e == cudaErrorInvalidValue)
            return setup_fail(c, DG_ERR_UNSUPPORTED, "dg_setup: k_quad with n=%d, m=%d does not fit in shared memory", n, quad);
        if (e != cudaSuccess) return setup_fail(c, DG_ERR_CUDA, "dg_setup: k_quad attributes: %s", cudaGetErrorString(e));
        c->kname = mesh->problem == DG_PROBLEM_DIFFREAC ? "k_quad_diffreac"
                   : mesh->problem == DG_PROBLEM_NLREAC ? "k_quad_nlreac"
                                                        : "k_quad";
    }
    if (mesh->problem == DG_PROBLEM_STOKES) {
        dg::HostTables Hp;
        if (dg::build_tables(n - 1, &Hp)) {
            return setup_fail(c, DG_ERR_INVALID, "tables n=%d", n - 1);
        }
        switch (n) {
        case 2: fill_stab<2>(H, Hp, c->stab); break;
        case 3: fill_stab<3>(H, Hp, c->stab); break;
        case 4: fill_stab<4>(H, Hp, c->stab); break;
        case 5: fill_stab<5>(H, Hp, c->stab); break;
        case 6: fill_stab<6>(H, Hp, c->stab); break;
        case 7: fill_stab<7>(H, Hp, c->stab); break;
        case 8: fill_stab<8>(H, Hp, c->stab); break;
        }
        cudaError_t e = cudaSuccess;
        c->launch = pick_stokes(n, &e);
        if (e != cudaSuccess) {
            return setup_fail(c, DG_ERR_CUDA, "dg_setup: k_stokes attributes: %s", cudaGetErrorString(e));
        }
        c->stokes = true;
        c->kname = "k_stokes";
        *out = c;
        return DG_OK;
    }
    if (!c->quad) {
        // k_gen when its tiles divide the mesh (odd n^3 needs even T2 and N2 for 16-B aligned bulk rows); otherwise
        // the cell-centric k_cell_general (any N >= 2). A failing attribute call or allocation is an error, not a
        // silent switch to another kernel.
        c->ginfo = pick_gen(n, mesh->geom_kind == DG_GEOM_AFFINE, mesh->coeff_kind == DG_COEFF_SINCOS);
        c->gen = mesh->N[1] % c->ginfo.T1 == 0 && mesh->N[2] % c->ginfo.T2 == 0 &&
                 ((n3 % 2 == 0) || (mesh->N[2] % 2 == 0 && c->ginfo.T2 % 2 == 0)) && getenv("DG_FORCE_GENERAL") == nullptr;
        if (c->gen) {
            cudaError_t e = c->ginfo.attr();
            if (e != cudaSuccess)
                return setup_fail(c, DG_ERR_CUDA, "dg_setup: k_gen shared-memory attribute (%d B): %s", c->ginfo.smem,
                                  cudaGetErrorString(e));
        }
        {
            // planes per work item: enough (chunk, tile) items for ~8 per SM, at most 128 planes (each chunk
            // re-evaluates the face below its first plane and reloads one plane: cfg4 with 32 / 64 / 128 planes per
            // chunk 33.24 / 32.87 / 32.74 ms), the chunks of a column balanced (64 planes: 2 x 32, not 55 + 9)
            const char* gc = getenv("DG_GEN_CHUNK");
            const long long items = (long long)(M.N1 / c->ginfo.T1) * (M.N2 / c->ginfo.T2) * M.L;
            long long ch = items / (8 * 148);
            ch = ch < 2 ? 2 : (ch > 128 ? 128 : ch);
            const long long nchunks = (M.L + ch - 1) / ch;
            ch = (M.L + nchunks - 1) / nchunks;
            c->gen_chunk = gc ? atoi(gc) : (int)ch;
        }
        // k_line for axis-aligned c = 1 meshes whose vectors are L2-resident (<= 32 MB; cfg0, cfg1): no plane pipeline
        c->line = mesh->geom_kind == DG_GEOM_AXIS && mesh->coeff_kind == DG_COEFF_ONE && mesh->problem == DG_PROBLEM_PERIODIC &&
                  8.0 * (double)c->local_dofs <= 32.0 * 1024 * 1024 && getenv("DG_FORCE_GENERAL") == nullptr &&
                  getenv("DG_NO_LINE") == nullptr;
        if (c->line) c->gen = false;
        if (c->gen || c->line) {
            switch (n) {
            case 2: fill_eotab<2>(H, mesh->penalty_scale * k * (k + 1), M.h, c->eotab); break;
            case 3: fill_eotab<3>(H, mesh->penalty_scale * k * (k + 1), M.h, c->eotab); break;
            case 4: fill_eotab<4>(H, mesh->penalty_scale * k * (k + 1), M.h, c->eotab); break;
            case 5: fill_eotab<5>(H, mesh->penalty_scale * k * (k + 1), M.h, c->eotab); break;
            case 6: fill_eotab<6>(H, mesh->penalty_scale * k * (k + 1), M.h, c->eotab); break;
            case 7: fill_eotab<7>(H, mesh->penalty_scale * k * (k + 1), M.h, c->eotab); break;
            case 8: fill_eotab<8>(H, mesh->penalty_scale * k * (k + 1), M.h, c->eotab); break;
            }
        }
        if (c->gen && mesh->geom_kind == DG_GEOM_AFFINE) {
            // per-cell geometry records for k_gen (k_geom, once)
            const long long nc = (long long)M.plane_cells * (M.L + 2);
            cudaError_t e = cudaMalloc(&c->d_geo, sizeof(double) * dg::GREC * (size_t)nc);
            if (e != cudaSuccess) { c->d_geo = nullptr; return setup_fail(c, DG_ERR_OOM, "dg_setup: geometry records: %s", cudaGetErrorString(e)); }
            dg::k_geom<<<(unsigned)((nc + 255) / 256), 256>>>(c->d_jac, c->d_geo, nc, M.plane_cells, M.N1, M.N2, M.L + 2);
            e = cudaDeviceSynchronize();
            if (e != cudaSuccess) return setup_fail(c, DG_ERR_CUDA, "dg_setup: k_geom: %s", cudaGetErrorString(e));
        }
        if (c->gen && mesh->coeff_kind == DG_COEFF_SINCOS) {
            // per-cell c(x) factor tables for k_gen (k_ctab, once)
            const long long nc = (long long)M.plane_cells * (M.L + 2);
            const long long nen = 2LL * 3 * (n + 1);
            const long long cfsz = (3LL * n * n + 1) / 2 * 2;
            cudaError_t e = cudaMalloc(&c->d_ctab, sizeof(double) * 2 * nen * (size_t)nc);
            if (e != cudaSuccess) { c->d_ctab = nullptr; return setup_fail(c, DG_ERR_OOM, "dg_setup: c(x) tables: %s", cudaGetErrorString(e)); }
            e = cudaMalloc(&c->d_cface, sizeof(double) * cfsz * (size_t)nc);
            if (e != cudaSuccess) { c->d_cface = nullptr; return setup_fail(c, DG_ERR_OOM, "dg_setup: face c(x) tables: %s", cudaGetErrorString(e)); }
            dg::XiTab X;
            for (int i = 0; i < 9; ++i) X.xi[i] = i < n ? H.xi[i] : 1.0;
            X.xi[n] = 1.0;
            const long long tot = nc * nen;
            const unsigned g = (unsigned)((tot + 255) / 256);
            switch (n) {
            case 2: dg::k_ctab<2><<<g, 256>>>(c->d_jac, c->d_ctab, nc, M, X); break;
            case 3: dg::k_ctab<3><<<g, 256>>>(c->d_jac, c->d_ctab, nc, M, X); break;
            case 4: dg::k_ctab<4><<<g, 256>>>(c->d_jac, c->d_ctab, nc, M, X); break;
            case 5: dg::k_ctab<5><<<g, 256>>>(c->d_jac, c->d_ctab, nc, M, X); break;
            case 6: dg::k_ctab<6><<<g, 256>>>(c->d_jac, c->d_ctab, nc, M, X); break;
            case 7: dg::k_ctab<7><<<g, 256>>>(c->d_jac, c->d_ctab, nc, M, X); break;
            case 8: dg::k_ctab<8><<<g, 256>>>(c->d_jac, c->d_ctab, nc, M, X); break;
            }
            const unsigned g2 = (unsigned)((nc * cfsz + 255) / 256);
            switch (n) {
            case 2: dg::k_cface<2><<<g2, 256>>>(c->d_jac, c->d_cface, nc, M, X); break;
            case 3: dg::k_cface<3><<<g2, 256>>>(c->d_jac, c->d_cface, nc, M, X); break;
            case 4: dg::k_cface<4><<<g2, 256>>>(c->d_jac, c->d_cface, nc, M, X); break;
            case 5: dg::k_cface<5><<<g2, 256>>>(c->d_jac, c->d_cface, nc, M, X); break;
            case 6: dg::k_cface<6><<<g2, 256>>>(c->d_jac, c->d_cface, nc, M, X); break;
            case 7: dg::k_cface<7><<<g2, 256>>>(c->d_jac, c->d_cface, nc, M, X); break;
            case 8: dg::k_cface<8><<<g2, 256>>>(c->d_jac, c->d_cface, nc, M, X); break;
            }
            e = cudaDeviceSynchronize();
            if (e != cudaSuccess) return setup_fail(c, DG_ERR_CUDA, "dg_setup: k_ctab / k_cface: %s", cudaGetErrorString(e));
        }
        if (c->gen) c->kname = "k_gen";
        if (c->line) c->kname = "k_line";
#ifdef DG_GEN_TRACE
        if (c->gen && getenv("DG_TRACE") && !c->dbg) {
            if (cudaMalloc(&c->dbg, sizeof(long long) * 1024 * 16 * 8) == cudaSuccess) {
                cudaMemset(c->dbg, 0, sizeof(long long) * 1024 * 16 * 8);
                cudaMemcpyToSymbol(dg::g_gen_dbg, &c->dbg, sizeof(long long*));
            } else {
                c->dbg = nullptr;
            }
        }
#endif
    }
    // axis-aligned Q7 fast path: tile T1 x T2 (env DG_AX8_TILE picks an AX8_VARIANTS entry for experiments)
    if (!c->quad) {
        const char* tv = getenv("DG_AX8_TILE");
        c->ax8_tile = 0;
        c->ax8_T1 = 2;
        c->ax8_T2 = 4;
#define AX8_PICK(ID, T1_, T2_, NT, MB)                                                                 \
    if (tv && !strcmp(tv, #T1_ "x" #T2_ "m" #MB)) { c->ax8_tile = ID; c->ax8_T1 = T1_; c->ax8_T2 = T2_; }
        AX8_VARIANTS(AX8_PICK)
#undef AX8_PICK
        const int T1 = c->ax8_T1, T2 = c->ax8_T2;
        const char* cl = getenv("DG_AX8_CHUNK");
        c->ax8_chunk = cl ? atoi(cl) : 16; // planes per work item (0: whole slab; cfg3: 12 -> 16 planes 3.196 -> 3.178 ms)
        c->ax8 = (n == 8 && mesh->geom_kind == DG_GEOM_AXIS && mesh->coeff_kind == DG_COEFF_ONE &&
                  mesh->N[1] % T1 == 0 && mesh->N[2] % T2 == 0 && getenv("DG_FORCE_GENERAL") == nullptr &&
                  getenv("DG_AX8_GEN") == nullptr);
    }
    if (c->ax8) {
        build_axis8(H, mesh->penalty_scale * k * (k + 1), M.h, &c->atab);
        cudaError_t e = cudaSuccess;
        switch (c->ax8_tile) {
#define AX8_ATTR(ID, T1, T2, NT, MB)                                                                                   \
    case ID:                                                                                                           \
        e = cudaFuncSetAttribute(dg::k_axis8<T1, T2, NT, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,             \
                                 dg::ax8::Cfg<T1, T2, NT>::SMEM_BYTES);                                                \
        break;
            AX8_VARIANTS(AX8_ATTR)
#undef AX8_ATTR
        }
        c->line = false; // the Q7 marching kernel on every size
        if (e != cudaSuccess)
            return setup_fail(c, DG_ERR_CUDA, "dg_setup: k_axis8 shared-memory attribute: %s", cudaGetErrorString(e));
        if (!get_encode()) return setup_fail(c, DG_ERR_CUDA, "dg_setup: cuTensorMapEncodeTiled unavailable (driver)");
        c->kname = "k_axis8";
        if (c->ax8 && getenv("DG_TRACE")) {
            if (cudaMalloc(&c->dbg, sizeof(long long) * 1024 * 16 * 8) != cudaSuccess) c->dbg = nullptr;
            else cudaMemset(c->dbg, 0, sizeof(long long) * 1024 * 16 * 8);
        }
    }
    *out = c;
    return DG_OK;
}

int dg_destroy(dg_ctx* c)
{
    if (!c) return DG_OK;
    cudaSetDevice(c->device);
    if (c->d_jac) cudaFree(c->d_jac);
    if (c->d_geo) cudaFree(c->d_geo);
    if (c->d_ctab) cudaFree(c->d_ctab);
    if (c->d_cface) cudaFree(c->d_cface);
    if (c->dbg) {
        // DG_TRACE: dump the stamps of the last launch
        static long long h[1024 * 16 * 8];
        if (cudaMemcpy(h, c->dbg, sizeof h, cudaMemcpyDeviceToHost) == cudaSuccess) {
            FILE* f = fopen(getenv("DG_TRACE"), "wb");
            if (f) { fwrite(h, sizeof h, 1, f); fclose(f); }
        }
        cudaFree(c->dbg);
    }
    if (c->hx_d) cudaFree(c->hx_d);
    if (c->hr_d) cudaFree(c->hr_d);
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    if (c->s_cmp) cudaStreamDestroy(c->s_cmp);
    for (int i = 0; i < 32; ++i) {
        if (c->ev_in[i]) cudaEventDestroy(c->ev_in[i]);
        if (c->ev_cmp[i]) cudaEventDestroy(c->ev_cmp[i]);
    }
    dist_release(c);
    free(c);
    return DG_OK;
}

int dg_set_stream(dg_ctx* c, void* stream)
{
    if (!c) return fail(DG_ERR_INVALID, "dg_set_stream: NULL ctx");
    c->stream = (cudaStream_t)stream;
    return DG_OK;
}

int64_t dg_local_ndofs(const dg_ctx* c) { return c ? c->local_dofs : -1; }
int64_t dg_local_offset(const dg_ctx* c) { return c ? (int64_t)c->mesh.plane_begin * c->plane_dofs : -1; }
int64_t dg_plane_ndofs(const dg_ctx* c) { return c ? c->plane_dofs : -1; }
int dg_launches_per_apply(const dg_ctx* c)
{
    if (!c) return -1;
    if (!c->comm) return 1;
    // collective: (pack) + interior + 2 boundary launches (L <= 2: one launch after the exchange)
    return (c->M.L > 2 ? 3 : 1) + (c->dist_tr ? 1 : 0);
}
const char* dg_kernel_name(const dg_ctx* c) { return c ? c->kname : ""; }

int dg_line_ops(int k, double penalty_scale, const double* x, const double* nb, double* out)
{
    if (!x || !nb || !out) return fail(DG_ERR_INVALID, "dg_line_ops: NULL argument");
    if (k < 1 || k > 7) return fail(DG_ERR_INVALID, "dg_line_ops: k=%d outside [1,7]", k);
    const int n = k + 1;
    dg::HostTables H;
    if (dg::build_tables(n, &H)) return fail(DG_ERR_INVALID, "tables n=%d", n);
    const double P = penalty_scale * k * (k + 1);
    switch (n) {
    case 2: return host_line_ops<2>(H, P, x, nb, out);
    case 3: return host_line_ops<3>(H, P, x, nb, out);
    case 4: return host_line_ops<4>(H, P, x, nb, out);
    case 5: return host_line_ops<5>(H, P, x, nb, out);
    case 6: return host_line_ops<6>(H, P, x, nb, out);
    case 7: return host_line_ops<7>(H, P, x, nb, out);
    default: return host_line_ops<8>(H, P, x, nb, out);
    }
}

int dg_line_ops_axis8(double penalty_scale, const double* x, const double* nb, double* out)
{
    if (!x || !nb || !out) return fail(DG_ERR_INVALID, "dg_line_ops_axis8: NULL argument");
    dg::HostTables H;
    if (dg::build_tables(8, &H)) return fail(DG_ERR_INVALID, "tables n=8");
    const double h[3] = {1.0, 1.0, 1.0};
    dg::AxisTab8 A;
    build_axis8(H, penalty_scale * 7 * 8, h, &A);
    double v[8], xe[4], xo[4], ye[4], yo[4];
    for (int j = 0; j < 8; ++j) v[j] = x[j];
    dg::ax8::split8(v, xe, xo);
    const dg::ax8::Sums t = dg::ax8::sums_eo(A, xe, xo);
    dg::ax8::line_eo(A, xe, xo, t, nb[0], nb[1], nb[2], nb[3], ye, yo);
    for (int i = 0; i < 4; ++i) {
        out[i] = ye[i] + yo[i];
        out[7 - i] = ye[i] - yo[i];
    }
    out[8] = t.TE + t.TO;
    out[9] = t.QE + t.QO;
    out[10] = t.TE - t.TO;
    out[11] = t.QO - t.QE;
    return DG_OK;
}

double dg_alg_flops(const dg_ctx* c)
{
    // collocated sum factorisation, each face once, multiply-add = 2 flops.
    //   axis-aligned Poisson : F = 12 n + 51 + 30/n              per DOF
    //   affine diffusion     : F = 12 n + 117 + Cc + 3 (32 + Cc)/n, Cc = 16 (nominal c(x) cost)
    if (!c) return -1.0;
    const double n = c->n;
    double F;
    if (c->stokes) {
        // Stokes (k_stokes, collocated velocity, pressure n-1 nodes): per cell volume 9 gradient sweeps and
        // their transposes (36 n^4), the pressure interpolation and its transpose
        // 4 (p^3 n + p^2 n^2 + p n^3) (p = n-1), 20 n^3 pointwise; each face once: velocity traces and
        // back-projections both sides (48 n^3), pressure traces / tangential interpolation and back
        // (4 p^3 + 8 (p^2 n + p n^2)), 40 n^2 flux
        const double p = n - 1;
        const double vol = 36 * n * n * n * n + 4 * (p * p * p * n + p * p * n * n + p * n * n * n) + 20 * n * n * n;
        const double face = 48 * n * n * n + 4 * p * p * p + 8 * (p * p * n + p * n * n) + 40 * n * n;
        return (vol + 3.0 * face) / (3 * n * n * n + p * p * p) * (double)c->local_dofs;
    }
    if (c->quad) {
        // general quadrature (k_quad, m points): the sum-factorisation contractions as executed (A != I):
        // volume 2 (4 n^3 m + 6 n^2 m^2 + 6 n m^3) + (21 + Cc) m^3 per cell; each face once:
        // 2 (8 n^3 + 9 n^2 m + 12 n m^2) + (40 + Cc) m^2 (traces both sides, interpolation / tangential
        // derivatives to the m^2 points, flux, back-projection)
        const double m = c->m, Cc = (c->mesh.coeff_kind == DG_COEFF_SINCOS) ? 16.0 : 0.0;
        const double vol = 2.0 * (4 * n * n * n * m + 6 * n * n * m * m + 6 * n * m * m * m) + (21.0 + Cc) * m * m * m;
        const double face = 2.0 * (8 * n * n * n + 9 * n * n * m + 12 * n * m * m) + (40.0 + Cc) * m * m;
        // the diffusion-reaction problem adds u at the M^3 points (2 n m^3), its back-projection (2 n m^3),
        // the full K (12 m^3) and the reaction / source term (3 m^3)
        // (the nonlinear variant: 6 more flops per point for c u^2 - f(x))
        const double dr = (c->mesh.problem == DG_PROBLEM_DIFFREAC) ? 4 * n * m * m * m + 15 * m * m * m
                          : (c->mesh.problem == DG_PROBLEM_NLREAC) ? 4 * n * m * m * m + 21 * m * m * m : 0.0;
        return (vol + dr + 3.0 * face) / (n * n * n) * (double)c->local_dofs;
    }
    if (c->mesh.geom_kind == DG_GEOM_AXIS && c->mesh.coeff_kind == DG_COEFF_ONE)
        F = 12.0 * n + 51.0 + 30.0 / n;
    else {
        const double Cc = (c->mesh.coeff_kind == DG_COEFF_SINCOS) ? 16.0 : 0.0;
        if (c->mesh.geom_kind == DG_GEOM_AXIS)
            F = 12.0 * n + 51.0 + 30.0 / n + Cc * (1.0 + 3.0 / n); // c(x) at volume + face points
        else
            F = 12.0 * n + 117.0 + Cc + 3.0 * (32.0 + Cc) / n;
    }
    return F * (double)c->local_dofs;
}

double dg_alg_bytes(const dg_ctx* c)
{
    if (!c) return -1.0;
    double b = 16.0 * (double)c->local_dofs;
    // 120 B per affine cell (J and the symmetric G~ = |det J| J^-1 J^-T)
    if (c->mesh.geom_kind == DG_GEOM_AFFINE) b += 120.0 * (double)c->M.plane_cells * c->M.L;
    return b;
}

static int apply_planes_impl(dg_ctx* c, const double* x, const double* xb, const double* xa, double* r, int p0, int p1,
                             const double* u0, int halo_tr = 0);

int dg_apply_planes(dg_ctx* c, const double* x, const double* xb, const double* xa, double* r, int p0, int p1)
{
    return apply_planes_impl(c, x, xb, xa, r, p0, p1, nullptr);
}

int64_t dg_halo_ndofs(const dg_ctx* c) { return c ? (int64_t)c->M.plane_cells * 2 * c->n * c->n : -1; }

int dg_apply_planes_tr(dg_ctx* c, const double* x, const double* tr_below, const double* tr_above, double* r, int p0,
                       int p1)
{
    if (!c) return fail(DG_ERR_INVALID, "dg_apply_planes_tr: NULL ctx");
    if (!(c->gen || c->ax8 || c->line))
        return fail(DG_ERR_UNSUPPORTED, "dg_apply_planes_tr: trace halos need k_gen, k_axis8 or k_line (context kernel %s)",
                    c->kname);
    return apply_planes_impl(c, x, tr_below, tr_above, r, p0, p1, nullptr, 3);
}

int dg_pack_halo(dg_ctx* c, const double* x, double* tr_lo, double* tr_hi)
{
    if (!c || !x || !tr_lo || !tr_hi) return fail(DG_ERR_INVALID, "dg_pack_halo: NULL argument");
    if (!(c->gen || c->ax8 || c->line))
        return fail(DG_ERR_UNSUPPORTED, "dg_pack_halo: trace halos need k_gen, k_axis8 or k_line (context kernel %s)", c->kname);
    if (((uintptr_t)x | (uintptr_t)tr_lo | (uintptr_t)tr_hi) & 15)
        return fail(DG_ERR_INVALID, "dg_pack_halo: pointers must be 16-byte aligned");
    const long long tot = 2LL * c->M.plane_cells * c->n * c->n;
    const unsigned g = (unsigned)((tot + 255) / 256);
    if (c->ax8) {
        dg::k_pack_traces8<<<g, 256, 0, c->stream>>>(x, tr_lo, tr_hi, c->M.plane_cells, c->M.L, c->atab);
    } else {
        switch (c->n) {
#define PACK_CASE(NN)                                                                                                  \
    case NN:                                                                                                           \
        dg::k_pack_traces<NN><<<g, 256, 0, c->stream>>>(x, tr_lo, tr_hi, c->M.plane_cells, c->M.L,                     \
                                                         *reinterpret_cast<const dg::EOTab<NN>*>(c->eotab));             \
        break;
            PACK_CASE(2) PACK_CASE(3) PACK_CASE(4) PACK_CASE(5) PACK_CASE(6) PACK_CASE(7) PACK_CASE(8)
#undef PACK_CASE
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(DG_ERR_CUDA, "dg_pack_halo: launch: %s", cudaGetErrorString(e));
    return DG_OK;
}

int dg_apply_jacobian_planes(dg_ctx* c, const double* u0, const double* z, const double* zb, const double* za, double* r,
                             int p0, int p1)
{
    if (!c) return fail(DG_ERR_INVALID, "dg_apply_jacobian: NULL ctx");
    if (c->mesh.problem != DG_PROBLEM_NLREAC || !c->launch_jac)
        return fail(DG_ERR_UNSUPPORTED, "dg_apply_jacobian: the context's problem (%d) is not DG_PROBLEM_NLREAC", c->mesh.problem);
    if (!u0) return fail(DG_ERR_INVALID, "dg_apply_jacobian: NULL u0");
    const size_t bytes = sizeof(double) * (size_t)c->local_dofs;
    const char *us = (const char*)u0, *rs = (const char*)r;
    if (r && us < rs + bytes && rs < us + bytes) return fail(DG_ERR_INVALID, "dg_apply_jacobian: u0 and r overlap");
    if ((uintptr_t)u0 & 7) return fail(DG_ERR_INVALID, "dg_apply_jacobian: u0 must be 8-byte aligned");
    return apply_planes_impl(c, z, zb, za, r, p0, p1, u0);
}

int dg_apply_jacobian(dg_ctx* c, const double* u0, const double* z, double* r)
{
    if (!c) return fail(DG_ERR_INVALID, "dg_apply_jacobian: NULL ctx");
    if (c->M.L != c->M.N0)
        return fail(DG_ERR_INVALID, "dg_apply_jacobian: context owns %d of %d planes; use dg_apply_jacobian_planes", c->M.L,
                    c->M.N0);
    if (!z || !r) return fail(DG_ERR_INVALID, "dg_apply_jacobian: NULL vector");
    return dg_apply_jacobian_planes(c, u0, z, z + (size_t)(c->M.L - 1) * c->plane_dofs, z, r, 0, c->M.L);
}

static int apply_planes_impl(dg_ctx* c, const double* x, const double* xb, const double* xa, double* r, int p0, int p1,
                             const double* u0, int halo_tr)
{
    if (!c || !x || !xb || !xa || !r) return fail(DG_ERR_INVALID, "dg_apply_planes: NULL argument");
    if (p0 < 0 || p1 > c->M.L || p0 > p1) return fail(DG_ERR_INVALID, "dg_apply_planes: planes [%d,%d) of %d", p0, p1, c->M.L);
    const size_t bytes = sizeof(double) * (size_t)c->local_dofs;
    const char *xs = (const char*)x, *rs = (const char*)r;
    if (xs < rs + bytes && rs < xs + bytes) return fail(DG_ERR_INVALID, "dg_apply: x and r overlap");
    // alignment contract (include/dg.h): 8 bytes for every pointer; 16 bytes for x, r and both halo planes of the
    // marching-tile kernels (k_gen, k_axis8: 16-B vector and bulk-copy accesses); x 128 bytes for k_axis8 (TMA
    // tensor map base)
    if (((uintptr_t)x | (uintptr_t)r | (uintptr_t)xb | (uintptr_t)xa) & 7)
        return fail(DG_ERR_INVALID, "dg_apply: pointers must be 8-byte aligned");
    if ((((uintptr_t)x | (uintptr_t)r | (uintptr_t)xb | (uintptr_t)xa) & 15) && (c->gen || c->ax8))
        return fail(DG_ERR_INVALID, "dg_apply: x, r, x_below and x_above must be 16-byte aligned (%s)", c->kname);
    if (((uintptr_t)x & 127) && c->ax8) return fail(DG_ERR_INVALID, "dg_apply: x must be 128-byte aligned (k_axis8)");
    cudaError_t e = launch_planes(c, x, xb, xa, r, p0, p1, c->stream, u0, halo_tr);
    if (e != cudaSuccess) return fail(DG_ERR_CUDA, "dg_apply: launch: %s", cudaGetErrorString(e));
    return DG_OK;
}

int dg_apply(dg_ctx* c, const double* x, double* r)
{
    if (!c) return fail(DG_ERR_INVALID, "dg_apply: NULL ctx");
    if (c->M.L != c->M.N0)
        return fail(DG_ERR_INVALID, "dg_apply: context owns %d of %d planes; use dg_apply_planes with halos", c->M.L,
                    c->M.N0);
    if (!x || !r) return fail(DG_ERR_INVALID, "dg_apply: NULL vector");
    return dg_apply_planes(c, x, x + (size_t)(c->M.L - 1) * c->plane_dofs, x, r, 0, c->M.L);
}

int dg_apply_host(dg_ctx* c, const double* xh, double* rh)
{
    if (!c || !xh || !rh) return fail(DG_ERR_INVALID, "dg_apply_host: NULL argument");
    if (c->M.L != c->M.N0) return fail(DG_ERR_INVALID, "dg_apply_host: whole-mesh context required");
    CU(cudaSetDevice(c->device));
    const size_t bytes = sizeof(double) * (size_t)c->local_dofs;
    // staging state, created on first use and owned by the context (each piece only once, so a failed first
    // call leaks nothing and a retry completes it; dg_destroy frees what exists)
    if (!c->hx_d) CU(cudaMalloc(&c->hx_d, bytes));
    if (!c->hr_d) CU(cudaMalloc(&c->hr_d, bytes));
    if (!c->s_h2d) CU(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    if (!c->s_d2h) CU(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    if (!c->s_cmp) CU(cudaStreamCreateWithFlags(&c->s_cmp, cudaStreamNonBlocking));
    for (int i = 0; i < 32; ++i) {
        if (!c->ev_in[i]) CU(cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming));
        if (!c->ev_cmp[i]) CU(cudaEventCreateWithFlags(&c->ev_cmp[i], cudaEventDisableTiming));
    }
    const int L = c->M.L;
    const int64_t pd = c->plane_dofs;
    const size_t pbytes = sizeof(double) * (size_t)pd;
    // chunks of planes; chunk i computes planes [b_i, e_i) once planes [b_i-1, e_i] are resident
    // up to 32 chunks: the transfers of the last chunk (compute of chunk i waits for chunk i+1's first plane, so
    // about two chunks of D2H trail the last H2D) are 1/16 of the step instead of 1/4 with 8 chunks
    int nch = L >= 32 ? 32 : L;
    if (const char* hc = getenv("DG_HOST_CHUNKS")) { // experiments only
        const int v = atoi(hc);
        if (v >= 1 && v <= 32) nch = v < L ? v : L;
    }
    int bnd[33];
    for (int i = 0; i <= nch; ++i) bnd[i] = (int)((int64_t)L * i / nch);
    cudaEvent_t* ev_in = c->ev_in;
    cudaEvent_t* ev_cmp = c->ev_cmp;
    // H2D: the last plane first (wrap halo of chunk 0), then chunks in order
    CU(cudaMemcpyAsync(c->hx_d + (size_t)(L - 1) * pd, xh + (size_t)(L - 1) * pd, pbytes, cudaMemcpyHostToDevice,
                       c->s_h2d));
    for (int i = 0; i < nch; ++i) {
        int b = bnd[i], e = bnd[i + 1];
        if (i == nch - 1) e = L - 1; // last plane already sent
        if (e > b)
            CU(cudaMemcpyAsync(c->hx_d + (size_t)b * pd, xh + (size_t)b * pd, pbytes * (size_t)(e - b),
                               cudaMemcpyHostToDevice, c->s_h2d));
        CU(cudaEventRecord(ev_in[i], c->s_h2d));
    }
    // compute chunk i after chunk i+1 arrived (needs plane e_i); the last chunk needs plane 0 (chunk 0)
    for (int i = 0; i < nch; ++i) {
        const int need = (i + 1 < nch) ? i + 1 : nch - 1;
        CU(cudaStreamWaitEvent(c->s_cmp, ev_in[need], 0));
        cudaError_t e = launch_planes(c, c->hx_d, c->hx_d + (size_t)(L - 1) * pd, c->hx_d, c->hr_d, bnd[i],
                                      bnd[i + 1], c->s_cmp);
        if (e != cudaSuccess) return fail(DG_ERR_CUDA, "dg_apply_host: launch: %s", cudaGetErrorString(e));
        CU(cudaEventRecord(ev_cmp[i], c->s_cmp));
        CU(cudaStreamWaitEvent(c->s_d2h, ev_cmp[i], 0));
        CU(cudaMemcpyAsync(rh + (size_t)bnd[i] * pd, c->hr_d + (size_t)bnd[i] * pd,
                           pbytes * (size_t)(bnd[i + 1] - bnd[i]), cudaMemcpyDeviceToHost, c->s_d2h));
    }
    CU(cudaStreamSynchronize(c->s_d2h));
    return DG_OK;
}

// ---------------------------------------------------------------------------------------------------------------
// Collective form: x0-slabs over nranks processes, one NCCL point-to-point halo step per
// application, overlapped with the interior planes (include/dg.h).

int dg_slab_range(int N0, int rank, int nranks, int32_t* plane_begin, int32_t* nplanes)
{
    if (!plane_begin || !nplanes) return fail(DG_ERR_INVALID, "dg_slab_range: NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks || N0 < nranks)
        return fail(DG_ERR_INVALID, "dg_slab_range: rank %d of %d on %d planes", rank, nranks, N0);
    const int b = (int)((int64_t)rank * N0 / nranks), e = (int)((int64_t)(rank + 1) * N0 / nranks);
    *plane_begin = b;
    *nplanes = e - b;
    return DG_OK;
}

int dg_get_unique_id(void* id)
{
    if (!id) return fail(DG_ERR_INVALID, "dg_get_unique_id: NULL argument");
    const NcclApi* N = nccl_api();
    if (!N) return fail(DG_ERR_NCCL, "dg_get_unique_id: libnccl.so.2 not found");
    ncclUniqueId u;
    const ncclResult_t e = N->GetUniqueId(&u);
    if (e != ncclSuccess) return fail(DG_ERR_NCCL, "ncclGetUniqueId: %s", N->GetErrorString(e));
    memcpy(id, &u, sizeof u);
    return DG_OK;
}

int dg_setup_dist(const dg_mesh* mesh, int k, int quad, int rank, int nranks, const void* nccl_id, dg_ctx** out)
{
    g_err.clear();
    if (!mesh || !out || !nccl_id) return fail(DG_ERR_INVALID, "dg_setup_dist: NULL argument");
    *out = nullptr;
    int32_t pb = 0, np = 0;
    int rc = dg_slab_range(mesh->N[0], rank, nranks, &pb, &np);
    if (rc != DG_OK) return rc;
    if (mesh->plane_begin != pb || mesh->nplanes != np)
        return fail(DG_ERR_INVALID, "dg_setup_dist: mesh slab [%d, +%d) is not rank %d's slab [%d, +%d) (dg_slab_range)",
                    mesh->plane_begin, mesh->nplanes, rank, pb, np);
    const NcclApi* N = nccl_api();
    if (!N) return fail(DG_ERR_NCCL, "dg_setup_dist: libnccl.so.2 not found");
    dg_ctx* c = nullptr;
    rc = dg_setup(mesh, k, quad, &c);
    if (rc != DG_OK) return rc;
    c->rank = rank;
    c->nranks = nranks;
    // trace halos where the kernel consumes them (dg_apply_planes_tr), else full boundary planes
    c->dist_tr = c->gen || c->ax8 || c->line;
    c->halo_n = c->dist_tr ? dg_halo_ndofs(c) : c->plane_dofs;
    const size_t hb = sizeof(double) * (size_t)c->halo_n;
    cudaError_t e = cudaMalloc(&c->d_hb, hb);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_ha, hb);
    if (e == cudaSuccess && c->dist_tr) e = cudaMalloc(&c->d_tlo, hb);
    if (e == cudaSuccess && c->dist_tr) e = cudaMalloc(&c->d_thi, hb);
    if (e != cudaSuccess) return setup_fail(c, DG_ERR_OOM, "dg_setup_dist: halo buffers: %s", cudaGetErrorString(e));
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    e = cudaStreamCreateWithPriority(&c->s_comm, cudaStreamNonBlocking, hi_prio);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_x, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming);
    if (e != cudaSuccess) return setup_fail(c, DG_ERR_CUDA, "dg_setup_dist: streams / events: %s", cudaGetErrorString(e));
    ncclUniqueId u;
    memcpy(&u, nccl_id, sizeof u);
    const ncclResult_t ne = N->CommInitRank(&c->comm, nranks, u, rank);
    if (ne != ncclSuccess) {
        c->comm = nullptr;
        return setup_fail(c, DG_ERR_NCCL, "ncclCommInitRank(rank %d of %d): %s", rank, nranks, N->GetErrorString(ne));
    }
    *out = c;
    return DG_OK;
}

int dg_apply_dist(dg_ctx* c, const double* x, double* r)
{
    if (!c || !x || !r) return fail(DG_ERR_INVALID, "dg_apply_dist: NULL argument");
    if (!c->comm) return fail(DG_ERR_INVALID, "dg_apply_dist: context was not created by dg_setup_dist");
    const NcclApi* N = nccl_api();
    const int L = c->M.L;
    const int below = (c->rank + c->nranks - 1) % c->nranks, above = (c->rank + 1) % c->nranks;
    const int halo_tr = c->dist_tr ? 3 : 0;
    CU(cudaSetDevice(c->device));
    const double *send_lo, *send_hi;
    if (c->dist_tr) {
        const int rc = dg_pack_halo(c, x, c->d_tlo, c->d_thi);
        if (rc != DG_OK) return rc;
        send_lo = c->d_tlo;
        send_hi = c->d_thi;
    } else {
        send_lo = x;
        send_hi = x + (size_t)(L - 1) * c->plane_dofs;
    }
    CU(cudaEventRecord(c->ev_x, c->stream));
    CU(cudaStreamWaitEvent(c->s_comm, c->ev_x, 0));
    // interior planes (their x0-neighbours are local; the halos are not read) overlap the exchange
    if (L > 2) {
        const int rc = apply_planes_impl(c, x, c->d_hb, c->d_ha, r, 1, L - 1, nullptr, halo_tr);
        if (rc != DG_OK) return rc;
    }
    // one exchange step: my lowest plane's payload -> rank below (its halo above), my highest -> rank above;
    // NCCL pairs the point-to-point operations between two ranks in posting order (also rank == peer)
    ncclResult_t ne = N->GroupStart();
    if (ne == ncclSuccess) ne = N->Send(send_lo, (size_t)c->halo_n, ncclDouble, below, c->comm, c->s_comm);
    if (ne == ncclSuccess) ne = N->Send(send_hi, (size_t)c->halo_n, ncclDouble, above, c->comm, c->s_comm);
    if (ne == ncclSuccess) ne = N->Recv(c->d_ha, (size_t)c->halo_n, ncclDouble, above, c->comm, c->s_comm);
    if (ne == ncclSuccess) ne = N->Recv(c->d_hb, (size_t)c->halo_n, ncclDouble, below, c->comm, c->s_comm);
    const ncclResult_t ge = N->GroupEnd();
    if (ne == ncclSuccess) ne = ge;
    if (ne != ncclSuccess) return fail(DG_ERR_NCCL, "dg_apply_dist: halo exchange: %s", N->GetErrorString(ne));
    CU(cudaEventRecord(c->ev_halo, c->s_comm));
    CU(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
    if (L <= 2) return apply_planes_impl(c, x, c->d_hb, c->d_ha, r, 0, L, nullptr, halo_tr);
    int rc = apply_planes_impl(c, x, c->d_hb, c->d_ha, r, 0, 1, nullptr, halo_tr);
    if (rc == DG_OK) rc = apply_planes_impl(c, x, c->d_hb, c->d_ha, r, L - 1, L, nullptr, halo_tr);
    return rc;
}

} // extern "C"
