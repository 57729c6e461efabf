// K_gen: the general sum-factorised SIPG operator (any degree n = k+1 in 2..8, per-cell affine
// geometry, c(x)) — the path of the affine configs (cfg2 Q5, cfg4 Q4) and of the axis-aligned
// configs other than Q7. Successor of the round-1 k_tile with the same mathematics:
//
//   Alg. assembly per cell, collocation (A = I, reading R8):
//     stage 1  grad_hat U = (D along d) X,
//     stage 2  Q = w_q c(x_q) |det J| J^{-1} J^{-T} grad_hat U,       P:L867-872 (Eq. diffreac_weak)
//     stage 3  R = sum_d (D^T along d) Q_d,
//   faces (P:L883-886, 1-point tables e0/e1/d0/d1 P:L143-146), SIPG flux of Eq. diffreac_weak
//   (theta = -1), geometry of T- (reading R11), c_F at the T- mapped point (R12).
//
// What is new against k_tile (design notes):
//  * every global input of a plane step (own blocks of the NEXT plane, ring blocks, geometry
//    records) arrives asynchronously one step ahead (cp.async.bulk + mbarrier; odd-sized ring
//    cells as 16-B aligned pairs): the compute phases touch only shared memory and registers;
//  * line sweeps in even/odd form (D is centro-antisymmetric on the symmetric Gauss nodes): about
//    half the FMAs of a plain n x n product and half-length dependency chains;
//  * faces are evaluated once per face (T- side owner), with the tangential parts of both sides
//    combined by linearity: {g} needs D_t (a-_t u- + a+_t u+), and the back-projection of the
//    gradient test term needs D_t^T Cg once per face (a+- constant on an affine face);
//  * the T+ half of the face to the next plane stays in the registers of the thread that owns the
//    same line position on the next plane (no pending buffer);
//  * stage-3 partial sums of directions 0 and 1 are written in place of Q_0 / Q_1 (one barrier
//    fewer); direction 2 stays in registers from stage 1 to stage 3.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "kernel_geom.cuh" // k_geom / GREC records, tl:: mbarrier + bulk-copy helpers

namespace dg {

// Even/odd (centro-(anti)symmetric) forms of the 1D tables, built on the host (dg_capi.cu).
// With xe_j = x_j + x_{n-1-j}, xo_j = x_j - x_{n-1-j} (j < H), xe_H = x_H (odd n):
//   y = D x      : S_q = sum_{j<H} Fm[q][j] xo_j, A_q = sum_{j<HE} Fp[q][j] xe_j, y_q = S_q + A_q,
//                  y_{n-1-q} = S_q - A_q (q < H); odd n: y_H = sum_{j<H} Fmid[j] xo_j
//   y = D^T x    : the same with the transposed halves (tm / tp below)
//   traces       : u_lo = TE + TO, u_hi = TE - TO, gn_lo = QE + QO, gn_hi = QO - QE with
//                  TE = sum Es xe, TO = sum Ea xo, QE = sum Ds xe, QO = sum Da xo
//   face terms of stage 3: S_i += Es_i (Vl + Vh) + Ds_i (Gl - Gh), A_i += Ea_i (Vl - Vh) + Da_i (Gl + Gh)
template <int N>
struct EOTab {
    static constexpr int H = N / 2, ODD = N & 1, HE = H + ODD;
    double Fm[H][H], Fp[H][HE], Fmid[H];
    double Es[HE], Ea[H], Ds[HE], Da[H];
    double D[N * N];   // plain D[q*N + j] (tangential face derivatives)
    double w[N], xi[N];
    // line-operator form (axis-aligned, c = 1; LINEOP): the centro-symmetric 1D SIPG line operator
    // B^ = D^T W D + 1/2 (e0 d0^T + d0 e0^T - e1 d1^T - d1 e1^T) + P (e0 e0^T + e1 e1^T) in even/odd form
    // (Se_i = sum Lp[i][j] xe_j, So_i = sum Lm[i][j] xo_j, y_i = Se + So, y_{n-1-i} = Se - So; odd middle
    // y_H = sum Lmid[j] xe_j) and its neighbour-trace couplings (Ae, Be on the sums, Ao, Bo on the differences)
    double Lp[H][HE], Lm[H][H], Lmid[HE];
    double Ae[HE], Be[HE], Ao[H], Bo[H];
    double Sc[3]; // h_t1 h_t2 / h_d
};

namespace gn {

struct RunD { // a face direction known only at run time (the warp-local face phase)
    int value;
};

using tl::bulk_g2s;
using tl::mbar_expect_tx;
using tl::mbar_init;
using tl::mbar_wait;
using tl::s32;


// split a line into even/odd halves
template <int N>
__host__ __device__ __forceinline__ void split(const double v[N], double xe[EOTab<N>::HE], double xo[EOTab<N>::H])
{
    constexpr int H = EOTab<N>::H;
#pragma unroll
    for (int j = 0; j < H; ++j) {
        xe[j] = v[j] + v[N - 1 - j];
        xo[j] = v[j] - v[N - 1 - j];
    }
    if (N & 1) xe[H] = v[H];
}

// The halves of D^T are those of D transposed (D centro-antisymmetric: D(n-1-j, q) = -D(j, n-1-q)): Tm[q][j] =
// Fp[j][q], Tp[q][j] = Fm[j][q] (j < H), Tp[q][H] = Fmid[q], Tmid[j] = Fp[j][H]. The sweeps read D's halves only, so a
// kernel keeps half the distinct table doubles live (sm_100a DFMA takes table operands from the 63 uniform registers).
template <int N>
__host__ __device__ __forceinline__ double tm(const EOTab<N>& E, int q, int j) { return E.Fp[j][q]; }
template <int N>
__host__ __device__ __forceinline__ double tp(const EOTab<N>& E, int q, int j)
{
    return j < EOTab<N>::H ? E.Fm[j][q] : E.Fmid[q];
}

// y = D x (TR = false) or y = D^T x (TR = true), plus optional stage-3 face terms at both ends
template <int N, bool TR, bool FACE>
__host__ __device__ __forceinline__ void sweep(const EOTab<N>& E, const double xe[EOTab<N>::HE], const double xo[EOTab<N>::H],
                                      double y[N], double Vl = 0, double Gl = 0, double Vh = 0, double Gh = 0)
{
    constexpr int H = EOTab<N>::H, HE = EOTab<N>::HE;
    const double sV = Vl + Vh, dV = Vl - Vh, sG = Gl + Gh, dG = Gl - Gh;
#pragma unroll
    for (int q = 0; q < H; ++q) {
        double S = FACE ? fma(E.Es[q], sV, E.Ds[q] * dG) : 0.0;
        double A = FACE ? fma(E.Ea[q], dV, E.Da[q] * sG) : 0.0;
#pragma unroll
        for (int j = 0; j < H; ++j) S = fma(TR ? tm(E, q, j) : E.Fm[q][j], xo[j], S);
#pragma unroll
        for (int j = 0; j < HE; ++j) A = fma(TR ? tp(E, q, j) : E.Fp[q][j], xe[j], A);
        y[q] = S + A;
        y[N - 1 - q] = S - A;
    }
    if (N & 1) {
        double m = FACE ? fma(E.Es[H], sV, E.Ds[H] * dG) : 0.0;
#pragma unroll
        for (int j = 0; j < H; ++j) m = fma(TR ? E.Fp[j][H] : E.Fmid[j], xo[j], m);
        y[H] = m;
    }
}

// traces of a line at both ends: u_lo = e0.x, u_hi = e1.x, g_lo = d0.x, g_hi = d1.x
template <int N>
__host__ __device__ __forceinline__ void traces(const EOTab<N>& E, const double xe[EOTab<N>::HE], const double xo[EOTab<N>::H],
                                       double& ulo, double& glo, double& uhi, double& ghi)
{
    constexpr int H = EOTab<N>::H, HE = EOTab<N>::HE;
    double te = 0, to = 0, qe = 0, qo = 0;
#pragma unroll
    for (int j = 0; j < HE; ++j) {
        te = fma(E.Es[j], xe[j], te);
        qe = fma(E.Ds[j], xe[j], qe);
    }
#pragma unroll
    for (int j = 0; j < H; ++j) {
        to = fma(E.Ea[j], xo[j], to);
        qo = fma(E.Da[j], xo[j], qo);
    }
    ulo = te + to;
    uhi = te - to;
    glo = qe + qo;
    ghi = qo - qe;
}

// y = B^ x + neighbour terms (line-operator form, LINEOP): uL, gL = (e1.x, d1.x) of the lower
// neighbour's line, uR, gR = (e0.x, d0.x) of the upper neighbour's line
template <int N>
__host__ __device__ __forceinline__ void lineop(const EOTab<N>& E, const double xe[EOTab<N>::HE], const double xo[EOTab<N>::H],
                                       double y[N], double uL, double gL, double uR, double gR)
{
    constexpr int H = EOTab<N>::H, HE = EOTab<N>::HE;
    const double su = uL + uR, du = uL - uR, sg = gL + gR, dg = gL - gR;
#pragma unroll
    for (int i = 0; i < H; ++i) {
        double e = fma(E.Ae[i], su, E.Be[i] * dg);
        double o = fma(E.Ao[i], du, E.Bo[i] * sg);
#pragma unroll
        for (int j = 0; j < HE; ++j) e = fma(E.Lp[i][j], xe[j], e);
#pragma unroll
        for (int j = 0; j < H; ++j) o = fma(E.Lm[i][j], xo[j], o);
        y[i] = e + o;
        y[N - 1 - i] = e - o;
    }
    if (N & 1) {
        double m = fma(E.Ae[H], su, E.Be[H] * dg);
#pragma unroll
        for (int j = 0; j < HE; ++j) m = fma(E.Lmid[j], xe[j], m);
        y[H] = m;
    }
}

__device__ __forceinline__ void cmul(double ar, double ai, double br, double bi, double& cr, double& ci)
{
    cr = fma(ar, br, -ai * bi);
    ci = fma(ar, bi, ai * br);
}

// a face point's (u, g) pair in two separate shared arrays, used like a double2
struct TRRef {
    double& x;
    double& y;
    __device__ __forceinline__ operator double2() const { return make_double2(x, y); }
    __device__ __forceinline__ void operator=(double2 v) { x = v.x; y = v.y; }
};
struct TRView {
    double* u;
    double* g;
    __device__ __forceinline__ TRRef operator[](int p) const { return TRRef{u[p], g[p]}; }
};

// lane -> task (fo N + l) of the warp-local face pass B (t2-lines); -1: idle lane. Tables from an offline search
// (tools/passb_perm.py) for the face-slot strides FSD = FB = TSEL mod 16 of Lay; identity for other n
__constant__ signed char c_passb3[32] = {26, 16, 11, 10, 23, 5, 29, 20, 28, 17, 13, 0, 19, 12, 14, 3,
                                        1, 7, 9, 22, 6, 21, 15, 8, 2, 24, 25, 27, 18, 4, -1, -1};
__constant__ signed char c_passb4[32] = {26, 17, 11, 10, 28, 1, 4, 7, 16, 9, 19, 13, 0, 23, 14, 18,
                                        5, 30, 22, 21, 29, 6, 12, 20, 15, 3, 31, 2, 24, 25, 27, 8};
__constant__ signed char c_passb5[32] = {26, 16, 11, 10, 23, 1, 5, 7, 20, 9, 28, 13, 19, 22, 6, 24,
                                        29, 17, 0, 12, 21, 14, 15, 3, 8, 2, 25, 27, 18, 4, -1, -1};
template <int N>
__device__ __forceinline__ int passb_task(int lane)
{
    if (N == 3) return c_passb3[lane];
    if (N == 4) return c_passb4[lane];
    if (N == 5) return c_passb5[lane];
    return lane < (32 / N) * N ? lane : -1;
}

// shared-memory layout (in doubles) of k_gen<N, AFFINE, COEFF, T1, T2>
template <int N, bool AFFINE, bool COEFF, int T1, int T2>
struct Lay {
    static constexpr int N2 = N * N, N3 = N * N * N, NC = T1 * T2;
    static constexpr int NACT = NC * N2;
    static constexpr int NT = (NACT + 31) / 32 * 32;
    static constexpr int NRL = T1 + T2, NRH = T1 + T2; // ring cells below / above the tile
    static constexpr int NF = 3 * NC + NRL;            // faces evaluated by the CTA per plane
    static constexpr int CXSZ = 2 * 3 * (N + 1) * 2;   // per cell: [coord k][axis b][q = 0..N] complex
    static constexpr int CFSZ = (3 * N2 + 1) / 2 * 2;  // per cell: c at the points of its 3 upper faces (even)
    static constexpr int NCG = NC + NRL;               // cells with geometry / c tables (own + ring below)
    // regions
    static constexpr int XS = 0;                                        // [2][NC][N3] own planes
    // ring blocks: bd1[T2] bd2[T1 slots] ad1[T2] ad2[T1 slots]; for odd n^3 a d = 2 ring slot holds the 16-B aligned
    // PAIR of cells around the needed one (one bulk copy instead of per-element cp.async: N2, T2 even)
    static constexpr int SL = (N3 % 2) == 0 ? 1 : 2;
    static constexpr int RB1 = 0, RB2 = T2, RA1 = T2 + SL * T1, RA2 = 2 * T2 + SL * T1;
    static constexpr int RXSZ = (2 * T2 + 2 * SL * T1) * N3;
    // affine face passes: per face line (N points per thread, 2 buffers, warp-local A -> B -> C) for n <= 6,
    // per face point (3 buffers, CTA barriers between the passes) for n >= 7
    static constexpr bool FACE_LINES = N <= 6;
    // face slots: [u-, u+, g-, g+] (N2 doubles each; u/V and gn/G kept apart so the 8-B reads of one of
    // them touch every bank). Face strides chosen against bank conflicts of the warp-local line tasks
    // (lane = face fo, line l; faces stored by their ordinal, fslot): FSD mod 16 = TSEL makes the t1-line
    // passes (lane-varying offset FSD fo + N l) conflict-free and the t2-line pass (FSD fo + l) at most
    // 2-way; the same for the 8-B line buffers (FB)
    static constexpr int TSEL = N == 2 ? 2 : (N == 3 ? 9 : (N == 4 ? 3 : (N == 5 ? 9 : 7)));
    static constexpr int pad16(int base) { return base % 16 == TSEL ? base : pad16(base + 1); }
    static constexpr int FSD = pad16(4 * N2);          // doubles per face slot
    static constexpr int FB = pad16(N2);               // doubles per face in the line buffers
    static constexpr int WCSZ = AFFINE ? (FACE_LINES ? 2 * NF * FB : 3 * NF * N2) : 0;
    static constexpr int RX = XS + 2 * NC * N3;                         // ring blocks, aliased by W / CG after P1
    static constexpr int RXEND = RX + (RXSZ > WCSZ ? RXSZ : WCSZ);
    static constexpr int GE = (RXEND + 1) / 2 * 2;                      // [2][NCG][GREC] geometry records
    // G0 / G1: [j2][cell][j0 + N j1] with the j2 stride padded (S0, S1) so that the d = 0 (G0) and d = 1 (G1)
    // line accesses of a half-warp spread over the banks
    static constexpr int P0 = N == 3 ? 10 : (N <= 6 ? 1 : 0);
    static constexpr int P1 = N == 2 ? 2 : (N == 3 ? 11 : (N == 4 ? 4 : (N == 5 ? 13 : (N == 6 ? 6 : 0))));
    static constexpr int S0 = NC * N2 + P0, S1 = NC * N2 + P1;
    static constexpr int G01 = GE + (AFFINE ? 2 * NCG * GREC : 0);      // G0 [N][S0], G1 [N][S1]: grad0/1 -> Q0/1 -> R0/1
    static constexpr int TRB = (G01 + N * (S0 + S1) + 1) / 2 * 2;                       // [NF][u|V, gn|G][side][N2] (+ pad)
    static constexpr int CX = (TRB + NF * FSD + 1) / 2 * 2;             // [2][NC][CXSZ] c(x) factor tables (volume; 16-B pairs)
    static constexpr int CF = CX + (COEFF ? 2 * NC * CXSZ : 0);         // [2][NCG][CFSZ] c(x) at upper-face points
    static constexpr int END = CF + (COEFF ? 2 * NCG * CFSZ : 0);
    static constexpr int BYTES = END * 8 + 64; // + 2 mbarriers
    static_assert(AFFINE || true, "");
};

} // namespace gn

// c(x) factor tables, once at setup (reading R13, c = 1 + 0.5 sin(2 pi x0) cos(2 pi x1) at the mapped
// points x = o_T + J_T xi): per cell of the L+2 planes (plane_begin-1 .. plane_begin+L, the
// jac / geo layout), E'_kb(q) = exp(2 pi i (J_kb xi_q + [b = 0] o_k)), k = 0, 1, b = 0..2, q = 0..N
// (xi_N = 1: the upper faces), stored as (cos, sin) pairs: [cell][k][b][q][2].
struct XiTab {
    double xi[9];
};
template <int N>
__global__ void k_ctab(const double* __restrict__ jac, double* __restrict__ out, long long ncell, const MeshArgs M,
                       const XiTab X)
{
    constexpr int NEN = 2 * 3 * (N + 1);
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncell * NEN) return;
    const long long c = t / NEN;
    const int e = (int)(t % NEN), k = e / (3 * (N + 1)), b = (e / (N + 1)) % 3, q = e % (N + 1);
    const int pl = (int)(c / M.plane_cells), rem = (int)(c % M.plane_cells), i1 = rem / M.N2;
    double Jkb;
    if (jac) Jkb = jac[c * 9 + 3 * k + b];
    else Jkb = (b == k) ? M.h[k] : 0.0;
    double ph = Jkb * X.xi[q];
    if (b == 0) {
        int g0 = (M.plane_begin - 1 + pl) % M.N0;
        if (g0 < 0) g0 += M.N0;
        ph += k == 0 ? (double)g0 / M.N0 : (double)i1 / M.N1;
    }
    double sv, cv;
    sincospi(2.0 * ph, &sv, &cv);
    out[t * 2] = cv;
    out[t * 2 + 1] = sv;
}

// c(x) at the points of each cell's 3 upper faces (reading R12: c_F = c(x_F) at the T- mapped point
// x_F = o_T + J_T xi, xi_d = 1, tangential Gauss nodes), once at setup: [cell][CFSZ], face d at d N^2.
template <int N>
__global__ void k_cface(const double* __restrict__ jac, double* __restrict__ out, long long ncell, const MeshArgs M,
                        const XiTab X)
{
    constexpr int N2 = N * N, CFSZ = (3 * N2 + 1) / 2 * 2;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncell * CFSZ) return;
    const long long c = t / CFSZ;
    const int e = (int)(t % CFSZ);
    if (e >= 3 * N2) { out[t] = 0.0; return; }
    const int d = e / N2, p = e % N2, a = p % N, b = p / N;
    const int pl = (int)(c / M.plane_cells), rem = (int)(c % M.plane_cells), i1 = rem / M.N2;
    int g0 = (M.plane_begin - 1 + pl) % M.N0;
    if (g0 < 0) g0 += M.N0;
    double xi[3];
    xi[d] = 1.0;
    xi[d == 0 ? 1 : 0] = X.xi[a];
    xi[d == 2 ? 1 : 2] = X.xi[b];
    double x0, x1;
    if (jac) {
        const double* J = jac + c * 9;
        x0 = (double)g0 / M.N0 + J[0] * xi[0] + J[1] * xi[1] + J[2] * xi[2];
        x1 = (double)i1 / M.N1 + J[3] * xi[0] + J[4] * xi[1] + J[5] * xi[2];
    } else {
        x0 = (g0 + xi[0]) * M.h[0];
        x1 = (i1 + xi[1]) * M.h[1];
    }
    out[t] = 1.0 + 0.5 * sinpi(2.0 * x0) * cospi(2.0 * x1);
}

// Halo traces of a slab (dg_pack_halo, SURVEY §8(e) traces-only payload): for every cell of the slab's first
// plane the lower-end traces (e0.x, d0.x) of its d = 0 lines, for its last plane the upper-end traces (e1.x,
// d1.x) — the 1-point face tables of, computed with the same even/odd line algebra as k_gen so that a
// neighbour consuming them reproduces the block-halo result bit for bit. Layout per cell: u[N2] then d_0 u[N2],
// point p = j1 + N j2 (the d = 0 face point order of the kernels).
template <int N>
__global__ void k_pack_traces(const double* __restrict__ x, double* __restrict__ lo, double* __restrict__ hi, int plane_cells,
                              int L, const EOTab<N> E)
{
    constexpr int N2 = N * N, N3 = N * N * N, H = EOTab<N>::H, HE = EOTab<N>::HE;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2LL * plane_cells * N2) return;
    const int side = (int)(t / ((long long)plane_cells * N2)); // 0: first plane -> lo, 1: last plane -> hi
    const long long rem = t - (long long)side * plane_cells * N2;
    const long long c = rem / N2;
    const int p = (int)(rem - c * N2), a = p % N, b = p / N;
    const double* blk = x + ((long long)(side ? L - 1 : 0) * plane_cells + c) * N3;
    double v[N];
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = blk[pidx<N>(0, j, a, b)];
    double xe[HE], xo[H > 0 ? H : 1];
    gn::split<N>(v, xe, xo);
    double ulo, glo, uhi, ghi;
    gn::traces<N>(E, xe, xo, ulo, glo, uhi, ghi);
    double* o = (side ? hi : lo) + c * 2 * N2;
    o[p] = side ? uhi : ulo;
    o[N2 + p] = side ? ghi : glo;
}

#ifdef DG_GEN_TRACE
// phase timestamps (experiments only): [block < 1024][step < 16][8] clock64 values, thread 0
__device__ long long* g_gen_dbg = nullptr;
#define GEN_STAMP(ph)                                                                                              \
    do {                                                                                                           \
        if (tid == 0 && g_gen_dbg && blockIdx.x < 1024 && s < 16) g_gen_dbg[(blockIdx.x * 16 + s) * 8 + (ph)] = clock64(); \
    } while (0)
#else
#define GEN_STAMP(ph) do { } while (0)
#endif

// grid: ntiles * nchunks CTAs (chunk-major), block Lay::NT, dynamic smem Lay::BYTES
template <int N, bool AFFINE, bool COEFF, int T1, int T2, int MINB>
__global__ void __launch_bounds__(gn::Lay<N, AFFINE, COEFF, T1, T2>::NT, MINB)
k_gen(const double* __restrict__ x, const double* __restrict__ xb, const double* __restrict__ xa, double* __restrict__ r,
      int p_begin, int p_end, int chunk_len, int halo_tr, const EOTab<N> E, const MeshArgs M, const double* __restrict__ geo,
      const double* __restrict__ ctab, const double* __restrict__ cface)
{
    using Y = gn::Lay<N, AFFINE, COEFF, T1, T2>;
    constexpr int N2 = Y::N2, N3 = Y::N3, NC = Y::NC, NT = Y::NT, NRL = Y::NRL, NRH = Y::NRH, NF = Y::NF;
    constexpr int NCG = Y::NCG, CXSZ = Y::CXSZ, CFSZ = Y::CFSZ;
    constexpr int H = EOTab<N>::H, HE = EOTab<N>::HE;
    // axis-aligned with c = 1: stage 1 -> 2 -> 3 along a direction collapses into the 1D SIPG line
    // operator B^ with neighbour-trace couplings (exact reordering, see kernel_axis8.cuh)
    constexpr bool LINEOP = !AFFINE && !COEFF;
    extern __shared__ __align__(16) double sm[];
    double* const XS = sm + Y::XS;
    double* const RX = sm + Y::RX;
    double* const BX = sm + Y::RX;           // face buffers (AFFINE, after P1, aliasing the ring blocks):
    constexpr int FSD = Y::FSD, FB = Y::FB;
    double* const BY = sm + Y::RX + NF * FB; // BX: w2 -> Cg, BY: D_t1 w1 -> D_t2^T Cg, [NF][FB]
    double* const PW = sm + Y::RX;              // point passes: W [NF][2][N2]
    double* const PCG = sm + Y::RX + 2 * NF * N2; //              Cg [NF][N2]
    constexpr bool FACE_LINES = Y::FACE_LINES;
    double* const GE = sm + Y::GE;
    double* const G0 = sm + Y::G01;
    double* const G1 = sm + Y::G01 + N * Y::S0;
    double* const TRB = sm + Y::TRB;
    double* const CX = sm + Y::CX;
    double* const CF = sm + Y::CF;
    uint64_t* const barA = reinterpret_cast<uint64_t*>(sm + Y::END);
    uint64_t* const barB = barA + 1;
    __shared__ double sXi[N + 1], sD[N * N], sW[N];

    const int tid = threadIdx.x;
    const int passb_t = gn::passb_task<N>(tid & 31); // warp-local face pass B lane order
    const int ntile2 = M.N2 / T2;
    const int ntiles = (M.N1 / T1) * ntile2;
    const int chunk = blockIdx.x / ntiles, tile = blockIdx.x % ntiles;
    const int ti1 = tile / ntile2, ti2 = tile % ntile2;
    {
        const int b = p_begin + chunk * chunk_len;
        p_end = min(p_end, b + chunk_len);
        p_begin = b;
    }
    const int nsteps = p_end - p_begin;
    if (nsteps <= 0) return;
    const int PC = M.plane_cells;
    auto wrap = [](int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); };
    auto cidx = [&](int lp, int i1, int i2) -> long long { return (long long)lp * PC + (long long)i1 * M.N2 + i2; };
    // source of plane lp's blocks (-1: halo below, L: halo above), and of its geometry records (L+2 planes from -1)
    auto xplane = [&](int lp) -> const double* { return lp < 0 ? xb : (lp >= M.L ? xa : x + (long long)lp * PC * N3); };
    // halo_tr bit 0 / 1: the halo plane below / above is given as its face traces only (dg_apply_planes_tr): per
    // cell of the plane, u[N2] then d_0 u[N2] at the d = 0 face points (upper end below, lower end above)
    auto is_tr = [&](int lp) { return (lp < 0 && (halo_tr & 1)) || (lp >= M.L && (halo_tr & 2)); };
    auto grec = [&](int lp, int i1, int i2) -> const double* { return geo + (cidx(lp + 1, i1, i2)) * GREC; };
    // face slots: (u, gn) -> (V, G) pairs per face f, side (0: T-, 1: T+), point p
    // TRp(f, side)[p]: (.x = u / V, .y = gn / G) of face f, side, point p, stored in separate arrays
    // storage slot of face f (own faces 3 c + d, ring faces 3 NC + r): its ordinal d NC + c / 3 NC + r, so
    // the faces of a warp's line tasks occupy consecutive slots
    auto fslot = [&](int f) { return f < 3 * NC ? (f % 3) * NC + f / 3 : f; };
    auto TRp = [&](int f, int side) {
        const int o = fslot(f);
        DG_CHECK(f >= 0 && f < NF && o >= 0 && o < NF && (side == 0 || side == 1));
        return gn::TRView{TRB + o * FSD + side * N2, TRB + o * FSD + (2 + side) * N2};
    };

    // the thread that issues the bulk copies: the last one (no stage-2 point, no face line for n >= 4), off
    // the critical path of the face phase
    constexpr int PROD = Y::NACT < NT ? NT - 1 : 0;
    // fixed thread coordinates: cell mc of the tile, line position (ma, mb)
    const bool act = tid < Y::NACT;
    const int mc = act ? tid / N2 : 0, mab = act ? tid % N2 : 0, ma = mab % N, mb = mab / N;
    const int mc1 = mc / T2, mc2 = mc % T2;
    // TR face index of the own cell's lower faces d = 1, 2 (in-tile: upper face of the cell below)
    const int flo1 = mc1 > 0 ? 3 * (mc - T2) + 1 : 3 * NC + mc2;
    const int flo2 = mc2 > 0 ? 3 * (mc - 1) + 2 : 3 * NC + T2 + mc1;
    // G0 / G1 layout [j2][cell][j0 + N j1]: the d = 2 line points of consecutive threads are consecutive
    // (conflict-free stage 2 and final sum); index of point j on the thread's d-line of its cell
    auto gixs = [&](int S, int d, int j) -> int {
        return d == 0 ? mb * S + mc * N2 + j + N * ma : (d == 1 ? mb * S + mc * N2 + ma + N * j : j * S + mc * N2 + mab);
    };
    auto gix0 = [&](int d, int j) { const int i = gixs(Y::S0, d, j); DG_CHECK(i >= 0 && i < N * Y::S0); return i; }; // G0 index
    auto gix1 = [&](int d, int j) { const int i = gixs(Y::S1, d, j); DG_CHECK(i >= 0 && i < N * Y::S1); return i; }; // G1 index

    if (tid < N) { sXi[tid] = E.xi[tid]; sW[tid] = E.w[tid]; }
    for (int i = tid; i < N * N; i += NT) sD[i] = E.D[i];
    if (tid == 0) {
        sXi[N] = 1.0;
        gn::mbar_init(barA, 1);
        gn::mbar_init(barB, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // ---------------- async staging ----------------
    constexpr uint32_t ROWB = T2 * N3 * 8;
    constexpr uint32_t ROWT = T2 * 2 * N2 * 8; // a tile row of halo traces
    auto xbytes = [&](int lp) -> uint32_t { return is_tr(lp) ? T1 * ROWT : T1 * ROWB; };
    auto issue_x = [&](int lp, double* dst) { // own blocks (or halo traces) of plane lp (T1 rows) on barA (caller: expect_tx)
        const double* src = xplane(lp);
        DG_CHECK(lp >= -1 && lp <= M.L && dst >= XS && dst + NC * N3 <= XS + 2 * NC * N3);
        DG_CHECK((ti1 + 1) * T1 <= M.N1 && (ti2 + 1) * T2 <= M.N2);
        if (is_tr(lp)) {
#pragma unroll
            for (int c1 = 0; c1 < T1; ++c1)
                gn::bulk_g2s(dst + c1 * T2 * 2 * N2, src + ((long long)(ti1 * T1 + c1) * M.N2 + ti2 * T2) * 2 * N2, ROWT, barA);
            return;
        }
#pragma unroll
        for (int c1 = 0; c1 < T1; ++c1)
            gn::bulk_g2s(dst + c1 * T2 * N3, src + ((long long)(ti1 * T1 + c1) * M.N2 + ti2 * T2) * N3, ROWB, barA);
    };
    // records (AFFINE) and c(x) factor tables (COEFF) of own + ring-below cells of plane lp into buffer `buf`
    auto issue_geo = [&](int lp, int buf) {
        DG_CHECK(lp >= -1 && lp <= M.L - 1 && (buf == 0 || buf == 1));
        auto rows = [&](const double* base, int per, double* dst, bool ring) {
            auto at = [&](int i1, int i2) { return base + cidx(lp + 1, i1, i2) * per; };
#pragma unroll
            for (int c1 = 0; c1 < T1; ++c1) gn::bulk_g2s(dst + c1 * T2 * per, at(ti1 * T1 + c1, ti2 * T2), T2 * per * 8, barA);
            if (!ring) return;
            gn::bulk_g2s(dst + NC * per, at(wrap(ti1 * T1 - 1, M.N1), ti2 * T2), T2 * per * 8, barA);
#pragma unroll
            for (int c1 = 0; c1 < T1; ++c1)
                gn::bulk_g2s(dst + (NC + T2 + c1) * per, at(ti1 * T1 + c1, wrap(ti2 * T2 - 1, M.N2)), per * 8, barA);
        };
        if (AFFINE) rows(geo, GREC, GE + buf * NCG * GREC, true);
        if (COEFF) {
            rows(ctab, CXSZ, CX + buf * NC * CXSZ, false);
            rows(cface, CFSZ, CF + buf * NCG * CFSZ, true);
        }
    };
    constexpr uint32_t GEOB = (AFFINE ? (uint32_t)(NCG * GREC * 8) : 0u) + (COEFF ? (uint32_t)((NC * CXSZ + NCG * CFSZ) * 8) : 0u);
    // ring blocks of plane lp: bulk copies on barB (one thread); d = 2 ring cells singly (even n^3) or as aligned pairs
    constexpr int SL = Y::SL;
    auto ring_b2 = [&](int c1) { return RX + (Y::RB2 + SL * c1 + (SL - 1)) * N3; }; // ring cell below (i2) of tile row c1
    auto ring_a2 = [&](int c1) { return RX + (Y::RA2 + SL * c1) * N3; };            // ring cell above (i2) of tile row c1
    auto issue_ring_bulk = [&](int lp) {
        DG_CHECK(lp >= 0 && lp < M.L);
        const double* src = x + (long long)lp * PC * N3;
        const uint32_t bytes = 2 * ROWB + 2 * T1 * SL * N3 * 8;
        gn::mbar_expect_tx(barB, bytes);
        gn::bulk_g2s(RX + Y::RB1 * N3, src + ((long long)wrap(ti1 * T1 - 1, M.N1) * M.N2 + ti2 * T2) * N3, ROWB, barB);
        gn::bulk_g2s(RX + Y::RA1 * N3, src + ((long long)wrap(ti1 * T1 + T1, M.N1) * M.N2 + ti2 * T2) * N3, ROWB, barB);
#pragma unroll
        for (int c1 = 0; c1 < T1; ++c1) {
            const long long i1 = ti1 * T1 + c1;
            gn::bulk_g2s(RX + (Y::RB2 + SL * c1) * N3, src + (i1 * M.N2 + wrap(ti2 * T2 - SL, M.N2)) * N3, SL * N3 * 8, barB);
            gn::bulk_g2s(RX + (Y::RA2 + SL * c1) * N3, src + (i1 * M.N2 + wrap(ti2 * T2 + T2, M.N2)) * N3, SL * N3 * 8, barB);
        }
    };

    const double* cxcur = CX; // c(x) factor tables of the plane being evaluated (set per step)
    const double* cfcur = CF; // c(x) at the upper-face points of its own / ring-below cells
    // ---------------- face passes (face f with normal DC, point p = (a, b)) ----------------
    // the T- record slot of face f: own upper faces 3c + d -> c, tile-boundary faces 3 NC + r -> NC + r
    auto face_rec = [&](int f) { return f < 3 * NC ? f / 3 : NC + (f - 3 * NC); };
    // 1/h_d once (axis-aligned faces: no double division per face point)
    const double ihx0 = 1.0 / M.h[0], ihx1 = 1.0 / M.h[1], ihx2 = 1.0 / M.h[2];
    // a-, a+ components (normal d, tangential t1, t2) and dS of face f from its T- record (16-B pairs)
    struct FaceA {
        double mdn, mt1, mt2, pdn, pt1, pt2, dS;
    };
    auto face_a = [&](auto DC, const double* gb, int f) -> FaceA {
        const int d = DC.value; // compile-time for integral_constant, runtime for RunD
        FaceA A;
        if (AFFINE) {
            // record pairs (a-_t1, a+_t1) (a-_t2, a+_t2) (a-_d, a+_d) (dS, 0): pass A reads the first two,
            // pass B the last two, pass C the first three
            const double2* fr = reinterpret_cast<const double2*>(gb + face_rec(f) * GREC + 12 + 8 * d);
            const double2 r0 = fr[0], r1 = fr[1], r2 = fr[2], r3 = fr[3];
            A.mt1 = r0.x;
            A.pt1 = r0.y;
            A.mt2 = r1.x;
            A.pt2 = r1.y;
            A.mdn = r2.x;
            A.pdn = r2.y;
            A.dS = r3.x;
        } else {
            A.mdn = A.pdn = d == 0 ? ihx0 : (d == 1 ? ihx1 : ihx2);
            A.mt1 = A.mt2 = A.pt1 = A.pt2 = 0.0;
            A.dS = M.h[(d + 1) % 3] * M.h[(d + 2) % 3];
        }
        return A;
    };
    // ---- affine faces, one thread per face point (used when the line tasks would leave threads idle) ----
    // pass A (AFFINE): w1 = a-_t1 u- + a+_t1 u+, w2 = a-_t2 u- + a+_t2 u+
    auto ptA = [&](auto DC, const double* gb, int f, int p, const double*, const double*) {
        const FaceA A = face_a(DC, gb, f);
        const double um = TRp(f, 0)[p].x, up = TRp(f, 1)[p].x;
        PW[(f * 2 + 0) * N2 + p] = fma(A.mt1, um, A.pt1 * up);
        PW[(f * 2 + 1) * N2 + p] = fma(A.mt2, um, A.pt2 * up);
    };
    // pass B: flux. AFFINE: Cv- -> TR(f,0).x, Cg -> CG. Axis: (V, G) of both sides directly.
    // Ra, Rb: rows a, b of D (registers for the thread's own faces)
    auto ptB = [&](auto DC, const double* gb, int f, int p, const double* Ra, const double* Rb) {
        const int d = DC.value; // compile-time for integral_constant, runtime for RunD
        const int a = p % N, b = p / N;
        const FaceA A = face_a(DC, gb, f);
        const double cF = COEFF ? cfcur[face_rec(f) * CFSZ + d * N2 + p] : 1.0; // c at x_F on T- (R12)
        const double2 m = TRp(f, 0)[p], pl = TRp(f, 1)[p];
        double s = fma(A.mdn, m.y, A.pdn * pl.y);
        if (AFFINE) {
            const double* W1 = PW + (f * 2 + 0) * N2 + N * b;
            const double* W2 = PW + (f * 2 + 1) * N2 + a;
#pragma unroll
            for (int k = 0; k < N; ++k) {
                s = fma(Ra[k], W1[k], s);
                s = fma(Rb[k], W2[N * k], s);
            }
        }
        const double Wt = sW[a] * sW[b] * A.dS;
        const double jump = m.x - pl.x;
        const double avg = 0.5 * cF * s;
        const double Cvm = Wt * fma(M.gamma[d], jump, -avg);
        const double Cg = -0.5 * Wt * jump * cF;
        if (AFFINE) {
            TRp(f, 0)[p].x = Cvm;
            PCG[f * N2 + p] = Cg;
        } else {
            TRp(f, 0)[p] = make_double2(Cvm, A.mdn * Cg);
            TRp(f, 1)[p] = make_double2(-Cvm, A.pdn * Cg);
        }
    };
    // pass C (AFFINE): V+- = +-Cv- + a+-_t1 (D^T_t1 Cg) + a+-_t2 (D^T_t2 Cg), G+- = a+-_d Cg
    // Ca, Cb: columns a, b of D
    auto ptC = [&](auto DC, const double* gb, int f, int p, const double* Ca, const double* Cb) {
        const int a = p % N, b = p / N;
        const FaceA A = face_a(DC, gb, f);
        const double* C1 = PCG + f * N2 + N * b;
        const double* C2 = PCG + f * N2 + a;
        double t1 = 0.0, t2 = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            t1 = fma(Ca[k], C1[k], t1);
            t2 = fma(Cb[k], C2[N * k], t2);
        }
        const double Cvm = TRp(f, 0)[p].x, Cg = PCG[f * N2 + p];
        TRp(f, 0)[p] = make_double2(fma(A.mt1, t1, fma(A.mt2, t2, Cvm)), A.mdn * Cg);
        TRp(f, 1)[p] = make_double2(fma(A.pt1, t1, fma(A.pt2, t2, -Cvm)), A.pdn * Cg);
    };
    // all faces of the plane step: the thread's 3 upper faces (fixed point, D rows / columns in
    // registers) + the tile-boundary lower faces. COLS: pass C wants columns of D, pass B rows.
    auto pt_faces = [&](auto pass, auto COLS, const double* gb) {
        constexpr bool cols = decltype(COLS)::value;
        if (act) {
            double Ra[N], Rb[N];
            if (AFFINE) {
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    Ra[k] = cols ? sD[k * N + ma] : sD[ma * N + k];
                    Rb[k] = cols ? sD[k * N + mb] : sD[mb * N + k];
                }
            }
            pass(std::integral_constant<int, 0>{}, gb, 3 * mc + 0, mab, Ra, Rb);
            pass(std::integral_constant<int, 1>{}, gb, 3 * mc + 1, mab, Ra, Rb);
            pass(std::integral_constant<int, 2>{}, gb, 3 * mc + 2, mab, Ra, Rb);
        }
        for (int t = tid; t < NRL * N2; t += NT) {
            const int rr = t / N2, p = t - rr * N2, a = p % N, b = p / N;
            double Ra[N], Rb[N];
            if (AFFINE) {
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    Ra[k] = cols ? sD[k * N + a] : sD[a * N + k];
                    Rb[k] = cols ? sD[k * N + b] : sD[b * N + k];
                }
            }
            if (rr < T2) pass(std::integral_constant<int, 1>{}, gb, 3 * NC + rr, p, Ra, Rb);
            else pass(std::integral_constant<int, 2>{}, gb, 3 * NC + rr, p, Ra, Rb);
        }
    };

    // ---- affine faces, one thread per face line (N points), tangential contractions as even/odd sweeps ----
    // line A (t1-line b): w1 = a-_t1 u- + a+_t1 u+ -> BY = D_t1 w1;  w2 = a-_t2 u- + a+_t2 u+ -> BX
    auto lineA = [&](auto DC, const double* gb, int f, int b) {
        const FaceA A = face_a(DC, gb, f);
        double w1[N];
#pragma unroll
        for (int a = 0; a < N; ++a) {
            const int p = a + N * b;
            const double um = TRp(f, 0)[p].x, up = TRp(f, 1)[p].x;
            w1[a] = fma(A.mt1, um, A.pt1 * up);
            BX[fslot(f) * FB + p] = fma(A.mt2, um, A.pt2 * up);
        }
        double xe[HE], xo[H > 0 ? H : 1], y[N];
        gn::split<N>(w1, xe, xo);
        gn::sweep<N, false, false>(E, xe, xo, y);
#pragma unroll
        for (int a = 0; a < N; ++a) BY[fslot(f) * FB + a + N * b] = y[a];
    };
    // line B (t2-line a): {c grad u . n} = c_F/2 (a-_d gn- + a+_d gn+ + D_t1 w1 + D_t2 w2), SIPG flux
    // (Eq. diffreac_weak, theta = -1): Cv- -> TR(f,0).x, Cg -> BX, D_t2^T Cg -> BY
    auto lineB = [&](auto DC, const double* gb, int f, int a) {
        const int d = DC.value; // compile-time for integral_constant, runtime for RunD
        const FaceA A = face_a(DC, gb, f);
        double w2[N];
#pragma unroll
        for (int k = 0; k < N; ++k) w2[k] = BX[fslot(f) * FB + a + N * k];
        double xe[HE], xo[H > 0 ? H : 1], s2[N];
        gn::split<N>(w2, xe, xo);
        gn::sweep<N, false, false>(E, xe, xo, s2);
        double cg[N];
        const double wa = sW[a];
#pragma unroll
        for (int b = 0; b < N; ++b) {
            const int p = a + N * b;
            const double2 m = TRp(f, 0)[p], pl = TRp(f, 1)[p];
            const double s = fma(A.mdn, m.y, fma(A.pdn, pl.y, BY[fslot(f) * FB + p] + s2[b]));
            const double cF = COEFF ? cfcur[face_rec(f) * CFSZ + d * N2 + p] : 1.0; // c at x_F on T- (R12)
            const double Wt = wa * sW[b] * A.dS;
            const double jump = m.x - pl.x;
            TRp(f, 0)[p].x = Wt * fma(d == 0 ? M.gamma[0] : (d == 1 ? M.gamma[1] : M.gamma[2]), jump, -0.5 * cF * s);
            cg[b] = -0.5 * Wt * jump * cF;
        }
        double t2[N];
        gn::split<N>(cg, xe, xo);
        gn::sweep<N, true, false>(E, xe, xo, t2);
#pragma unroll
        for (int b = 0; b < N; ++b) {
            BX[fslot(f) * FB + a + N * b] = cg[b];
            BY[fslot(f) * FB + a + N * b] = t2[b];
        }
    };
    // line C (t1-line b): V+- = +-Cv- + a+-_t1 D_t1^T Cg + a+-_t2 D_t2^T Cg, G+- = a+-_d Cg
    auto lineC = [&](auto DC, const double* gb, int f, int b) {
        const FaceA A = face_a(DC, gb, f);
        double cg[N];
#pragma unroll
        for (int k = 0; k < N; ++k) cg[k] = BX[fslot(f) * FB + k + N * b];
        double xe[HE], xo[H > 0 ? H : 1], t1[N];
        gn::split<N>(cg, xe, xo);
        gn::sweep<N, true, false>(E, xe, xo, t1);
#pragma unroll
        for (int a = 0; a < N; ++a) {
            const int p = a + N * b;
            const double Cvm = TRp(f, 0)[p].x, t2 = BY[fslot(f) * FB + p];
            TRp(f, 0)[p] = make_double2(fma(A.mt1, t1[a], fma(A.mt2, t2, Cvm)), A.mdn * cg[a]);
            TRp(f, 1)[p] = make_double2(fma(A.pt1, t1[a], fma(A.pt2, t2, -Cvm)), A.pdn * cg[a]);
        }
    };
    // the plane step's faces as line tasks, grouped by direction (ordinal o: own d=0, d=1, d=2 faces,
    // then the tile-boundary lower faces d=1, d=2); nf0 = NC restricts to the d=0 own faces (prologue)
    // OFAST: consecutive threads take the same line of consecutive faces (t1-line passes A, C);
    // otherwise consecutive lines of one face (t2-line pass B) — both bank-conflict free with FS
    auto face_lines = [&](auto line, auto OFAST, const double* gb, int nfo) {
        constexpr bool of = decltype(OFAST)::value;
        for (int t = tid; t < nfo * N; t += NT) {
            int g0, G;
            if (t < NC * N) { g0 = 0; G = NC; }
            else if (t < 2 * NC * N) { g0 = NC; G = NC; }
            else if (t < 3 * NC * N) { g0 = 2 * NC; G = NC; }
            else if (t < (3 * NC + T2) * N) { g0 = 3 * NC; G = T2; }
            else { g0 = 3 * NC + T2; G = T1; }
            const int u = t - g0 * N;
            const int oo = of ? u % G : u / N, l = of ? u / G : u % N;
            const int o = g0 + oo;
            if (o < NC) line(std::integral_constant<int, 0>{}, gb, 3 * o, l);
            else if (o < 2 * NC) line(std::integral_constant<int, 1>{}, gb, 3 * (o - NC) + 1, l);
            else if (o < 3 * NC) line(std::integral_constant<int, 2>{}, gb, 3 * (o - 2 * NC) + 2, l);
            else if (o < 3 * NC + T2) line(std::integral_constant<int, 1>{}, gb, o, l);
            else line(std::integral_constant<int, 2>{}, gb, o, l);
        }
    };
    // warp-local face phase (affine, n <= 5): the N lines of a face are N consecutive lanes of one warp, so
    // passes A -> B -> C of a face need only __syncwarp (no CTA barriers between them); the face direction
    // is a run-time value (faces of several directions share a warp)
    auto face_warp = [&](const double* gb) {
        // n = 6: whole faces per half-warp (2 x 2 faces, lanes 12-15 idle) — with FSD = 7 mod 16 every pass
        // is bank-conflict free; otherwise 32 / n faces on consecutive lanes
        constexpr bool HALF = N == 6;
        constexpr int FPH = 16 / N;
        constexpr int FPW = HALF ? 2 * FPH : 32 / N; // faces per warp and round
        constexpr int NWARP = NT / 32;
        const int warp = tid >> 5, lane = tid & 31;
        const int hl = HALF ? (lane & 15) : lane;
        const int fo = HALF ? (lane >> 4) * FPH + hl / N : lane / N;
        const int l = hl - (hl / N) * N;
        const bool lane_on = HALF ? hl < FPH * N : lane < FPW * N;
        // pass B (t2-lines, lane offsets FSD fo + l) under the lane order of passes A / C is 2-way bank conflicted;
        // its own lane -> (face, line) order (searched offline: one half-warp with distinct FSD fo + l mod 16, the
        // other with at most two 2-way pairs) serves the same warp-local tasks: 3 wavefronts instead of 4
        const int tb = passb_t;
        const int foB = HALF ? fo : (tb >= 0 ? tb / N : 0), lB = HALF ? l : (tb >= 0 ? tb - (tb / N) * N : 0);
        const bool onB_lane = HALF ? lane_on : tb >= 0;
        auto face_of = [&](int o, int& f, int& d) {
            if (o < NC) { f = 3 * o; d = 0; }
            else if (o < 2 * NC) { f = 3 * (o - NC) + 1; d = 1; }
            else if (o < 3 * NC) { f = 3 * (o - 2 * NC) + 2; d = 2; }
            else { f = o; d = (o < 3 * NC + T2) ? 1 : 2; }
        };
        for (int base = 0; base < NF; base += FPW * NWARP) {
            const int o = base + warp * FPW + fo;
            const bool on = lane_on && o < NF;
            int f = 0, d = 0;
            if (on) face_of(o, f, d);
            const gn::RunD DC{d};
            const int oB = base + warp * FPW + foB;
            const bool onB = onB_lane && oB < NF;
            int fB = 0, dB = 0;
            if (onB) face_of(oB, fB, dB);
            if (on) lineA(DC, gb, f, l);
            __syncwarp();
            if (onB) lineB(gn::RunD{dB}, gb, fB, lB);
            __syncwarp();
            if (on) lineC(DC, gb, f, l);
            __syncwarp();
        }
    };
    // axis-aligned faces (no tangential terms): flux per point, (V, G) of both sides directly
    auto passB = [&](auto DC, const double* gb, int f, int p, const double*, const double*) {
        const int d = DC.value; // compile-time for integral_constant, runtime for RunD
        const int a = p % N, b = p / N;
        const FaceA A = face_a(DC, gb, f);
        const double cF = COEFF ? cfcur[face_rec(f) * CFSZ + d * N2 + p] : 1.0;
        const double2 m = TRp(f, 0)[p], pl = TRp(f, 1)[p];
        const double s = fma(A.mdn, m.y, A.pdn * pl.y);
        const double Wt = sW[a] * sW[b] * A.dS;
        const double jump = m.x - pl.x;
        const double Cvm = Wt * fma(M.gamma[d], jump, -0.5 * cF * s);
        const double Cg = -0.5 * Wt * jump * cF;
        TRp(f, 0)[p] = make_double2(Cvm, A.mdn * Cg);
        TRp(f, 1)[p] = make_double2(-Cvm, A.pdn * Cg);
    };
    // axis-aligned faces of the plane step: the thread's 3 upper faces + the tile-boundary lower faces
    auto all_faces = [&](auto pass, const double* gb) {
        if (act) {
            pass(std::integral_constant<int, 0>{}, gb, 3 * mc + 0, mab, nullptr, nullptr);
            pass(std::integral_constant<int, 1>{}, gb, 3 * mc + 1, mab, nullptr, nullptr);
            pass(std::integral_constant<int, 2>{}, gb, 3 * mc + 2, mab, nullptr, nullptr);
        }
        for (int t = tid; t < NRL * N2; t += NT) {
            const int rr = t / N2, p = t - rr * N2;
            if (rr < T2) pass(std::integral_constant<int, 1>{}, gb, 3 * NC + rr, p, nullptr, nullptr);
            else pass(std::integral_constant<int, 2>{}, gb, 3 * NC + rr, p, nullptr, nullptr);
        }
    };

    // foreign traces: ring cells (their ends facing the tile) and the next plane's lower ends,
    // grouped by line direction (d = 1: rings along i1, d = 2: rings along i2, d = 0: next plane)
    auto trace_task = [&](auto DC, const double* blk, int p, int f, int side) {
        const int d = DC.value; // compile-time for integral_constant, runtime for RunD
        const int a = p % N, b = p / N;
        double v[N];
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = blk[pidx<N>(d, j, a, b)];
        double xe[HE], xo[H > 0 ? H : 1];
        gn::split<N>(v, xe, xo);
        double ulo, glo, uhi, ghi;
        gn::traces<N>(E, xe, xo, ulo, glo, uhi, ghi);
        TRp(f, side)[p] = side ? make_double2(ulo, glo) : make_double2(uhi, ghi); // T- faces the tile with its upper end
    };
    auto foreign = [&](const double* XN, bool xn_tr) {
        for (int t = tid; t < 2 * T2 * N2; t += NT) {
            const int k = t / N2, p = t - k * N2;
            if (k < T2) trace_task(std::integral_constant<int, 1>{}, RX + (Y::RB1 + k) * N3, p, 3 * NC + k, 0);
            else trace_task(std::integral_constant<int, 1>{}, RX + (Y::RA1 + k - T2) * N3, p, 3 * ((T1 - 1) * T2 + k - T2) + 1, 1);
        }
        for (int t = tid; t < 2 * T1 * N2; t += NT) {
            const int k = t / N2, p = t - k * N2;
            if (k < T1) trace_task(std::integral_constant<int, 2>{}, ring_b2(k), p, 3 * NC + T2 + k, 0);
            else trace_task(std::integral_constant<int, 2>{}, ring_a2(k - T1), p, 3 * ((k - T1) * T2 + T2 - 1) + 2, 1);
        }
        for (int t = tid; t < NC * N2; t += NT) {
            const int q = t / N2, p = t - q * N2;
            if (xn_tr) { // halo above given as traces (u, d_0 u at the lower end)
                const double* tb = XN + q * 2 * N2;
                TRp(3 * q, 1)[p] = make_double2(tb[p], tb[N2 + p]);
            } else {
                trace_task(std::integral_constant<int, 0>{}, XN + q * N3, p, 3 * q, 1);
            }
        }
    };

    // ---------------- prologue: the lower d=0 face of plane p_begin (T- = plane p_begin - 1) ----------------
    double pendV = 0.0, pendG = 0.0; // T+ half of the d=0 face below the thread's line (a, b) of cell mc
    {
        if (tid == PROD) {
            gn::mbar_expect_tx(barA, xbytes(p_begin - 1) + xbytes(p_begin) + GEOB);
            issue_x(p_begin - 1, XS + NC * N3);
            issue_x(p_begin, XS);
            if (AFFINE || COEFF) issue_geo(p_begin - 1, 1);
        }
        gn::mbar_wait(barA, 0);
        cxcur = CX + NC * CXSZ;
        cfcur = CF + NCG * CFSZ;
        // T- upper-end traces (plane p_begin - 1) -> TR(3c, 0), T+ lower-end traces (plane p_begin) -> TR(3c, 1)
        const bool below_tr = is_tr(p_begin - 1);
        for (int t = tid; t < NC * N2; t += NT) {
            const int c = t / N2, p = t - c * N2;
            if (below_tr) { // the halo's traces as received (u, d_0 u at the upper end of each d = 0 line)
                const double* tb = XS + NC * N3 + c * 2 * N2;
                TRp(3 * c, 0)[p] = make_double2(tb[p], tb[N2 + p]);
            } else {
                trace_task(std::integral_constant<int, 0>{}, XS + NC * N3 + c * N3, p, 3 * c, 0);
            }
            trace_task(std::integral_constant<int, 0>{}, XS + c * N3, p, 3 * c, 1);
        }
        if (LINEOP) {
            // the lower neighbour's (e1.x, d1.x) of the thread's d=0 line, from plane p_begin - 1
            if (act && below_tr) {
                const double* tb = XS + NC * N3 + mc * 2 * N2;
                pendV = tb[mab];
                pendG = tb[N2 + mab];
            } else if (act) {
                double v[N];
#pragma unroll
                for (int j = 0; j < N; ++j) v[j] = XS[NC * N3 + mc * N3 + pidx<N>(0, j, ma, mb)];
                double xe[HE], xo[H > 0 ? H : 1];
                gn::split<N>(v, xe, xo);
                double ulo, glo;
                gn::traces<N>(E, xe, xo, ulo, glo, pendV, pendG);
            }
        }
        __syncthreads();
        const double* gb = GE + NCG * GREC;
        if (AFFINE && FACE_LINES) {
            face_lines(lineA, std::true_type{}, gb, NC);
            __syncthreads();
            face_lines(lineB, std::false_type{}, gb, NC);
            __syncthreads();
            face_lines(lineC, std::true_type{}, gb, NC);
            __syncthreads();
        } else if (AFFINE) {
            double Ra[N], Rb[N], Ca[N], Cb[N];
#pragma unroll
            for (int k = 0; k < N; ++k) {
                Ra[k] = sD[ma * N + k];
                Rb[k] = sD[mb * N + k];
                Ca[k] = sD[k * N + ma];
                Cb[k] = sD[k * N + mb];
            }
            if (act) ptA(std::integral_constant<int, 0>{}, gb, 3 * mc, mab, Ra, Rb);
            __syncthreads();
            if (act) ptB(std::integral_constant<int, 0>{}, gb, 3 * mc, mab, Ra, Rb);
            __syncthreads();
            if (act) ptC(std::integral_constant<int, 0>{}, gb, 3 * mc, mab, Ca, Cb);
            __syncthreads();
        } else if (!LINEOP) {
            if (act) passB(std::integral_constant<int, 0>{}, gb, 3 * mc, mab, nullptr, nullptr);
            __syncthreads();
        }
        if (act && !LINEOP) {
            const double2 vg = TRp(3 * mc, 1)[mab];
            pendV = vg.x;
            pendG = vg.y;
        }
        __syncthreads();
        if (tid == PROD) {
            gn::mbar_expect_tx(barA, xbytes(p_begin + 1) + GEOB);
            issue_x(p_begin + 1, XS + NC * N3);
            if (AFFINE || COEFF) issue_geo(p_begin, 0);
            issue_ring_bulk(p_begin);
        }
    }

    for (int s = 0; s < nsteps; ++s) {
        const int lp = p_begin + s;
        const double* XC = XS + (s & 1) * NC * N3;     // own plane lp
        const double* XN = XS + ((s + 1) & 1) * NC * N3; // next plane lp + 1
        const double* gb = GE + (s & 1) * NCG * GREC;
        GEN_STAMP(0);
        gn::mbar_wait(barA, (s + 1) & 1);
        gn::mbar_wait(barB, s & 1);
        __syncthreads();
        GEN_STAMP(1);

        if constexpr (LINEOP) {
            // ---- L1: own line traces (kept lines in registers) + foreign traces ----
            double xe[3][HE], xo[3][H > 0 ? H : 1];
            double nU = 0.0, nG = 0.0;
            if (act) {
                const double* xc = XC + mc * N3;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    double v[N];
#pragma unroll
                    for (int j = 0; j < N; ++j) v[j] = xc[pidx<N>(d, j, ma, mb)];
                    gn::split<N>(v, xe[d], xo[d]);
                    double ulo, glo, uhi, ghi;
                    gn::traces<N>(E, xe[d], xo[d], ulo, glo, uhi, ghi);
                    TRp(3 * mc + d, 0)[mab] = make_double2(uhi, ghi);
                    if (d == 0) { nU = uhi; nG = ghi; }
                    if (d == 1) TRp(flo1, 1)[mab] = make_double2(ulo, glo);
                    if (d == 2) TRp(flo2, 1)[mab] = make_double2(ulo, glo);
                }
            }
            foreign(XN, is_tr(lp + 1));
            __syncthreads();
            if (s + 1 < nsteps) { // own plane buffer and ring buffer are free
                if (tid == PROD) {
                    gn::mbar_expect_tx(barA, xbytes(lp + 2));
                    issue_x(lp + 2, XS + (s & 1) * NC * N3);
                    issue_ring_bulk(lp + 1);
                }
            }
            // ---- L2: line operators; directions 0, 1 -> shared memory, 2 -> registers ----
            double y2[N];
            if (act) {
                const double wab = sW[ma] * sW[mb];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    double uL, gL;
                    if (d == 0) { uL = pendV; gL = pendG; }
                    else { const double2 lo = TRp(d == 1 ? flo1 : flo2, 0)[mab]; uL = lo.x; gL = lo.y; }
                    const double2 hi = TRp(3 * mc + d, 1)[mab];
                    double y[N];
                    gn::lineop<N>(E, xe[d], xo[d], y, uL, gL, hi.x, hi.y);
                    const double S = wab * E.Sc[d];
                    if (d == 0) {
#pragma unroll
                        for (int j = 0; j < N; ++j) G0[gix0(0, j)] = S * y[j];
                    } else if (d == 1) {
#pragma unroll
                        for (int j = 0; j < N; ++j) G1[gix1(1, j)] = S * y[j];
                    } else {
#pragma unroll
                        for (int j = 0; j < N; ++j) y2[j] = S * y[j];
                    }
                }
                pendV = nU;
                pendG = nG;
            }
            __syncthreads();
            // ---- L3: sum of the three directions, write r once ----
            if (act) {
                double* dst = r + (cidx(lp, ti1 * T1 + mc1, ti2 * T2 + mc2)) * N3;
            DG_CHECK(lp >= 0 && lp < M.L && cidx(lp, ti1 * T1 + mc1, ti2 * T2 + mc2) < (long long)M.L * PC);
                DG_CHECK(lp >= 0 && lp < M.L && cidx(lp, ti1 * T1 + mc1, ti2 * T2 + mc2) < (long long)M.L * PC);
#pragma unroll
                for (int j = 0; j < N; ++j) dst[pidx<N>(2, j, ma, mb)] = y2[j] + G0[gix0(2, j)] + G1[gix1(2, j)];
            }
            continue;
        }

        // ---------------- P1: stage 1 + own traces; foreign traces; c(x) tables ----------------
        double g2[N];
        if (act) {
            const double* xc = XC + mc * N3;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                double v[N];
#pragma unroll
                for (int j = 0; j < N; ++j) v[j] = xc[pidx<N>(d, j, ma, mb)];
                double xe[HE], xo[H > 0 ? H : 1];
                gn::split<N>(v, xe, xo);
                double ulo, glo, uhi, ghi;
                gn::traces<N>(E, xe, xo, ulo, glo, uhi, ghi);
                double y[N];
                gn::sweep<N, false, false>(E, xe, xo, y);
                TRp(3 * mc + d, 0)[mab] = make_double2(uhi, ghi);
                if (d == 0) {
#pragma unroll
                    for (int j = 0; j < N; ++j) G0[gix0(0, j)] = y[j];
                } else if (d == 1) {
#pragma unroll
                    for (int j = 0; j < N; ++j) G1[gix1(1, j)] = y[j];
                    TRp(flo1, 1)[mab] = make_double2(ulo, glo);
                } else {
#pragma unroll
                    for (int j = 0; j < N; ++j) g2[j] = y[j];
                    TRp(flo2, 1)[mab] = make_double2(ulo, glo);
                }
            }
        }
        foreign(XN, is_tr(lp + 1));
        cxcur = CX + (s & 1) * NC * CXSZ;
        cfcur = CF + (s & 1) * NCG * CFSZ;
        __syncthreads();
        GEN_STAMP(2);

        // stream the next step's own blocks (plane lp + 2) and geometry (plane lp + 1) behind the compute
        if (tid == PROD && s + 1 < nsteps) {
            gn::mbar_expect_tx(barA, xbytes(lp + 2) + GEOB);
            issue_x(lp + 2, XS + (s & 1) * NC * N3);
            if (AFFINE || COEFF) issue_geo(lp + 1, (s + 1) & 1);
        }

        // ---------------- P2: stage 2 at the thread's d=2 line points (a, b, q); face pass A ----------------
        double q2[N];
        if (act) {
            // geometry (G~, 16-B pairs) and c(x) factors ((cos, sin) pairs) as 16-B loads: one shared-memory
            // wavefront per warp instruction for these cell-uniform / row-uniform values
            double gt[6];
            if (AFFINE) {
                const double2* g2p = reinterpret_cast<const double2*>(gb + mc * GREC);
                const double2 ga = g2p[0], gbb = g2p[1], gc = g2p[2];
                gt[0] = ga.x; gt[1] = ga.y; gt[2] = gbb.x; gt[3] = gbb.y; gt[4] = gc.x; gt[5] = gc.y;
            } else {
#pragma unroll
                for (int i = 0; i < 6; ++i) gt[i] = 0.0;
            }
            double z0r = 0, z0i = 0, z1r = 0, z1i = 0;
            const double2* cx2 = reinterpret_cast<const double2*>(cxcur + mc * CXSZ); // [k][b][q] (cos, sin)
            if (COEFF) {
                const double2 a0 = cx2[(0 * 3 + 0) * (N + 1) + ma], b0 = cx2[(0 * 3 + 1) * (N + 1) + mb];
                const double2 a1 = cx2[(1 * 3 + 0) * (N + 1) + ma], b1 = cx2[(1 * 3 + 1) * (N + 1) + mb];
                gn::cmul(a0.x, a0.y, b0.x, b0.y, z0r, z0i);
                gn::cmul(a1.x, a1.y, b1.x, b1.y, z1r, z1i);
            }
            const double wab = sW[ma] * sW[mb];
#pragma unroll
            for (int q = 0; q < N; ++q) {
                const int P = gix0(2, q), P1 = gix1(2, q);
                double cW = wab * E.w[q];
                if (COEFF) {
                    const double2 e0 = cx2[(0 * 3 + 2) * (N + 1) + q];
                    const double2 e1 = cx2[(1 * 3 + 2) * (N + 1) + q];
                    const double s0 = fma(z0r, e0.y, z0i * e0.x);  // Im(z0 e0) = sin(2 pi x0)
                    const double c1 = fma(z1r, e1.x, -z1i * e1.y); // Re(z1 e1) = cos(2 pi x1)
                    cW *= fma(0.5 * s0, c1, 1.0);
                }
                const double a0 = G0[P], a1 = G1[P1], a2 = g2[q];
                if (AFFINE) {
                    G0[P] = cW * fma(gt[0], a0, fma(gt[3], a1, gt[4] * a2));
                    G1[P1] = cW * fma(gt[3], a0, fma(gt[1], a1, gt[5] * a2));
                    q2[q] = cW * fma(gt[4], a0, fma(gt[5], a1, gt[2] * a2));
                } else {
                    const double adet = M.h[0] * M.h[1] * M.h[2];
                    G0[P] = cW * (adet / (M.h[0] * M.h[0])) * a0;
                    G1[P1] = cW * (adet / (M.h[1] * M.h[1])) * a1;
                    q2[q] = cW * (adet / (M.h[2] * M.h[2])) * a2;
                }
            }
        }
        if (AFFINE && !FACE_LINES) {
            pt_faces(ptA, std::false_type{}, gb);
            __syncthreads();
            pt_faces(ptB, std::false_type{}, gb);
            __syncthreads();
            pt_faces(ptC, std::true_type{}, gb);
            __syncthreads();
        } else if (AFFINE) {
#ifdef DG_GEN_CTA_FACES
            face_lines(lineA, std::true_type{}, gb, NF);
            __syncthreads();
            GEN_STAMP(3);
            // ---------------- P3: face line pass B (flux) ----------------
            face_lines(lineB, std::false_type{}, gb, NF);
            __syncthreads();
            GEN_STAMP(4);
            // ---------------- P4: face line pass C (tangential back-projection) ----------------
            face_lines(lineC, std::true_type{}, gb, NF);
            __syncthreads();
            GEN_STAMP(5);
#else
            // ---------------- P3: face passes A -> B -> C, warp-local ----------------
            GEN_STAMP(4);
            face_warp(gb);
            GEN_STAMP(5);
            __syncthreads();
            GEN_STAMP(3);
#endif
        } else {
            all_faces(passB, gb);
            __syncthreads();
        }
        // the ring buffer (aliased by the face buffers) is free: stream the next plane's ring blocks
        if (s + 1 < nsteps) {
            if (tid == PROD) issue_ring_bulk(lp + 1);
        }

        // ---------------- P5: stage 3 + face back-projection; d = 0, 1 in place, d = 2 -> r ----------------
        if (act) {
            {
                double v[N];
#pragma unroll
                for (int j = 0; j < N; ++j) v[j] = G0[gix0(0, j)];
                double xe[HE], xo[H > 0 ? H : 1];
                gn::split<N>(v, xe, xo);
                double y[N];
                const double2 hi = TRp(3 * mc, 0)[mab];
                gn::sweep<N, true, true>(E, xe, xo, y, pendV, pendG, hi.x, hi.y);
#pragma unroll
                for (int j = 0; j < N; ++j) G0[gix0(0, j)] = y[j];
                const double2 nx = TRp(3 * mc, 1)[mab]; // the T+ half of this face is the next plane's lower face
                pendV = nx.x;
                pendG = nx.y;
            }
            {
                double v[N];
#pragma unroll
                for (int j = 0; j < N; ++j) v[j] = G1[gix1(1, j)];
                double xe[HE], xo[H > 0 ? H : 1];
                gn::split<N>(v, xe, xo);
                double y[N];
                const double2 lo = TRp(flo1, 1)[mab], hi = TRp(3 * mc + 1, 0)[mab];
                gn::sweep<N, true, true>(E, xe, xo, y, lo.x, lo.y, hi.x, hi.y);
#pragma unroll
                for (int j = 0; j < N; ++j) G1[gix1(1, j)] = y[j];
            }
        }
        __syncthreads();
        GEN_STAMP(6);
        if (act) {
            double xe[HE], xo[H > 0 ? H : 1];
            gn::split<N>(q2, xe, xo);
            double y[N];
            const double2 lo = TRp(flo2, 1)[mab], hi = TRp(3 * mc + 2, 0)[mab];
            gn::sweep<N, true, true>(E, xe, xo, y, lo.x, lo.y, hi.x, hi.y);
            double* dst = r + (cidx(lp, ti1 * T1 + mc1, ti2 * T2 + mc2)) * N3;
            DG_CHECK(lp >= 0 && lp < M.L && cidx(lp, ti1 * T1 + mc1, ti2 * T2 + mc2) < (long long)M.L * PC);
#pragma unroll
            for (int j = 0; j < N; ++j) dst[pidx<N>(2, j, ma, mb)] = y[j] + G0[gix0(2, j)] + G1[gix1(2, j)];
        }
        GEN_STAMP(7);
        // (the barrier at the top of the next step orders these reads before the next writes)
    }
}

} // namespace dg
