// K_quad: the SIPG operator with a general Gauss rule of M > n points per direction (SURVEY §8(f2):
// overintegration, "quadrature with m points"), i.e. the paper's general sum factorisation
// with interpolation A = [l_j(xi_q)] != I (Eq. lowcomplex, Alg. assembly):
//
//   stage 1  grad_hat U at the M^3 points:  d0 = D0 A1 A2 X,  d1 = A0 D1 A2 X,  d2 = A0 A1 D2 X
//            (shared partial contractions: A2 X / D2 X along j2 first, then j1, then j0)
//   stage 2  Q = w_q c(x_q) |det J| J^{-1} J^{-T} grad_hat U at the M^3 points
//   stage 3  R = D0^T A1^T A2^T Q0 + A0^T D1^T A2^T Q1 + A0^T A1^T D2^T Q2  (transposes, reverse order)
//   faces    traces along the face normal with the 1-point tables e, d (normal first
//            P:L884), then A (values, normal derivative) and D (tangential derivatives) on the face to
//            its M^2 points, SIPG flux (Eq. diffreac_weak, theta = -1, geometry of T- R11,
//            c_F at the T- mapped points R12), back-projection with the transposed face contractions.
//
// Cell-centric (each cell evaluates its 6 faces with the neighbour's traces read from L2; r written
// once); CPB cells per CTA, every contraction a 1D sweep over the lines of a shared-memory array,
// distributed over the CTA's threads. A correctness-first path for the general case (no config of
// BASELINE.json uses it); k_gen is the tuned collocation path.
#pragma once

#include "common.cuh"

namespace dg {

// Even/odd form of an LO x LIN table T with T[LO-1-q][LIN-1-j] = S T[q][j] (S = +1: the interpolation A, S = -1:
// the derivative D; both on symmetric nodes and symmetric Gauss points, and their transposes): with
// xe_j = x_j + x_{LIN-1-j}, xo_j = x_j - x_{LIN-1-j} (j < LIN/2; xe holds the middle entry of an odd line),
//   E_q = Pe[q] . xe, O_q = Po[q] . xo, y_q = E_q + O_q, y_{LO-1-q} = S (E_q - O_q)   (q < LO/2),
//   y_mid = Pm . xe (S = +1) or Pm . xo (S = -1)                                       (odd LO).
// Half the FMAs of the plain product and half the distinct table doubles (sm_100a DFMA takes table operands from
// the uniform registers, 31 doubles).
template <int LO, int LIN, int S>
struct EOMat {
    static constexpr int HO = LO / 2, HI = LIN / 2, HEI = HI + (LIN & 1);
    double Pe[HO > 0 ? HO : 1][HEI];
    double Po[HO > 0 ? HO : 1][HI > 0 ? HI : 1];
    double Pm[HEI];
};

template <int N, int M>
struct QTab {
    double A[M * N];  // A[q*N + j] = l_j(xi_q) at the M Gauss points (basis: Lagrange on the N Gauss nodes)
    double Dq[M * N]; // l_j'(xi_q)
    double wq[M], xq[M];
    double e0[N], e1[N], d0[N], d1[N];
    EOMat<M, N, 1> eA;   // A, D and their transposes in even/odd form (the sweeps)
    EOMat<M, N, -1> eD;
    EOMat<N, M, 1> eAt;
    EOMat<N, M, -1> eDt;
};

template <int LO, int LIN, int S>
__host__ __device__ __forceinline__ void eo_apply(const EOMat<LO, LIN, S>& T, const double v[LIN], double y[LO])
{
    constexpr int HO = LO / 2, HI = LIN / 2, HEI = HI + (LIN & 1);
    double xe[HEI], xo[HI > 0 ? HI : 1];
#pragma unroll
    for (int j = 0; j < HI; ++j) {
        xe[j] = v[j] + v[LIN - 1 - j];
        xo[j] = v[j] - v[LIN - 1 - j];
    }
    if (LIN & 1) xe[HI] = v[HI];
#pragma unroll
    for (int q = 0; q < HO; ++q) {
        double e = 0.0, o = 0.0;
#pragma unroll
        for (int j = 0; j < HEI; ++j) e = fma(T.Pe[q][j], xe[j], e);
#pragma unroll
        for (int j = 0; j < HI; ++j) o = fma(T.Po[q][j], xo[j], o);
        y[q] = e + o;
        y[LO - 1 - q] = S > 0 ? e - o : o - e;
    }
    if (LO & 1) {
        double m = 0.0;
        if (S > 0) {
#pragma unroll
            for (int j = 0; j < HEI; ++j) m = fma(T.Pm[j], xe[j], m);
        } else {
#pragma unroll
            for (int j = 0; j < HI; ++j) m = fma(T.Pm[j], xo[j], m);
        }
        y[HO] = m;
    }
}

namespace qd {

// 1D contraction along dimension DIM of a 3D array with extents (E0, E1, E2) (dimension 0 fastest):
// out[.., q, ..] (+)= sum_j T(q, j) in[.., j, ..]; T(q, j) = TRN ? T[j*LO + q] : T[q*LIN + j].
// T is a table of the kernel parameter (constant bank): the indices are compile-time after unrolling,
// so the coefficients are uniform operands (no per-FMA shared-memory load).
template <int E0, int E1, int E2, int DIM, int LO, bool TRN, bool ACC>
struct Sw3 {
    static constexpr int LIN = DIM == 0 ? E0 : (DIM == 1 ? E1 : E2);
    static constexpr int NL = (E0 * E1 * E2) / LIN; // lines
    static constexpr int O0 = DIM == 0 ? LO : E0, O1 = DIM == 1 ? LO : E1;
    __device__ static void line(const double* in, double* out, const double* T, int l)
    {
        int ib, ist, ob, ost;
        if (DIM == 0) { ib = E0 * l; ist = 1; ob = O0 * l; ost = 1; }
        else if (DIM == 1) { const int i0 = l % E0, i2 = l / E0; ib = i0 + E0 * E1 * i2; ist = E0; ob = i0 + O0 * O1 * i2; ost = O0; }
        else { ib = l; ist = E0 * E1; ob = l; ost = O0 * O1; }
        double v[LIN];
#pragma unroll
        for (int j = 0; j < LIN; ++j) v[j] = in[ib + ist * j];
#pragma unroll
        for (int q = 0; q < LO; ++q) {
            double a = 0.0;
#pragma unroll
            for (int j = 0; j < LIN; ++j) a = fma(TRN ? T[j * LO + q] : T[q * LIN + j], v[j], a);
            out[ob + ost * q] = ACC ? out[ob + ost * q] + a : a;
        }
    }
    // one input line, two tables -> two outputs (the line is loaded once and a warp runs one sweep body)
    __device__ static void line2(const double* in, double* out1, const double* T1, double* out2, const double* T2, int l)
    {
        int ib, ist, ob, ost;
        if (DIM == 0) { ib = E0 * l; ist = 1; ob = O0 * l; ost = 1; }
        else if (DIM == 1) { const int i0 = l % E0, i2 = l / E0; ib = i0 + E0 * E1 * i2; ist = E0; ob = i0 + O0 * O1 * i2; ost = O0; }
        else { ib = l; ist = E0 * E1; ob = l; ost = O0 * O1; }
        double v[LIN];
#pragma unroll
        for (int j = 0; j < LIN; ++j) v[j] = in[ib + ist * j];
#pragma unroll
        for (int q = 0; q < LO; ++q) {
            double a = 0.0, b = 0.0;
#pragma unroll
            for (int j = 0; j < LIN; ++j) {
                a = fma(TRN ? T1[j * LO + q] : T1[q * LIN + j], v[j], a);
                b = fma(TRN ? T2[j * LO + q] : T2[q * LIN + j], v[j], b);
            }
            out1[ob + ost * q] = ACC ? out1[ob + ost * q] + a : a;
            out2[ob + ost * q] = ACC ? out2[ob + ost * q] + b : b;
        }
    }
    // the same with tables in even/odd form (EOMat)
    template <int S>
    __device__ static void line(const double* in, double* out, const EOMat<LO, LIN, S>& T, int l)
    {
        int ib, ist, ob, ost;
        idx(l, ib, ist, ob, ost);
        double v[LIN], y[LO];
#pragma unroll
        for (int j = 0; j < LIN; ++j) v[j] = in[ib + ist * j];
        eo_apply(T, v, y);
#pragma unroll
        for (int q = 0; q < LO; ++q) out[ob + ost * q] = ACC ? out[ob + ost * q] + y[q] : y[q];
    }
    template <int S1, int S2>
    __device__ static void line2(const double* in, double* out1, const EOMat<LO, LIN, S1>& T1, double* out2,
                                 const EOMat<LO, LIN, S2>& T2, int l)
    {
        int ib, ist, ob, ost;
        idx(l, ib, ist, ob, ost);
        double v[LIN], y[LO];
#pragma unroll
        for (int j = 0; j < LIN; ++j) v[j] = in[ib + ist * j];
        eo_apply(T1, v, y);
#pragma unroll
        for (int q = 0; q < LO; ++q) out1[ob + ost * q] = ACC ? out1[ob + ost * q] + y[q] : y[q];
        eo_apply(T2, v, y);
#pragma unroll
        for (int q = 0; q < LO; ++q) out2[ob + ost * q] = ACC ? out2[ob + ost * q] + y[q] : y[q];
    }
    __device__ static void idx(int l, int& ib, int& ist, int& ob, int& ost)
    {
        if (DIM == 0) { ib = E0 * l; ist = 1; ob = O0 * l; ost = 1; }
        else if (DIM == 1) { const int i0 = l % E0, i2 = l / E0; ib = i0 + E0 * E1 * i2; ist = E0; ob = i0 + O0 * O1 * i2; ost = O0; }
        else { ib = l; ist = E0 * E1; ob = l; ost = O0 * O1; }
    }
};

// the same for a 2D array with extents (E0, E1)
template <int E0, int E1, int DIM, int LO, bool TRN, bool ACC>
struct Sw2 {
    static constexpr int LIN = DIM == 0 ? E0 : E1;
    static constexpr int NL = (E0 * E1) / LIN;
    static constexpr int O0 = DIM == 0 ? LO : E0;
    __device__ static void line(const double* in, double* out, const double* T, int l)
    {
        const int ib = DIM == 0 ? E0 * l : l, ist = DIM == 0 ? 1 : E0;
        const int ob = DIM == 0 ? O0 * l : l, ost = DIM == 0 ? 1 : O0;
        double v[LIN];
#pragma unroll
        for (int j = 0; j < LIN; ++j) v[j] = in[ib + ist * j];
#pragma unroll
        for (int q = 0; q < LO; ++q) {
            double a = 0.0;
#pragma unroll
            for (int j = 0; j < LIN; ++j) a = fma(TRN ? T[j * LO + q] : T[q * LIN + j], v[j], a);
            out[ob + ost * q] = ACC ? out[ob + ost * q] + a : a;
        }
    }
    template <int S>
    __device__ static void line(const double* in, double* out, const EOMat<LO, LIN, S>& T, int l)
    {
        const int ib = DIM == 0 ? E0 * l : l, ist = DIM == 0 ? 1 : E0;
        const int ob = DIM == 0 ? O0 * l : l, ost = DIM == 0 ? 1 : O0;
        double v[LIN], y[LO];
#pragma unroll
        for (int j = 0; j < LIN; ++j) v[j] = in[ib + ist * j];
        eo_apply(T, v, y);
#pragma unroll
        for (int q = 0; q < LO; ++q) out[ob + ost * q] = ACC ? out[ob + ost * q] + y[q] : y[q];
    }
};

template <int N, int M, bool U0 = false>
struct QLay {
    static constexpr int NT = 256;
    // thread groups: each group of GT threads owns one cell and synchronises with a named barrier of its own,
    // so the cells of a CTA progress independently (n <= 4: 4 groups of 64; n = 5, 6: 2 of 128; else 1 of 256)
    static constexpr int GT = N <= 4 ? 64 : (N <= 6 ? 128 : 256);
    static constexpr int CPB = NT / GT;
    static constexpr int N2 = N * N, N3 = N * N * N, M2 = M * M, M3 = M * M * M, NM = N * M;
    // per cell (doubles). Region A = X, R, Y2, Y2d and the face traces FT is dead from P3 to P5 and holds the
    // face flux coefficients C of P4 -> P5 there (when they fit; n <= 3: a region of their own)
    //   FT [face][4][N2] (own u, own g, nb u, nb g) -> later FB2 [2][N2] (V2, G2)
    //   F1 [face][6][NM] (own Ua1, Ud1, Ga1; nb Ua1, Ud1, Ga1) -> later FB1 [3][NM] (Pv, Pt, Pn)
    //   C  [face][4][M2] (Cv, Ct1, Ct2, Cn): the face values at the M^2 points are formed in P4 directly from F1
    static constexpr int X = 0, R = X + N3, Y2 = R + N3, Y2d = Y2 + N2 * M, FT = Y2d + N2 * M;
    // per-face strides made odd: the face sweeps run with lanes over (face, line), and an even stride that is a
    // multiple of 16 doubles put the same line of every face on the same banks (4-8-way conflicts)
    // (measured: n = 4 2 % faster; n = 6 0.5 % slower, kept dense there)
    static constexpr int ODD = N < 6 ? 1 : 0;
    static constexpr int FTS = (4 * N2) | ODD, F1S = (6 * NM) | ODD, CS = (4 * M2) | ODD;
    static constexpr int AEND = FT + 6 * FTS;
    static constexpr bool CALIAS = 6 * CS <= AEND;
    static constexpr int Z = AEND, Zd1 = Z + N * M2, Zd2 = Zd1 + N * M2, G0 = Zd2 + N * M2, G1 = G0 + M3, G2 = G1 + M3;
    static constexpr int GU = G2 + M3;      // u at the M^3 points (diffusion-reaction: reaction / source terms)
    static constexpr int U0Q = GU + M3;     // U0: the linearization point u0 at the M^3 points (Jacobian action)
    static constexpr int T2U = U0Q + (U0 ? M3 : 0); // U0: u0 after the j2 and j1 sweeps [N][M][M]
    static constexpr int F1 = T2U + (U0 ? N * M2 : 0);
    static constexpr int C = CALIAS ? X : F1 + 6 * F1S;
    static constexpr int GEO = F1 + 6 * F1S + (CALIAS ? 0 : 6 * CS); // per cell: Gt[6], J rows 0-1 [6], o[2]; per face 16
    static constexpr int CELL = GEO + 14 + 6 * 16;
    static constexpr int CELLP = (CELL + 1) / 2 * 2;
    static constexpr int TAB = CPB * CELLP;   // shared tables: A, Dq (M N each), wq, xq (M), e0, e1, d0, d1 (N)
    static constexpr int END = TAB + 2 * M * N + 2 * M + 4 * N;
    static constexpr int BYTES = END * 8;
    // resident CTAs per SM the shared memory allows (the register cap follows from it)
    // (at most 2 for n >= 6: their sweeps need ~128 registers; 85 spill heavily)
    static constexpr int MINB_SMEM = (BYTES + 2048) * 4 <= 228 * 1024 ? 4 : ((BYTES + 2048) * 3 <= 228 * 1024 ? 3 : ((BYTES + 2048) * 2 <= 228 * 1024 ? 2 : 1));
    // (at most 3 otherwise: 4 would cap the registers at 64 and spill heavily)
    static constexpr int MINB = (N >= 6 && MINB_SMEM > 2) ? 2 : (MINB_SMEM > 3 ? 3 : MINB_SMEM);
};

} // namespace qd

// grid: ceil(cells / CPB), block NT, dynamic smem QLay::BYTES. Cells [c_begin, c_end) of the slab
// (local, canonical order).
// DR: the paper's diffusion-reaction problem (axiparallel mesh of the
// non-periodic unit cube): K(x) = x x^T + I in place of c I, reaction c = 10 and source f = -6 in the
// volume (u at the quadrature points: the 4th quantity of the stacked stage 1, Eq. fusedtensor),
// boundary faces with the Dirichlet data g = |x|^2 (one-sided flux, [u] -> u - g), penalty
// alpha k (k+2) |F| / |T| (alpha = penalty_scale, set in M.gamma by dg_setup).
// PR: 0 the periodic operator; 1 the paper's (linear) diffusion-reaction residual; 2 its nonlinear variant
// (reading R26: reaction c u^2, f = c|x|^4 - 10|x|^2 - 6); 3 the action of that variant's
// Jacobian J(u0) x: u0, the linearization point, is evaluated at the M^3 points by
// the same A A A sweeps (a second input of the fused stage 1), the reaction becomes 2 c u0 x, the f and g
// terms drop out (they do not depend on the solution).
template <int N, int M, bool AFFINE, bool COEFF, int PR = 0>
__global__ void __launch_bounds__(256, qd::QLay<N, M, PR == 3>::MINB) // as many CTAs / SM as shared memory allows
k_quad(const double* __restrict__ x, const double* __restrict__ xb, const double* __restrict__ xa, double* __restrict__ r,
       long long c_begin, long long c_end, const __grid_constant__ QTab<N, M> T, const MeshArgs M_,
       const double* __restrict__ u0)
{
    constexpr bool DR = PR != 0;
    using L = qd::QLay<N, M, PR == 3>;
    constexpr int CPB = L::CPB, NT = L::NT, GT = L::GT, N2 = L::N2, N3 = L::N3, M2 = L::M2, M3 = L::M3, NM = L::NM;
    const MeshArgs& Ms = M_;
    extern __shared__ __align__(16) double sm[];
    double* const sA = sm + L::TAB;
    double* const sDq = sA + M * N;
    double* const sw = sDq + M * N;
    double* const sxq = sw + M;
    double* const se0 = sxq + M;
    double* const se1 = se0 + N;
    double* const sd0 = se1 + N;
    double* const sd1 = sd0 + N;
    const int tid = threadIdx.x;
    const int grp = tid / GT, gtid = tid - grp * GT; // this thread's group (= its cell in the CTA)
    const long long cfirst = c_begin + (long long)blockIdx.x * CPB + grp;
    const int ncell = cfirst < c_end ? 1 : 0;        // cells of the group
    auto cellp = [&](int c) { return sm + (grp + c) * L::CELLP; };
    // group barrier (named barrier 1 + grp over the group's GT threads; the CTA barrier when one group)
    auto gsync = [&]() {
        if constexpr (GT == NT) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(GT) : "memory");
    };
    // first task of this thread in a loop that follows `before` tasks of the same phase (dealt round-robin from
    // thread 0): the loop starts where the previous one ended, so the threads that got a task more there get one
    // less here (the phases end at a group barrier: its wait is the phase's most loaded thread). Measured: n = 6
    // (128-thread groups) 2-6 % faster; n = 4 (64-thread groups, neighbour traces prefetched) 9 % slower: n >= 6 only
    auto rot = [&](int before) { return N >= 6 ? (gtid - before % GT + GT) % GT : gtid; };
    // n < 6 (64-thread groups): the task kinds of a stage loop start on warp boundaries (each kind's range padded to
    // a multiple of 32), so a warp runs one sweep body; n >= 6 keeps the dense ranges the rot() balance assumes
    constexpr auto kpad = [](int nl) { return N < 6 ? (nl + 31) / 32 * 32 : nl; };
    auto ftp = [&](int c, int f) { return cellp(c) + L::FT + f * L::FTS; };  // face traces / FB2
    auto f1p = [&](int c, int f) { return cellp(c) + L::F1 + f * L::F1S; };  // t1 contractions / FB1
    auto cfp = [&](int c, int f) { return cellp(c) + L::C + f * L::CS; };    // flux coefficients

    for (int i = tid; i < M * N; i += NT) { sA[i] = T.A[i]; sDq[i] = T.Dq[i]; }
    for (int i = tid; i < M; i += NT) { sw[i] = T.wq[i]; sxq[i] = T.xq[i]; }
    for (int i = tid; i < N; i += NT) { se0[i] = T.e0[i]; se1[i] = T.e1[i]; sd0[i] = T.d0[i]; sd1[i] = T.d1[i]; }
    for (int c = 0; c < ncell; ++c)
        for (int i = gtid; i < N3; i += GT) cellp(c)[L::X + i] = __ldg(x + (cfirst + c) * N3 + i);
    if (PR == 3) // the linearization point, into R (unused until stage 3)
        for (int c = 0; c < ncell; ++c)
            for (int i = gtid; i < N3; i += GT) cellp(c)[L::R + i] = __ldg(u0 + (cfirst + c) * N3 + i);

    // cell coordinates, computed once per cell (32-bit: a slab has < 2^31 cells)
    __shared__ int s_co[CPB][5]; // lp, rem, i0, i1, i2
    if (gtid == 0 && ncell) {
        const int lc = (int)cfirst;
        const int lp = lc / Ms.plane_cells, rem = lc - lp * Ms.plane_cells;
        s_co[grp][0] = lp;
        s_co[grp][1] = rem;
        s_co[grp][2] = (Ms.plane_begin + lp) % Ms.N0;
        s_co[grp][3] = rem / Ms.N2;
        s_co[grp][4] = rem - (rem / Ms.N2) * Ms.N2;
    }
    __syncthreads(); // (tables are shared by the groups; from here on each group syncs on its own)
    if (!ncell) return;
    auto coords = [&](int c, int& lp, int& rem, int ig[3]) {
        lp = s_co[grp + c][0];
        rem = s_co[grp + c][1];
        ig[0] = s_co[grp + c][2];
        ig[1] = s_co[grp + c][3];
        ig[2] = s_co[grp + c][4];
    };
    auto jac_of = [&](int lp, int rem, double* J) {
        const double* jp = Ms.jac + ((long long)(lp + 1) * Ms.plane_cells + rem) * 9;
#pragma unroll
        for (int i = 0; i < 9; ++i) J[i] = __ldg(jp + i);
    };
    // neighbour (local plane, in-plane index, global coords) across face (d, side)
    auto neighbour = [&](int lp, int rem, const int ig[3], int d, int side, int& nlp, int& nrem, int nig[3]) {
        const int Nd = d == 0 ? Ms.N0 : (d == 1 ? Ms.N1 : Ms.N2);
        nig[0] = ig[0]; nig[1] = ig[1]; nig[2] = ig[2];
        nig[d] = (ig[d] + (side ? 1 : Nd - 1)) % Nd;
        nlp = lp;
        nrem = rem;
        if (d == 0) nlp = lp + (side ? 1 : -1);
        else nrem = nig[1] * Ms.N2 + nig[2];
    };

    // ---------------- P0: geometry (one thread per cell for the volume, per (cell, face) for the faces) --------
    for (int t = gtid; t < ncell * 7; t += GT) {
        const int c = t / 7, f = t % 7;
        int lp, rem, ig[3];
        coords(c, lp, rem, ig);
        double* g = cellp(c) + L::GEO;
        if (!AFFINE) {
            // axis-aligned: J = diag(h), no inverse needed
            const double h0 = Ms.h[0], h1 = Ms.h[1], h2 = Ms.h[2], ad = h0 * h1 * h2;
            if (f == 6) {
                g[0] = ad / (h0 * h0); g[1] = ad / (h1 * h1); g[2] = ad / (h2 * h2); g[3] = g[4] = g[5] = 0.0;
                g[6] = h0; g[7] = 0.0; g[8] = 0.0; g[9] = 0.0; g[10] = h1; g[11] = 0.0;
                g[12] = (double)ig[0] / Ms.N0;
                g[13] = (double)ig[1] / Ms.N1;
                continue;
            }
            const int d = f >> 1, side = f & 1;
            const int Nd = d == 0 ? Ms.N0 : (d == 1 ? Ms.N1 : Ms.N2);
            double* fg = g + 14 + 16 * f;
            fg[0] = ad / Ms.h[d];
            for (int e = 0; e < 3; ++e) fg[1 + e] = fg[4 + e] = (e == d) ? 1.0 / Ms.h[d] : 0.0;
            fg[7] = h0; fg[8] = 0.0; fg[9] = 0.0; fg[10] = 0.0; fg[11] = h1; fg[12] = 0.0;
            const int mi0 = (d == 0 && !side) ? (ig[0] + Ms.N0 - 1) % Ms.N0 : ig[0];
            const int mi1 = (d == 1 && !side) ? (ig[1] + Ms.N1 - 1) % Ms.N1 : ig[1];
            fg[13] = (double)mi0 / Ms.N0;
            fg[14] = (double)mi1 / Ms.N1;
            fg[15] = (DR && (side ? ig[d] == Nd - 1 : ig[d] == 0)) ? 1.0 : 0.0;
            continue;
        }
        double J[9], Ji[9];
        jac_of(lp, rem, J);
        const double det = inv3(J, Ji);
        if (f == 6) {
            const double ad = fabs(det);
            auto gg = [&](int a, int b) { return ad * (Ji[3 * a] * Ji[3 * b] + Ji[3 * a + 1] * Ji[3 * b + 1] + Ji[3 * a + 2] * Ji[3 * b + 2]); };
            g[0] = gg(0, 0); g[1] = gg(1, 1); g[2] = gg(2, 2); g[3] = gg(0, 1); g[4] = gg(0, 2); g[5] = gg(1, 2);
            for (int i = 0; i < 6; ++i) g[6 + i] = J[i];
            g[12] = (double)ig[0] / Ms.N0;
            g[13] = (double)ig[1] / Ms.N1;
            continue;
        }
        const int d = f >> 1, side = f & 1; // face f = 2d + side; side 1: upper face (cell is T-)
        int nlp, nrem, nig[3];
        neighbour(lp, rem, ig, d, side, nlp, nrem, nig);
        double Jn[9], Jni[9];
        if (AFFINE) jac_of(nlp, d == 0 ? rem : nrem, Jn);
        else for (int i = 0; i < 9; ++i) Jn[i] = J[i];
        inv3(Jn, Jni);
        const double* Jm = side ? J : Jn;   // T-
        const double* Jmi = side ? Ji : Jni;
        const double* Jpi = side ? Jni : Ji;
        const double detm = side ? det : det3(Jn);
        const double nu0 = Jmi[3 * d], nu1 = Jmi[3 * d + 1], nu2 = Jmi[3 * d + 2];
        const double nn = sqrt(nu0 * nu0 + nu1 * nu1 + nu2 * nu2);
        const double n0 = nu0 / nn, n1 = nu1 / nn, n2 = nu2 / nn;
        double* fg = g + 14 + 16 * f;
        fg[0] = fabs(detm) * nn; // dS (Nanson)
        for (int e = 0; e < 3; ++e) {
            fg[1 + e] = Jmi[3 * e] * n0 + Jmi[3 * e + 1] * n1 + Jmi[3 * e + 2] * n2; // a- = J_-^{-1} n_F
            fg[4 + e] = Jpi[3 * e] * n0 + Jpi[3 * e + 1] * n1 + Jpi[3 * e + 2] * n2; // a+ = J_+^{-1} n_F
        }
        for (int i = 0; i < 6; ++i) fg[7 + i] = Jm[i];
        const int* mig = side ? ig : nig;
        fg[13] = (double)mig[0] / Ms.N0;
        fg[14] = (double)mig[1] / Ms.N1;
        // DR: 1 on the boundary of the (non-periodic) cube
        const int Nd = d == 0 ? Ms.N0 : (d == 1 ? Ms.N1 : Ms.N2);
        fg[15] = (DR && (side ? ig[d] == Nd - 1 : ig[d] == 0)) ? 1.0 : 0.0;
    }
    gsync();

    // (Jacobian: u0 at the M^3 points, U0Q = A0 A1 A2 u0, by three sweeps riding along with stage 1a-1c in
    // P1-P3: R -> T1 (the G0 area, free until P3) -> T2U -> U0Q)
    auto u0_T1 = [&](int c) { return cellp(c) + L::G0; }; // (G0 is first written in P3)

    // ---------------- P1: stage 1a (along j2); face traces along the normal (own from smem, neighbour from L2) ----
    {
        // the neighbour values of this thread's trace tasks are loaded before the stage-1a sweeps and consumed
        // after them (L2 latency behind the sweeps; n <= 5, where the registers allow it)
        constexpr bool PREF = N <= 5;
        // the face-trace tasks follow the stage-1a sweeps (and the Jacobian's u0 sweeps)
        const int P1_BEFORE = ncell * qd::Sw3<N, N, N, 2, M, false, false>::NL * (PR == 3 ? 2 : 1);
        constexpr int NFT = PREF ? (6 * N2 + GT - 1) / GT : 1;
        double vnb[NFT][N];
        auto nb_of = [&](int c, int f) -> const double* {
            const int d = f >> 1, side = f & 1;
            int lp, rem, ig[3];
            coords(c, lp, rem, ig);
            int nlp, nrem, nig[3];
            neighbour(lp, rem, ig, d, side, nlp, nrem, nig);
            if (d == 0) return nlp < 0 ? xb + (long long)rem * N3 : (nlp >= Ms.L ? xa + (long long)rem * N3 : x + ((long long)nlp * Ms.plane_cells + rem) * N3);
            return x + ((long long)lp * Ms.plane_cells + nrem) * N3;
        };
        if constexpr (PREF) {
#pragma unroll
            for (int k = 0; k < NFT; ++k) {
                const int t = rot(P1_BEFORE) + k * GT;
                if (t < ncell * 6 * N2) {
                    const int c = t / (6 * N2), f = (t / N2) % 6, p = t % N2, a = p % N, bq = p / N;
                    const bool bnd = DR && cellp(c)[L::GEO + 14 + 16 * f + 15] != 0.0;
                    const double* nbx = nb_of(c, f);
#pragma unroll
                    for (int j = 0; j < N; ++j) vnb[k][j] = bnd ? 0.0 : __ldg(nbx + pidx<N>(f >> 1, j, a, bq));
                }
            }
        }
        using S = qd::Sw3<N, N, N, 2, M, false, false>;
        for (int t = gtid; t < ncell * S::NL; t += GT) {
            const int c = t / S::NL, l = t % S::NL;
            double* b = cellp(c);
            S::line2(b + L::X, b + L::Y2, T.eA, b + L::Y2d, T.eD, l); // A2 X and D2 X from one load of the line
        }
        if (PR == 3)
            for (int t = rot(ncell * S::NL); t < ncell * S::NL; t += GT) S::line(cellp(t / S::NL) + L::R, u0_T1(t / S::NL), T.eA, t % S::NL);
        constexpr int NFL = PREF ? NFT : (6 * N2 + GT - 1) / GT;
#pragma unroll
        for (int k = 0; k < NFL; ++k) {
            const int t = rot(P1_BEFORE) + k * GT;
            if (t >= ncell * 6 * N2) break;
            const int c = t / (6 * N2), f = (t / N2) % 6, p = t % N2, a = p % N, bq = p / N;
            const int d = f >> 1, side = f & 1;
            const double* nbx = PREF ? nullptr : nb_of(c, f);
            const double* xo = cellp(c) + L::X;
            const bool bnd = DR && cellp(c)[L::GEO + 14 + 16 * f + 15] != 0.0;
            double uo = 0, go = 0, un = 0, gn = 0;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double vo = xo[pidx<N>(d, j, a, bq)];
                const double vn = PREF ? vnb[k][j] : (bnd ? 0.0 : __ldg(nbx + pidx<N>(d, j, a, bq)));
                uo = fma(side ? se1[j] : se0[j], vo, uo);
                go = fma(side ? sd1[j] : sd0[j], vo, go);
                un = fma(side ? se0[j] : se1[j], vn, un);
                gn = fma(side ? sd0[j] : sd1[j], vn, gn);
            }
            double* FT = ftp(c, f);
            FT[p] = uo;
            FT[N2 + p] = go;
            FT[2 * N2 + p] = un;
            FT[3 * N2 + p] = gn;
        }
    }
    gsync();
    // ---------------- P2: stage 1b (along j1); face contraction along t1 ----------------
    {
        using SA = qd::Sw3<N, N, M, 1, M, false, false>;
        constexpr int NLp = kpad(SA::NL);
        for (int t = gtid; t < ncell * 2 * NLp; t += GT) {
            const int c = t / (2 * NLp), k = (t / NLp) % 2, l = t % NLp;
            if (l >= SA::NL) continue;
            double* b = cellp(c);
            if (k == 0) SA::line2(b + L::Y2, b + L::Z, T.eA, b + L::Zd1, T.eD, l); // A1 (A2 X), D1 (A2 X)
            else SA::line(b + L::Y2d, b + L::Zd2, T.eA, l);
        }
        if (PR == 3)
            for (int t = rot(ncell * 2 * SA::NL); t < ncell * SA::NL; t += GT) SA::line(u0_T1(t / SA::NL), cellp(t / SA::NL) + L::T2U, T.eA, t % SA::NL);
        using F = qd::Sw2<N, N, 0, M, false, false>; // [t1][t2]: N x N -> M x N
        for (int t = rot(ncell * SA::NL * (PR == 3 ? 3 : 2)); t < ncell * 6 * 6 * F::NL; t += GT) {
            // kind-major task order (the A-table kinds 0, 2, 3, 5, then the D-table kinds 1, 4): the lanes of a warp
            // run one sweep body instead of interleaving the kinds every F::NL lanes
            const int c = t / (36 * F::NL), kk = (t / (6 * F::NL)) % 6, f = (t / F::NL) % 6, l = t % F::NL;
            const int k = kk == 0 ? 0 : (kk == 1 ? 2 : (kk == 2 ? 3 : (kk == 3 ? 5 : (kk == 4 ? 1 : 4))));
            double* FT = ftp(c, f);
            double* F1 = f1p(c, f);
            // k: 0 own Ua1 = A u, 1 own Ud1 = D u, 2 own Ga1 = A g, 3..5 the same for the neighbour
            const double* src = FT + ((k < 3) ? (k == 2 ? N2 : 0) : (k == 5 ? 3 * N2 : 2 * N2));
            if (k % 3 == 1) F::line(src, F1 + k * NM, T.eD, l);
            else F::line(src, F1 + k * NM, T.eA, l);
        }
    }
    gsync();
    // ---------------- P3: stage 1c (along j0); face contraction along t2 ----------------
    {
        using SB = qd::Sw3<N, M, M, 0, M, false, false>;
        // (k = 0: Z -> G0 with D0 and, for the diffusion-reaction problems, Z -> GU = u with A0 from the same
        // line; k = 1, 2: the A0 sweeps of Zd1, Zd2 — one sweep body per task kind)
        constexpr int NLp = kpad(SB::NL);
        for (int t = gtid; t < ncell * 3 * NLp; t += GT) {
            const int c = t / (3 * NLp), k = (t / NLp) % 3, l = t % NLp;
            if (l >= SB::NL) continue;
            double* b = cellp(c);
            if (k == 0) {
                if (DR) SB::line2(b + L::Z, b + L::G0, T.eD, b + L::GU, T.eA, l);
                else SB::line(b + L::Z, b + L::G0, T.eD, l);
            } else {
                SB::line(b + (k == 1 ? L::Zd1 : L::Zd2), b + (k == 1 ? L::G1 : L::G2), T.eA, l);
            }
        }
        if (PR == 3)
            for (int t = rot(ncell * 3 * SB::NL); t < ncell * SB::NL; t += GT) SB::line(cellp(t / SB::NL) + L::T2U, cellp(t / SB::NL) + L::U0Q, T.eA, t % SB::NL);
        // (the face values at the M^2 points are formed pointwise in P4 from F1: no stored [8][M^2] array)
    }
    gsync();
    // ---------------- P4: stage 2 (pointwise at the M^3 points); face fluxes at the M^2 points ----------------
    for (int t = gtid; t < ncell * M3; t += GT) {
        const int c = t / M3, P = t % M3, q0 = P % M, q1 = (P / M) % M, q2 = P / M2;
        double* b = cellp(c);
        const double* g = b + L::GEO;
        double cW = sw[q0] * sw[q1] * sw[q2];
        if (COEFF) {
            const double xi0 = sxq[q0], xi1 = sxq[q1], xi2 = sxq[q2];
            cW *= coeff_sincos(g[12] + g[6] * xi0 + g[7] * xi1 + g[8] * xi2, g[13] + g[9] * xi0 + g[10] * xi1 + g[11] * xi2);
        }
        const double a0 = b[L::G0 + P], a1 = b[L::G1 + P], a2 = b[L::G2 + P];
        if (DR) {
            // (K grad u, grad v) + (c u - f, v), K = x x^T + I, c = 10, f = -6
            const double h0 = Ms.h[0], h1 = Ms.h[1], h2 = Ms.h[2];
            const double W = sw[q0] * sw[q1] * sw[q2] * h0 * h1 * h2;
            int lp_, rem_, ig_[3];
            coords(c, lp_, rem_, ig_);
            const double x0 = (ig_[0] + sxq[q0]) * h0, x1 = (ig_[1] + sxq[q1]) * h1, x2 = (ig_[2] + sxq[q2]) * h2;
            // (1/h by multiplication: a double division is a ~20-instruction sequence with a slow-path branch)
            const double ih0 = 1.0 / h0, ih1 = 1.0 / h1, ih2 = 1.0 / h2; // (loop-invariant: hoisted)
            const double p0 = a0 * ih0, p1 = a1 * ih1, p2 = a2 * ih2; // physical gradient
            const double xg = x0 * p0 + x1 * p1 + x2 * p2;        // K grad u = x (x . grad u) + grad u
            b[L::G0 + P] = W * fma(x0, xg, p0) * ih0;
            b[L::G1 + P] = W * fma(x1, xg, p1) * ih1;
            b[L::G2 + P] = W * fma(x2, xg, p2) * ih2;
            const double uq = b[L::GU + P];
            double react;
            if (PR == 1) {
                react = 10.0 * uq + 6.0;                              // c u - f
            } else if (PR == 2) {
                const double s2 = x0 * x0 + x1 * x1 + x2 * x2;
                react = 10.0 * uq * uq - (10.0 * s2 * s2 - 10.0 * s2 - 6.0); // c u^2 - f (R26)
            } else {
                react = 20.0 * b[L::U0Q + P] * uq;                    // 2 c u0 x
            }
            b[L::GU + P] = W * react;
            continue;
        }
        b[L::G0 + P] = cW * fma(g[0], a0, fma(g[3], a1, g[4] * a2));
        b[L::G1 + P] = cW * fma(g[3], a0, fma(g[1], a1, g[5] * a2));
        b[L::G2 + P] = cW * fma(g[4], a0, fma(g[5], a1, g[2] * a2));
    }
    for (int t = rot(ncell * M3); t < ncell * 6 * M2; t += GT) {
        const int c = t / (6 * M2), f = (t / M2) % 6, p = t % M2, a = p % M, bq = p / M;
        const int d = f >> 1, side = f & 1;
        const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
        double* F2 = cfp(c, f); // coefficients out
        const double* fg = cellp(c) + L::GEO + 14 + 16 * f;
        // own (s=0) and neighbour (s=1) -> T- / T+: the t2 contractions of F1 at the point (a, bq):
        // U_s = A Ua1_s, Gn_s = A Ga1_s, Gt1_s = A Ud1_s, Gt2_s = D Ua1_s
        double Uo = 0, Un = 0, Gno = 0, Gnn = 0, T1o = 0, T1n = 0, T2o = 0, T2n = 0;
        {
            const double* F1 = f1p(c, f) + a;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double Aj = sA[bq * N + j], Dj = sDq[bq * N + j];
                const double ua0 = F1[0 * NM + M * j], ud0 = F1[1 * NM + M * j], ga0 = F1[2 * NM + M * j];
                const double ua1 = F1[3 * NM + M * j], ud1 = F1[4 * NM + M * j], ga1 = F1[5 * NM + M * j];
                Uo = fma(Aj, ua0, Uo);
                Un = fma(Aj, ua1, Un);
                Gno = fma(Aj, ga0, Gno);
                Gnn = fma(Aj, ga1, Gnn);
                T1o = fma(Aj, ud0, T1o);
                T1n = fma(Aj, ud1, T1n);
                T2o = fma(Dj, ua0, T2o);
                T2n = fma(Dj, ua1, T2n);
            }
        }
        const double um = side ? Uo : Un, up = side ? Un : Uo;
        const double gnm = side ? Gno : Gnn, gnp = side ? Gnn : Gno;
        const double t1m = side ? T1o : T1n, t1p = side ? T1n : T1o;
        const double t2m = side ? T2o : T2n, t2p = side ? T2n : T2o;
        const double* am = fg + 1;
        const double* ap = fg + 4;
        if (DR) {
            // physical face point (own cell, xi_d = side) and K = x x^T + I
            int lp_, rem_, ig_[3];
            coords(c, lp_, rem_, ig_);
            const double xa_ = sxq[a], xb_ = sxq[bq];
            const double xi0 = d == 0 ? (double)side : xa_;
            const double xi1 = d == 1 ? (double)side : (d == 0 ? xa_ : xb_);
            const double xi2 = d == 2 ? (double)side : xb_;
            const double X0 = (ig_[0] + xi0) * Ms.h[0], X1 = (ig_[1] + xi1) * Ms.h[1], X2 = (ig_[2] + xi2) * Ms.h[2];
            const double Xd = d == 0 ? X0 : (d == 1 ? X1 : X2);
            const double Xt1 = d == 0 ? X1 : X0, Xt2 = d == 2 ? X1 : X2;
            const double hd = Ms.h[d], ht1 = Ms.h[t1], ht2 = Ms.h[t2];
            // (K e)_d for e = d, t1, t2 (K symmetric), scaled to reference derivatives (1/h_e)
            const double ih0 = 1.0 / Ms.h[0], ih1 = 1.0 / Ms.h[1], ih2 = 1.0 / Ms.h[2]; // (loop-invariant: hoisted)
            const double ihd = d == 0 ? ih0 : (d == 1 ? ih1 : ih2), iht1 = t1 == 0 ? ih0 : ih1, iht2 = t2 == 1 ? ih1 : ih2;
            const double kd = (Xd * Xd + 1.0) * ihd, kt1 = Xd * Xt1 * iht1, kt2 = Xd * Xt2 * iht2;
            const double W = sw[a] * sw[bq] * ht1 * ht2;
            const double gam = Ms.gamma[d];
            const double Kgo = kd * Gno + kt1 * T1o + kt2 * T2o; // (K grad u)_d of the own side
            double Cv, s;
            if (fg[15] != 0.0) {
                // boundary face: outer normal sn e_d, [u] = u - g (theta and penalty terms), one-sided flux
                const double sn = side ? 1.0 : -1.0;
                const double jmp = PR == 3 ? Uo : Uo - (X0 * X0 + X1 * X1 + X2 * X2); // Jacobian: g = 0
                Cv = W * (-sn * Kgo + gam * jmp);
                s = -W * jmp * sn;
            } else {
                const double Kgn = kd * Gnn + kt1 * T1n + kt2 * T2n;
                const double jmp = um - up;
                const double Cvm = W * (-0.5 * (Kgo + Kgn) + gam * jmp);
                Cv = side ? Cvm : -Cvm;
                s = -0.5 * W * jmp;
            }
            F2[0 * M2 + p] = Cv;
            F2[1 * M2 + p] = s * kt1;
            F2[2 * M2 + p] = s * kt2;
            F2[3 * M2 + p] = s * kd;
            continue;
        }
        double cF = 1.0;
        if (COEFF) {
            const double xa_ = sxq[a], xb_ = sxq[bq];
            const double xi0 = d == 0 ? 1.0 : xa_;
            const double xi1 = d == 1 ? 1.0 : (d == 0 ? xa_ : xb_);
            const double xi2 = d == 2 ? 1.0 : xb_;
            cF = coeff_sincos(fg[13] + fg[7] * xi0 + fg[8] * xi1 + fg[9] * xi2,
                              fg[14] + fg[10] * xi0 + fg[11] * xi1 + fg[12] * xi2);
        }
        const double gm = cF * (am[d] * gnm + am[t1] * t1m + am[t2] * t2m);
        const double gp = cF * (ap[d] * gnp + ap[t1] * t1p + ap[t2] * t2p);
        const double W = sw[a] * sw[bq] * fg[0];
        const double jump = um - up;
        const double avg = 0.5 * (gm + gp);
        const double gam = Ms.gamma[d];
        const double Cvm = W * (-avg + gam * jump);
        const double Cg = -0.5 * W * jump * cF;
        const double* ao = side ? am : ap;
        F2[0 * M2 + p] = side ? Cvm : -Cvm; // value coefficient of this cell's side
        F2[1 * M2 + p] = ao[t1] * Cg;       // tangential-gradient coefficients (a_self . e_t Cg)
        F2[2 * M2 + p] = ao[t2] * Cg;
        F2[3 * M2 + p] = ao[d] * Cg;        // normal-gradient coefficient
    }
    gsync();
    // ---------------- P5: stage 3a (D0^T / A0^T along j0); face back-projection along t2 ----------------
    {
        using SB = qd::Sw3<M, M, M, 0, N, true, false>; // M^3 -> N x M x M
        constexpr int NLp = kpad(SB::NL);
        for (int t = gtid; t < ncell * 3 * NLp; t += GT) {
            const int c = t / (3 * NLp), k = (t / NLp) % 3, l = t % NLp;
            if (l >= SB::NL) continue;
            double* b = cellp(c);
            if (k == 0) {
                SB::line(b + L::G0, b + L::Z, T.eDt, l); // V
                if (DR) qd::Sw3<M, M, M, 0, N, true, true>::line(b + L::GU, b + L::Z, T.eAt, l); // + A0^T (c u - f)
            }
            else if (k == 1) SB::line(b + L::G1, b + L::Zd1, T.eAt, l); // W1
            else SB::line(b + L::G2, b + L::Zd2, T.eAt, l);             // W2
        }
        // Pv = A^T_t2 Cv + D^T_t2 Ct2, Pt = A^T_t2 Ct1, Pn = A^T_t2 Cn   ([t1 = M][t2 = N])
        using F = qd::Sw2<M, M, 1, N, true, false>;
        using FA = qd::Sw2<M, M, 1, N, true, true>;
        // kind-major (the two-sweep kind 0 first, padded to a warp boundary for n < 6; a group holds one cell)
        constexpr int K0 = 6 * F::NL, K0p = kpad(K0);
        for (int t = rot(ncell * 3 * SB::NL); t < ncell * (K0p + 2 * K0); t += GT) {
            int k, q;
            if (t < K0p) { if (t >= K0) continue; k = 0; q = t; }
            else { k = 1 + (t - K0p) / K0; q = (t - K0p) % K0; }
            const int c = 0, f = q / F::NL, l = q % F::NL;
            double* F1 = f1p(c, f);
            const double* C = cfp(c, f);
            if (k == 0) { F::line(C + 0 * M2, F1 + 0 * NM, T.eAt, l); FA::line(C + 2 * M2, F1 + 0 * NM, T.eDt, l); }
            else if (k == 1) F::line(C + 1 * M2, F1 + 1 * NM, T.eAt, l);
            else F::line(C + 3 * M2, F1 + 2 * NM, T.eAt, l);
        }
    }
    gsync();
    // ---------------- P6: stage 3b (along j1); face back-projection along t1 ----------------
    {
        using SA = qd::Sw3<N, M, M, 1, N, true, false>;  // N x M x M -> N x N x M
        using SAa = qd::Sw3<N, M, M, 1, N, true, true>;
        constexpr int NLp = kpad(SA::NL);
        for (int t = gtid; t < ncell * 2 * NLp; t += GT) {
            const int c = t / (2 * NLp), k = (t / NLp) % 2, l = t % NLp;
            if (l >= SA::NL) continue;
            double* b = cellp(c);
            if (k == 0) { SA::line(b + L::Z, b + L::Y2, T.eAt, l); SAa::line(b + L::Zd1, b + L::Y2, T.eDt, l); } // Ya
            else SA::line(b + L::Zd2, b + L::Y2d, T.eAt, l);                                                   // Yb
        }
        // V2 = A^T_t1 Pv + D^T_t1 Pt, G2 = A^T_t1 Pn   ([t1 = N][t2 = N], into FT)
        using F = qd::Sw2<M, N, 0, N, true, false>;
        using FA = qd::Sw2<M, N, 0, N, true, true>;
        constexpr int K0 = 6 * F::NL, K0p = kpad(K0);
        for (int t = rot(ncell * 2 * SA::NL); t < ncell * (K0p + K0); t += GT) {
            int k, q;
            if (t < K0p) { if (t >= K0) continue; k = 0; q = t; }
            else { k = 1; q = t - K0p; }
            const int c = 0, f = q / F::NL, l = q % F::NL;
            double* FT = ftp(c, f);
            const double* P = f1p(c, f);
            if (k == 0) { F::line(P + 0 * NM, FT, T.eAt, l); FA::line(P + 1 * NM, FT, T.eDt, l); }
            else F::line(P + 2 * NM, FT + N2, T.eAt, l);
        }
    }
    gsync();
    // ---------------- P7: stage 3c (along j2) into R ----------------
    {
        using S = qd::Sw3<N, N, M, 2, N, true, false>;
        using Sa = qd::Sw3<N, N, M, 2, N, true, true>;
        for (int t = gtid; t < ncell * S::NL; t += GT) {
            const int c = t / S::NL, l = t % S::NL;
            double* b = cellp(c);
            S::line(b + L::Y2, b + L::R, T.eAt, l);
            Sa::line(b + L::Y2d, b + L::R, T.eDt, l);
        }
    }
    gsync();
    // ---------------- P8: add the face back-projections along the normals, write r once ----------------
    for (int t = gtid; t < ncell * N3; t += GT) {
        const int c = t / N3, P = t % N3;
        const int j[3] = {P % N, (P / N) % N, P / N2};
        double v = cellp(c)[L::R + P];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
            const int p = j[t1] + N * j[t2];
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                const double* FT = ftp(c, 2 * d + side);
                const double e = side ? se1[j[d]] : se0[j[d]], dd = side ? sd1[j[d]] : sd0[j[d]];
                v = fma(e, FT[p], fma(dd, FT[N2 + p], v));
            }
        }
        r[(cfirst + c) * N3 + P] = v;
    }
}

} // namespace dg
