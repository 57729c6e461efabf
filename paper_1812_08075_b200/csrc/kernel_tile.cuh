// K_tile: the general sum-factorised SIPG operator (any degree, per-cell affine geometry, c(x))
// as a marching-tile kernel — the path of the affine configs (cfg2 Q5, cfg4 Q4) and of the
// axis-aligned configs other than Q7.
//
// A CTA owns a T1 x T2 tile of cells in (i1, i2) and marches along i0 through the planes
// [p_begin, p_end); the blocks of plane s+1 arrive by 1D bulk TMA (cp.async.bulk, one copy per
// tile row) into a double buffer while plane s is computed. Per plane (P = paper passages):
//   P1  stage 1 (Alg. assembly part 1): grad_hat U = D along d of X (collocation:
//       U = X), and from the same line in registers its traces u, d_n u at both ends (1-point
//       face tables e0/e1, d0/d1); traces of the neighbours outside the tile (ring
//       cells in-plane, the next plane's lower ends).
//   P2  stage 2 (part 2): Q = w_q c(x_q) |det J| J^{-1} J^{-T} grad_hat U, pointwise,
//       with c(x) from per-cell factorised exponentials; tangential derivatives of every face
//       u-trace by D on the face.
//   P3  SIPG fluxes (Eq. diffreac_weak, theta = -1), each face ONCE where both cells
//       are on this CTA (T- = lower cell; geometry from T-, reading R11); faces to cells of other
//       CTAs are evaluated for this CTA's side only; the face to the next plane is evaluated at
//       this step and its T+ half carried to the next step.
//   P4  V = Cv + D^T-tangential(a_t Cg) on every face side.
//   P5  stage 3 (part 3) fused with the face back-projection, per line along d:
//       r_line = D^T Q_d,line + e_lo V_lo + d_lo G_lo + e_hi V_hi + d_hi G_hi, summed over d;
//       the d = 0 pass writes r once.
// Geometry per cell comes precomputed by dg_setup (k_geom): G~ = |det J| J^{-1} J^{-T}, the rows
// of J that map to x0, x1 (for c), and for each upper face (cell = T-): dS, a- = J_-^{-1} n_F,
// a+ = J_+^{-1} n_F.
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

// (ar + i ai)(br + i bi)
__device__ __forceinline__ void cmul(double ar, double ai, double br, double bi, double& cr, double& ci)
{
    cr = fma(ar, br, -ai * bi);
    ci = fma(ar, bi, ai * br);
}

template <int N, int T1, int T2>
struct Lay {
    static constexpr int N2 = N * N, N3 = N * N * N, NC = T1 * T2;
    static constexpr int NACT = NC * N2;     // threads with a fixed (cell, a, b)
    static constexpr int NR = 2 * (T1 + T2); // ring cells: d=1 low[T2] high[T2], d=2 low[T1] high[T1]
    // face slots (N2 points each, 4 quantity arrays):
    //   own cells: slot c*6 + 2*d + side   (side 0: lower face, 1: upper face)
    //   ring:      slot 6 NC + r           (the ring cell's side facing the tile)
    //   next:      slot 6 NC + NR + c      (the lower face of the next-plane cell above c)
    static constexpr int NS = 6 * NC + NR + NC;
    static constexpr int QSZ = NS * N2;
    static constexpr int CXSZ = 2 * 3 * (N + 1) * 2; // c(x) tables per cell: [coord k][axis b][q = 0..N] complex
    // offsets in doubles
    static constexpr int XB = 0;                       // current plane (TMA)
    static constexpr int G = XB + NC * N3;             // 3 arrays: grad_hat U -> flux Q -> partial residuals
    static constexpr int TQ = G + 3 * NC * N3;         // 4 arrays: u|Cv|V, gn|G, gt1|Ct1, gt2|Ct2
    static constexpr int PEND = TQ + 4 * QSZ;          // 2 (ping-pong) x {V+, G+} x [NC][N2]
    static constexpr int GEO = PEND + 2 * 2 * NC * N2; // geometry records of own [NC] and ring [NR] cells
    static constexpr int CX = GEO + (NC + NR) * GREC;
    static constexpr int CO = CX + (NC + NR) * CXSZ;  // origin phases e^{2 pi i o_k}, k = 0, 1
    static constexpr int END = CO + (NC + NR) * 4;
    static constexpr int BYTES = END * 8 + 64;
};

} // namespace tl

// Thread mapping: thread t < NC N2 owns cell c = t / N2 of the tile and the position (a, b) = (t % N, t / N % N)
// of the cell's lines in every direction and of every face of the cell; all per-thread loops below run
// over compile-time directions / quadrature indices (no per-task index arithmetic).
template <int N, bool AFFINE, bool COEFF, int T1, int T2, int NT>
__global__ void __launch_bounds__(NT)
k_tile(const double* __restrict__ x, const double* __restrict__ xb, const double* __restrict__ xa,
       double* __restrict__ r, int p_begin, int p_end, const Tab<N> T, const MeshArgs M, const double* __restrict__ geo)
{
    using Y = tl::Lay<N, T1, T2>;
    constexpr int N2 = Y::N2, N3 = Y::N3, NC = Y::NC, NR = Y::NR, QSZ = Y::QSZ;
    constexpr int SNEXT = 6 * NC + NR; // first "next" slot
    static_assert(Y::NACT <= NT, "one thread per (cell, line position)");
    extern __shared__ __align__(16) double sm[];
    double* const XB = sm + Y::XB;
    double* const G = sm + Y::G;
    double* const TQ = sm + Y::TQ;
    double* const GEO = sm + Y::GEO;
    double* const CX = sm + Y::CX;
    double* const CO = sm + Y::CO;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + Y::END);
    __shared__ double sD[N * N], sW[N], sXi[N + 1];

    const int tid = threadIdx.x;
    const int ntile2 = M.N2 / T2;
    const int ti1 = blockIdx.x / ntile2, ti2 = blockIdx.x % ntile2;
    const int PC = M.plane_cells;
    const int nsteps = p_end - p_begin;
    if (nsteps <= 0) return;
    auto cidx = [&](int lp, int i1, int i2) -> long long { return (long long)lp * PC + (long long)i1 * M.N2 + i2; };
    auto gidx = [&](int lp, int i1, int i2) -> long long { return (long long)(lp + 1) * PC + (long long)i1 * M.N2 + i2; };
    auto wrap = [](int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); };
    auto Q = [&](int q, int slot) { return TQ + q * QSZ + slot * N2; };

    // fixed thread coordinates
    const bool act = tid < Y::NACT;
    const int mc = act ? tid / N2 : 0, mab = act ? tid % N2 : 0, ma = mab % N, mb = mab / N;
    const int mc1 = mc / T2, mc2 = mc % T2;
    const long long minpl = (long long)(ti1 * T1 + mc1) * M.N2 + ti2 * T2 + mc2; // in-plane index of cell mc

    for (int i = tid; i < N * N; i += NT) sD[i] = T.D[i];
    for (int i = tid; i < N; i += NT) { sW[i] = T.w[i]; sXi[i] = T.xi[i]; }
    if (tid == 0) {
        sXi[N] = 1.0;
        tl::mbar_init(&bar[0], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int step) {
        const int lp = p_begin + step;
        tl::mbar_expect_tx(&bar[0], NC * N3 * 8);
#pragma unroll
        for (int c1 = 0; c1 < T1; ++c1)
            tl::bulk_g2s(XB + c1 * T2 * N3, x + cidx(lp, ti1 * T1 + c1, ti2 * T2) * N3, T2 * N3 * 8, &bar[0]);
    };
    if (tid == 0) issue(0);

    // ring cell rr -> in-plane (i1, i2), the face direction it borders, and whether it is below the tile
    auto ring_cell = [&](int rr, int& i1, int& i2, int& d, bool& low) {
        if (rr < 2 * T2) {
            d = 1;
            low = rr < T2;
            const int c2 = low ? rr : rr - T2;
            i1 = low ? wrap(ti1 * T1 - 1, M.N1) : wrap(ti1 * T1 + T1, M.N1);
            i2 = ti2 * T2 + c2;
        } else {
            const int q = rr - 2 * T2;
            d = 2;
            low = q < T1;
            const int c1 = low ? q : q - T1;
            i1 = ti1 * T1 + c1;
            i2 = low ? wrap(ti2 * T2 - 1, M.N2) : wrap(ti2 * T2 + T2, M.N2);
        }
    };

    // c(x) at a point of the cell in table slot cc; q0, q1, q2 index sXi (N = the face coordinate 1)
    auto cval = [&](int cc, int q0, int q1, int q2) -> double {
        const double* cx = CX + cc * Y::CXSZ;
        double z[2][2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const double* e0 = cx + ((k * 3 + 0) * (N + 1) + q0) * 2;
            const double* e1 = cx + ((k * 3 + 1) * (N + 1) + q1) * 2;
            const double* e2 = cx + ((k * 3 + 2) * (N + 1) + q2) * 2;
            double tr, ti, ur, ui;
            tl::cmul(CO[cc * 4 + 2 * k], CO[cc * 4 + 2 * k + 1], e0[0], e0[1], tr, ti);
            tl::cmul(tr, ti, e1[0], e1[1], ur, ui);
            tl::cmul(ur, ui, e2[0], e2[1], z[k][0], z[k][1]);
        }
        return 1.0 + 0.5 * z[0][1] * z[1][0]; // 1 + 0.5 sin(2 pi x0) cos(2 pi x1)  (reading R13)
    };
    constexpr int NE = 2 * 3 * (N + 1);
    auto ctab_task = [&](int cc, int rem, int g0, int i1) {
        double sv, cv;
        if (rem < NE) {
            const int k = rem / (3 * (N + 1)), rem2 = rem % (3 * (N + 1)), bax = rem2 / (N + 1), q = rem2 % (N + 1);
            const double Jkb = AFFINE ? GEO[cc * GREC + 6 + 3 * k + bax] : (bax == k ? M.h[k] : 0.0);
            sincospi(2.0 * Jkb * sXi[q], &sv, &cv);
            double* e = CX + cc * Y::CXSZ + ((k * 3 + bax) * (N + 1) + q) * 2;
            e[0] = cv;
            e[1] = sv;
        } else {
            const int k = rem - NE;
            const double o = k == 0 ? (double)g0 / M.N0 : (double)i1 / M.N1;
            sincospi(2.0 * o, &sv, &cv);
            CO[cc * 4 + 2 * k] = cv;
            CO[cc * 4 + 2 * k + 1] = sv;
        }
    };
    // tangential derivatives (D on the face) of the u-trace of slot `slot` at point (a, b)
    auto tangential = [&](int slot, int a, int b) {
        const double* U = Q(0, slot);
        double v1 = 0.0, v2 = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            v1 = fma(sD[a * N + j], U[j + N * b], v1);
            v2 = fma(sD[b * N + j], U[a + N * j], v2);
        }
        Q(2, slot)[a + N * b] = v1;
        Q(3, slot)[a + N * b] = v2;
    };
    // same with the thread's D rows in registers (Da = D[a][.], Db = D[b][.])
    auto tangential_r = [&](int slot, int a, int b, const double* Da, const double* Db) {
        const double* U = Q(0, slot);
        double v1 = 0.0, v2 = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            v1 = fma(Da[j], U[j + N * b], v1);
            v2 = fma(Db[j], U[a + N * j], v2);
        }
        Q(2, slot)[a + N * b] = v1;
        Q(3, slot)[a + N * b] = v2;
    };
    // V with the thread's D columns in registers (Ca = D[.][a], Cb = D[.][b])
    auto vface_r = [&](int slot, int a, int b, const double* Ca, const double* Cb) -> double {
        double v = Q(0, slot)[a + N * b];
        if (AFFINE) {
            const double* C1 = Q(2, slot);
            const double* C2 = Q(3, slot);
#pragma unroll
            for (int j = 0; j < N; ++j) {
                v = fma(Ca[j], C1[j + N * b], v);
                v = fma(Cb[j], C2[a + N * j], v);
            }
        }
        return v;
    };
    // V = Cv + D^T_t1 Ct1 + D^T_t2 Ct2 at point (a, b) of a slot
    auto vface = [&](int slot, int a, int b) -> double {
        double v = Q(0, slot)[a + N * b];
        if (AFFINE) {
            const double* C1 = Q(2, slot);
            const double* C2 = Q(3, slot);
#pragma unroll
            for (int j = 0; j < N; ++j) {
                v = fma(sD[j * N + a], C1[j + N * b], v);
                v = fma(sD[j * N + b], C2[a + N * j], v);
            }
        }
        return v;
    };
    // SIPG flux at point (a, b) of the face with normal d between slots sMinus (T-) and sPlus (T+);
    // geometry / c tables from cell-record slot gs (= T-). Writes the coefficients (Cv, G, Ct1, Ct2)
    // of the requested sides into their own slots (read-before-write of the same point only).
    auto face = [&](int d, int a, int b, int sMinus, int sPlus, int gs, bool wMinus, bool wPlus) {
        const int ab = a + N * b;
        const double jump = Q(0, sMinus)[ab] - Q(0, sPlus)[ab];
        const double gmd = Q(1, sMinus)[ab], gpd = Q(1, sPlus)[ab];
        double cF = 1.0;
        if (COEFF) {
            const int q0 = (d == 0) ? N : a, q1 = (d == 1) ? N : (d == 0 ? a : b), q2 = (d == 2) ? N : b;
            cF = cval(gs, q0, q1, q2); // x_F on the T- cell at xi_d = 1
        }
        const double gam = d == 0 ? M.gamma[0] : (d == 1 ? M.gamma[1] : M.gamma[2]);
        double Cvm, Cvp, Cg, am_d, am_t1, am_t2, ap_d, ap_t1, ap_t2;
        if (!AFFINE) {
            const double hd = d == 0 ? M.h[0] : (d == 1 ? M.h[1] : M.h[2]);
            const double W = sW[a] * sW[b] * (M.h[0] * M.h[1] * M.h[2] / hd);
            const double avg = 0.5 * cF * (gmd + gpd) / hd;
            Cvm = W * (-avg + gam * jump);
            Cvp = W * (avg - gam * jump);
            Cg = -0.5 * W * jump * cF;
            am_d = ap_d = 1.0 / hd;
            am_t1 = am_t2 = ap_t1 = ap_t2 = 0.0;
        } else {
            const double* f = GEO + gs * GREC + 12 + 8 * d;
            am_t1 = f[0];
            ap_t1 = f[1];
            am_t2 = f[2];
            ap_t2 = f[3];
            am_d = f[4];
            ap_d = f[5];
            const double gm = cF * (am_d * gmd + am_t1 * Q(2, sMinus)[ab] + am_t2 * Q(3, sMinus)[ab]);
            const double gp = cF * (ap_d * gpd + ap_t1 * Q(2, sPlus)[ab] + ap_t2 * Q(3, sPlus)[ab]);
            const double avg = 0.5 * (gm + gp);
            const double W = sW[a] * sW[b] * f[6];
            Cvm = W * (-avg + gam * jump);
            Cvp = W * (avg - gam * jump);
            Cg = -0.5 * W * jump * cF;
        }
        if (wMinus) {
            Q(0, sMinus)[ab] = Cvm;
            Q(1, sMinus)[ab] = am_d * Cg;
            Q(2, sMinus)[ab] = am_t1 * Cg;
            Q(3, sMinus)[ab] = am_t2 * Cg;
        }
        if (wPlus) {
            Q(0, sPlus)[ab] = Cvp;
            Q(1, sPlus)[ab] = ap_d * Cg;
            Q(2, sPlus)[ab] = ap_t1 * Cg;
            Q(3, sPlus)[ab] = ap_t2 * Cg;
        }
    };

    // ---------------- prologue: the lower d=0 face of plane p_begin (T- = plane p_begin - 1) ----------------
    // Evaluated once here; its T+ half (V+, G+) is left in PEND[0] exactly as a regular step leaves it.
    // Temporary slot use: T- traces -> "next" slots, T+ traces -> own lower d0 slots, T- geometry / c
    // tables -> own-cell slots.
    int pend = 0;
    {
        const int lpm = p_begin - 1;
        const int g0m = wrap(M.plane_begin + lpm, M.N0);
        if (act) {
#pragma unroll
            for (int which = 0; which < 2; ++which) {
                const double* src = which ? x + (cidx(p_begin, 0, 0) + minpl) * N3
                                          : ((p_begin == 0) ? xb + minpl * N3 : x + (cidx(lpm, 0, 0) + minpl) * N3);
                double u = 0.0, g = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    const double v = __ldg(src + pidx<N>(0, j, ma, mb));
                    u = fma(which ? T.e0[j] : T.e1[j], v, u);
                    g = fma(which ? T.d0[j] : T.d1[j], v, g);
                }
                const int slot = which ? mc * 6 + 0 : SNEXT + mc;
                Q(0, slot)[mab] = u;
                Q(1, slot)[mab] = g;
            }
        }
        if (AFFINE) {
            for (int t = tid; t < NC * GREC; t += NT) {
                const int c = t / GREC, k = t % GREC;
                GEO[t] = __ldg(geo + gidx(lpm, ti1 * T1 + c / T2, ti2 * T2 + c % T2) * GREC + k);
            }
        }
        __syncthreads();
        if (COEFF)
            for (int t = tid; t < NC * (NE + 2); t += NT) ctab_task(t / (NE + 2), t % (NE + 2), g0m, ti1 * T1 + (t / (NE + 2)) / T2);
        if (AFFINE && act) {
            tangential(mc * 6 + 0, ma, mb);
            tangential(SNEXT + mc, ma, mb);
        }
        __syncthreads();
        if (act) {
            // face below cell mc; T- = cell below (record / c tables in own slot mc), T+ = mc
            face(0, ma, mb, SNEXT + mc, mc * 6 + 0, mc, false, true);
        }
        __syncthreads();
        double* P = sm + Y::PEND;
        if (act) {
            P[mc * N2 + mab] = vface(mc * 6 + 0, ma, mb);
            P[NC * N2 + mc * N2 + mab] = Q(1, mc * 6 + 0)[mab];
        }
        __syncthreads();
    }

    for (int s = 0; s < nsteps; ++s) {
        const int lp = p_begin + s;
        const int ig0 = wrap(M.plane_begin + lp, M.N0);
        const bool lastp = (s == nsteps - 1);
        const double* Pin = sm + Y::PEND + pend * 2 * NC * N2;  // lower d=0 face of this plane (from last step)
        double* Pout = sm + Y::PEND + (pend ^ 1) * 2 * NC * N2; // lower d=0 face of the next plane

        // ---------------- P0: geometry records (own + ring), c(x) tables ----------------
        if (AFFINE) {
            for (int t = tid; t < (NC + NR) * GREC; t += NT) {
                const int cc = t / GREC, k = t % GREC;
                int i1, i2;
                if (cc < NC) { i1 = ti1 * T1 + cc / T2; i2 = ti2 * T2 + cc % T2; }
                else { int d_; bool lo_; ring_cell(cc - NC, i1, i2, d_, lo_); }
                GEO[t] = __ldg(geo + gidx(lp, i1, i2) * GREC + k);
            }
            if (COEFF) __syncthreads();
        }
        if (COEFF) {
            for (int t = tid; t < (NC + NR) * (NE + 2); t += NT) {
                const int cc = t / (NE + 2);
                int i1, i2;
                if (cc < NC) { i1 = ti1 * T1 + cc / T2; i2 = ti2 * T2 + cc % T2; }
                else { int d_; bool lo_; ring_cell(cc - NC, i1, i2, d_, lo_); }
                ctab_task(cc, t % (NE + 2), ig0, i1);
            }
        }
        tl::mbar_wait(&bar[0], s & 1);
        __syncthreads();

        // ---------------- P1: stage 1 + own traces (fixed mapping); next-plane traces; ring traces ----------------
        if (act) {
            const double* xc = XB + mc * N3;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                double v[N];
#pragma unroll
                for (int j = 0; j < N; ++j) v[j] = xc[pidx<N>(d, j, ma, mb)];
                double* gd = G + (d * NC + mc) * N3;
                double u0 = 0, u1 = 0, g0 = 0, g1 = 0;
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    u0 = fma(T.e0[j], v[j], u0);
                    u1 = fma(T.e1[j], v[j], u1);
                    g0 = fma(T.d0[j], v[j], g0);
                    g1 = fma(T.d1[j], v[j], g1);
                }
#pragma unroll
                for (int q = 0; q < N; ++q) {
                    double acc = 0.0;
#pragma unroll
                    for (int j = 0; j < N; ++j) acc = fma(T.D[q * N + j], v[j], acc);
                    gd[pidx<N>(d, q, ma, mb)] = acc;
                }
                Q(0, mc * 6 + 2 * d + 0)[mab] = u0;
                Q(0, mc * 6 + 2 * d + 1)[mab] = u1;
                Q(1, mc * 6 + 2 * d + 0)[mab] = g0;
                Q(1, mc * 6 + 2 * d + 1)[mab] = g1;
            }
            // the lower end of the line above (next plane; halo x_above at the slab's last plane)
            const double* src = !lastp ? x + (cidx(lp + 1, 0, 0) + minpl) * N3
                                       : ((p_end == M.L) ? xa + minpl * N3 : x + (cidx(p_end, 0, 0) + minpl) * N3);
            double u = 0, g = 0;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double v = __ldg(src + pidx<N>(0, j, ma, mb));
                u = fma(T.e0[j], v, u);
                g = fma(T.d0[j], v, g);
            }
            Q(0, SNEXT + mc)[mab] = u;
            Q(1, SNEXT + mc)[mab] = g;
        }
        for (int t = tid; t < NR * N2; t += NT) {
            const int rr = t / N2, ab = t % N2, a = ab % N, b = ab / N;
            int i1, i2, d;
            bool low;
            ring_cell(rr, i1, i2, d, low);
            const double* src = x + cidx(lp, i1, i2) * N3;
            double u = 0, g = 0;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double v = __ldg(src + pidx<N>(d == 1 ? 1 : 2, j, a, b));
                u = fma(low ? T.e1[j] : T.e0[j], v, u); // a ring cell below the tile faces it with its upper end
                g = fma(low ? T.d1[j] : T.d0[j], v, g);
            }
            Q(0, 6 * NC + rr)[ab] = u;
            Q(1, 6 * NC + rr)[ab] = g;
        }
        __syncthreads();
        // the plane buffer is no longer read this step: stream the next plane in behind the compute
        if (tid == 0 && s + 1 < nsteps) issue(s + 1);

        // ---------------- P2: flux transform at (a, b, q); tangential derivatives ----------------
        if (act) {
            double gt[6];
#pragma unroll
            for (int i = 0; i < 6; ++i) gt[i] = AFFINE ? GEO[mc * GREC + i] : 0.0;
            // c(x) at (a, b, q) = 1 + 0.5 Im(z0 E02[q]) Re(z1 E12[q]) with z_k = e^{2 pi i o_k} E_k0[a] E_k1[b]
            double z0r = 0, z0i = 0, z1r = 0, z1i = 0;
            if (COEFF) {
                const double* cx = CX + mc * Y::CXSZ;
                double tr, ti;
                tl::cmul(CO[mc * 4 + 0], CO[mc * 4 + 1], cx[((0 * 3 + 0) * (N + 1) + ma) * 2], cx[((0 * 3 + 0) * (N + 1) + ma) * 2 + 1], tr, ti);
                tl::cmul(tr, ti, cx[((0 * 3 + 1) * (N + 1) + mb) * 2], cx[((0 * 3 + 1) * (N + 1) + mb) * 2 + 1], z0r, z0i);
                tl::cmul(CO[mc * 4 + 2], CO[mc * 4 + 3], cx[((1 * 3 + 0) * (N + 1) + ma) * 2], cx[((1 * 3 + 0) * (N + 1) + ma) * 2 + 1], tr, ti);
                tl::cmul(tr, ti, cx[((1 * 3 + 1) * (N + 1) + mb) * 2], cx[((1 * 3 + 1) * (N + 1) + mb) * 2 + 1], z1r, z1i);
            }
            const double wab = sW[ma] * sW[mb];
            double* g0 = G + (0 * NC + mc) * N3;
            double* g1 = G + (1 * NC + mc) * N3;
            double* g2 = G + (2 * NC + mc) * N3;
#pragma unroll
            for (int q = 0; q < N; ++q) {
                const int P = mab + N2 * q;
                double cW = wab * T.w[q];
                if (COEFF) {
                    const double* cx = CX + mc * Y::CXSZ;
                    const double* e0 = cx + ((0 * 3 + 2) * (N + 1) + q) * 2;
                    const double* e1 = cx + ((1 * 3 + 2) * (N + 1) + q) * 2;
                    const double s0 = fma(z0r, e0[1], z0i * e0[0]);  // Im(z0 e0) = sin(2 pi x0)
                    const double c1 = fma(z1r, e1[0], -z1i * e1[1]); // Re(z1 e1) = cos(2 pi x1)
                    cW *= fma(0.5 * s0, c1, 1.0);
                }
                const double a0 = g0[P], a1 = g1[P], a2 = g2[P];
                if (AFFINE) {
                    g0[P] = cW * (gt[0] * a0 + gt[3] * a1 + gt[4] * a2);
                    g1[P] = cW * (gt[3] * a0 + gt[1] * a1 + gt[5] * a2);
                    g2[P] = cW * (gt[4] * a0 + gt[5] * a1 + gt[2] * a2);
                } else {
                    const double adet = M.h[0] * M.h[1] * M.h[2];
                    g0[P] = cW * (adet / (M.h[0] * M.h[0])) * a0;
                    g1[P] = cW * (adet / (M.h[1] * M.h[1])) * a1;
                    g2[P] = cW * (adet / (M.h[2] * M.h[2])) * a2;
                }
            }
            if (AFFINE) {
                double Da[N], Db[N];
#pragma unroll
                for (int j = 0; j < N; ++j) { Da[j] = sD[ma * N + j]; Db[j] = sD[mb * N + j]; }
#pragma unroll
                for (int f = 1; f < 6; ++f) tangential_r(mc * 6 + f, ma, mb, Da, Db); // the lower d0 side is pending
                tangential_r(SNEXT + mc, ma, mb, Da, Db);
            }
        }
        if (AFFINE) {
            for (int t = tid; t < NR * N2; t += NT) {
                const int rr = t / N2, ab = t % N2;
                tangential(6 * NC + rr, ab % N, ab / N);
            }
        }
        __syncthreads();

        // ---------------- P3: face fluxes (each face once on this CTA) ----------------
        if (act) {
            // upper faces of cell mc (T- = mc)
            face(0, ma, mb, mc * 6 + 1, SNEXT + mc, mc, true, true);
            {
                const bool in = mc1 + 1 < T1;
                const int sp = in ? ((mc1 + 1) * T2 + mc2) * 6 + 2 : 6 * NC + T2 + mc2;
                face(1, ma, mb, mc * 6 + 3, sp, mc, true, in);
            }
            {
                const bool in = mc2 + 1 < T2;
                const int sp = in ? (mc1 * T2 + mc2 + 1) * 6 + 4 : 6 * NC + 2 * T2 + T1 + mc1;
                face(2, ma, mb, mc * 6 + 5, sp, mc, true, in);
            }
            // lower faces on the tile's low boundary (T- = ring cell below)
            if (mc1 == 0) face(1, ma, mb, 6 * NC + mc2, mc * 6 + 2, NC + mc2, false, true);
            if (mc2 == 0) face(2, ma, mb, 6 * NC + 2 * T2 + mc1, mc * 6 + 4, NC + 2 * T2 + mc1, false, true);
            // the lower d=0 side was evaluated on the previous step: V+, G+
            Q(0, mc * 6 + 0)[mab] = Pin[mc * N2 + mab];
            Q(1, mc * 6 + 0)[mab] = Pin[NC * N2 + mc * N2 + mab];
        }
        __syncthreads();

        // ---------------- P4: V on every own side (in place of Cv) and on the next plane's T+ half ----------------
        if (act) {
            double Ca[N], Cb[N];
#pragma unroll
            for (int j = 0; j < N; ++j) { Ca[j] = sD[j * N + ma]; Cb[j] = sD[j * N + mb]; }
            double v[6];
#pragma unroll
            for (int f = 1; f < 6; ++f) v[f] = vface_r(mc * 6 + f, ma, mb, Ca, Cb);
            const double vn = vface_r(SNEXT + mc, ma, mb, Ca, Cb);
            // (other threads read only Ct1 / Ct2 of these slots, never Cv: in-place update is safe)
#pragma unroll
            for (int f = 1; f < 6; ++f) Q(0, mc * 6 + f)[mab] = v[f];
            Pout[mc * N2 + mab] = vn;
            Pout[NC * N2 + mc * N2 + mab] = Q(1, SNEXT + mc)[mab];
        }
        __syncthreads();

        // ---------------- P5: stage 3 + face back-projection; passes d = 1, 2 (in place), 0 (to r) ----------------
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {
            const int d = (pass == 2) ? 0 : pass + 1;
            if (act) {
                double* qd = G + (d * NC + mc) * N3;
                double q[N];
#pragma unroll
                for (int j = 0; j < N; ++j) q[j] = qd[pidx<N>(d, j, ma, mb)];
                const double Vl = Q(0, mc * 6 + 2 * d + 0)[mab], Vh = Q(0, mc * 6 + 2 * d + 1)[mab];
                const double Gl = Q(1, mc * 6 + 2 * d + 0)[mab], Gh = Q(1, mc * 6 + 2 * d + 1)[mab];
                const double* prev = G + ((pass == 1 ? 1 : 2) * NC + mc) * N3; // partial sums of the earlier passes
                double* dst = r + (cidx(lp, 0, 0) + minpl) * N3;
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    double acc = fma(T.e0[i], Vl, fma(T.d0[i], Gl, fma(T.e1[i], Vh, T.d1[i] * Gh)));
#pragma unroll
                    for (int j = 0; j < N; ++j) acc = fma(T.D[j * N + i], q[j], acc);
                    const int P = pidx<N>(d, i, ma, mb);
                    if (pass == 0) qd[P] = acc;                 // R1 in place of Q1
                    else if (pass == 1) qd[P] = acc + prev[P];  // R1 + R2 in place of Q2
                    else dst[P] = acc + prev[P];                // r = R1 + R2 + R0
                }
            }
            __syncthreads();
        }
        pend ^= 1;
    }
}

} // namespace dg
