// k_stokes: the residual of the paper's Stokes problem (Eq. stokes_weak;
// DESIGN.md readings R27/R28), axiparallel mesh of (0,1)^3, mu = 1, theta = -1:
//
//   volume   (grad u, grad v) - (p, div v) - (div u, q)
//   faces    -({grad u} n, [v]) + theta([u], {grad v} n) + gamma([u], [v]) + ({p}, [v].n) + ([u].n, {q})
//            on interior and Dirichlet faces (Gamma_D = boundary without x_0 = 1), with
//            -theta(g, grad v n) - gamma(g, v) - (g.n, q) on Dirichlet faces, g = (4 x_1 (1 - x_1), 0, 0);
//            the Neumann face x_0 = 1 has no terms.
//
// Velocity Q_k collocated on the n = k+1 Gauss points (A = I; gradients by D sweeps), pressure Q_{k-1}
// (n-1 Gauss nodes) interpolated to the points by A_p = [psi_j(xi_q)] sweeps and tested with A_p^T: the
// velocity and pressure evaluations are the stacked stage 1 of the paper (Eq. fusedtensor: 9
// gradient sweeps of 3 components + 3 interpolation sweeps of the pressure from one staging of the cell).
// Faces: traces along the normal with the 1-point tables, the pressure additionally
// interpolated tangentially to the face points; each cell evaluates its 6 faces (neighbour traces from
// L2) and writes its rows once. Cell-centric, one cell per CTA, every contraction a 1D sweep of the
// shared qd::Sw3 / qd::Sw2 helpers. Correctness-first (like k_quad).
#pragma once

#include "common.cuh"
#include "kernel_quad.cuh" // qd::Sw3 / Sw2, EOMat
#include "kernel_quad.cuh"

namespace dg {

template <int N>
struct STab {
    static constexpr int NP = N - 1;
    double D[N * N];    // D[q*N + j] = l_j'(xi_q)  (velocity basis, collocated)
    double AP[N * NP];  // AP[q*NP + j] = psi_j(xi_q)  (pressure basis at the velocity nodes)
    double w[N], xi[N];
    double e0[N], e1[N], d0[N], d1[N];
    double ep0[NP], ep1[NP];
    EOMat<N, N, -1> eD;    // D, D^T, AP, AP^T in even/odd form (kernel_quad.cuh, EOMat): the sweeps
    EOMat<N, N, -1> eDt;
    EOMat<N, NP, 1> eAP;
    EOMat<NP, N, 1> eAPt;
};

namespace sk {
template <int N>
struct SLay {
    static constexpr int NP = N - 1;
    static constexpr int N2 = N * N, N3 = N * N * N, NP2 = NP * NP, NP3 = NP * NP * NP;
    static constexpr int B = 3 * N3 + NP3; // DOFs per cell: [u_0 | u_1 | u_2 | p]
    // n <= 3: one round of the 9 n^2 gradient lines (measured: k = 2 1.52 -> 1.26 ms); n = 4, 5: 128 (k = 4:
    // 1.24 -> 1.11 ms on 40^3); else 256
    static constexpr int NT = N <= 3 ? (9 * N * N + 31) / 32 * 32 : (N <= 5 ? 128 : 256);
    // velocity / gradient blocks: point (j0, j1, j2) at j0 + N j1 + PS j2. n = 4: PS = 20, so that the 16 lines of a
    // j1-sweep (lanes (j0, j2), stride 4 along the line) fall on 16 distinct banks (dense: 4-way conflicts); the
    // j2-sweeps stay conflict-free
    static constexpr int PS = N == 4 ? 20 : N2;
    static constexpr int NB = N * PS;
    // per-cell shared buffers (doubles)
    static constexpr int U = 0;            // velocity (3 blocks of NB), later the velocity residual RU
    static constexpr int PR = U + 3 * NB;  // pressure (NP3), later the pressure residual RP
    static constexpr int G = PR + (NP3 + 1) / 2 * 2; // 9 reference gradients [c][e] (NB each, 16-B aligned), later the fluxes Q[c][e]
    static constexpr int PQ = G + 9 * NB;  // p at the points (dense N3), later -W div u
    static constexpr int TA = PQ + N3;     // [NP][NP][N]
    static constexpr int TB = TA + NP2 * N; // [NP][N][N]
    // per face: TR [3][4][N2] (own u, own du/dn_hat, nb u, nb du/dn_hat) -> coefficients Cv = TR[c][0],
    //           Cn = TR[c][1]; PT [2][NP2] (own, nb p traces) -> CQ2 = PT[0]; PF1 [2][N NP] -> CQ1 = PF1[0];
    //           PF2 [2][N2] (own, nb p at the face points) -> Cq = PF2[0]
    static constexpr int TR = 0, PT = 12 * N2, PF1 = PT + 2 * NP2, PF2 = PF1 + 2 * N * NP;
    static constexpr int FACE = PF2 + 2 * N2;
    static constexpr int F = TB + NP * N2;
    static constexpr int END = F + 6 * FACE;
    static constexpr int BYTES = END * 8;
};
// 1D sweep along DIM of a velocity / gradient block with plane stride PS (the line numbering of qd::Sw3 for an
// N^3 cube), tables in even/odd form
template <int N, int PS, int DIM, bool ACC>
struct SwC {
    template <int S>
    __device__ static void line(const double* in, double* out, const EOMat<N, N, S>& T, int l)
    {
        int ib, ist;
        if (DIM == 0) { const int i1 = l % N, i2 = l / N; ib = N * i1 + PS * i2; ist = 1; }
        else if (DIM == 1) { const int i0 = l % N, i2 = l / N; ib = i0 + PS * i2; ist = N; }
        else { const int i0 = l % N, i1 = l / N; ib = i0 + N * i1; ist = PS; }
        double v[N], y[N];
        if constexpr (DIM == 0 && PS != N * N) { // (padded n = 4 blocks: a j0 line is 16-B aligned: 2 x 16-B accesses)
#pragma unroll
            for (int j = 0; j < N; j += 2) {
                const double2 t = *reinterpret_cast<const double2*>(in + ib + j);
                v[j] = t.x;
                v[j + 1] = t.y;
            }
        } else {
#pragma unroll
            for (int j = 0; j < N; ++j) v[j] = in[ib + ist * j];
        }
        eo_apply(T, v, y);
        if constexpr (DIM == 0 && PS != N * N) {
#pragma unroll
            for (int q = 0; q < N; q += 2) {
                double2* o = reinterpret_cast<double2*>(out + ib + q);
                if (ACC) {
                    const double2 t = *o;
                    *o = make_double2(t.x + y[q], t.y + y[q + 1]);
                } else {
                    *o = make_double2(y[q], y[q + 1]);
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < N; ++q) out[ib + ist * q] = ACC ? out[ib + ist * q] + y[q] : y[q];
        }
    }
};
// padded index of the dense point P = j0 + N j1 + N^2 j2
template <int N, int PS>
__device__ __forceinline__ int pad_pt(int P) { return P + (PS - N * N) * (P / (N * N)); }
} // namespace sk

// grid: one CTA per cell of [c_begin, c_end) (local canonical order), block SLay::NT, dynamic smem
// SLay::BYTES. x, r: the slab's blocks of B doubles per cell; xb / xa: the halo planes below / above.
template <int N>
__global__ void __launch_bounds__(sk::SLay<N>::NT)
k_stokes(const double* __restrict__ x, const double* __restrict__ xb, const double* __restrict__ xa, double* __restrict__ r,
         long long c_begin, long long c_end, const __grid_constant__ STab<N> T, const MeshArgs M_)
{
    using L = sk::SLay<N>;
    constexpr int NP = L::NP, N2 = L::N2, N3 = L::N3, NP2 = L::NP2, NP3 = L::NP3, B = L::B, NT = L::NT;
    const MeshArgs& Ms = M_;
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x;
    const long long lc = c_begin + blockIdx.x;
    if (lc >= c_end) return;
    const int lp = (int)(lc / Ms.plane_cells), rem = (int)(lc - (long long)lp * Ms.plane_cells);
    const int ig0 = Ms.plane_begin + lp, ig1 = rem / Ms.N2, ig2 = rem % Ms.N2;
    // (selects instead of run-time indexed arrays: no local memory)
    auto on_bnd = [&](int d, int side) {
        const int i = d == 0 ? ig0 : (d == 1 ? ig1 : ig2);
        const int Nd = d == 0 ? Ms.N0 : (d == 1 ? Ms.N1 : Ms.N2);
        return side ? i == Nd - 1 : i == 0;
    };
    double* const U = sm + L::U;
    double* const PR = sm + L::PR;
    double* const G = sm + L::G;
    double* const PQ = sm + L::PQ;
    double* const TA = sm + L::TA;
    double* const TB = sm + L::TB;
    auto face = [&](int f) { return sm + L::F + f * L::FACE; };
    // the small tables indexed by run-time point indices, in shared memory: a constant-bank load with lane-varying
    // addresses is serialised over the distinct addresses of a warp
    __shared__ double sTab[6 * N + 2 * NP];
    double* const sE0 = sTab;
    double* const sE1 = sTab + N;
    double* const sD0 = sTab + 2 * N;
    double* const sD1 = sTab + 3 * N;
    double* const sW = sTab + 4 * N;
    double* const sXi = sTab + 5 * N;
    double* const sEp0 = sTab + 6 * N;
    double* const sEp1 = sTab + 6 * N + NP;
    for (int i = tid; i < N; i += NT) {
        sE0[i] = T.e0[i];
        sE1[i] = T.e1[i];
        sD0[i] = T.d0[i];
        sD1[i] = T.d1[i];
        sW[i] = T.w[i];
        sXi[i] = T.xi[i];
        if (i < NP) {
            sEp0[i] = T.ep0[i];
            sEp1[i] = T.ep1[i];
        }
    }
    // neighbour block across face f = 2d + side, or nullptr on the boundary of the cube
    auto nbp = [&](int f) -> const double* {
        const int d = f >> 1, side = f & 1;
        if (on_bnd(d, side)) return nullptr;
        if (d == 0) {
            const int nl = lp + (side ? 1 : -1);
            if (nl < 0) return xb + (long long)rem * B;
            if (nl >= Ms.L) return xa + (long long)rem * B;
            return x + ((long long)nl * Ms.plane_cells + rem) * B;
        }
        const int stride = d == 1 ? Ms.N2 : 1;
        return x + (lc + (side ? stride : -stride)) * B;
    };

    // ---------------- P0: stage the cell's block (velocity + pressure, contiguous in both) ----------------
    for (int i = tid; i < B; i += NT) {
        const double v = __ldg(x + lc * B + i);
        if (i < 3 * N3) U[(i / N3) * L::NB + sk::pad_pt<N, L::PS>(i % N3)] = v;
        else PR[i - 3 * N3] = v;
    }
    __syncthreads();

    // ---------------- P1: gradients (9 D sweeps), pressure A_p along j2, face traces ----------------
    // the neighbours' values for this thread's face-trace tasks are loaded first (from L2) and consumed after
    // the gradient sweeps, so their latency hides behind the sweeps instead of stalling the P1 barrier
    // (n <= 5; for larger n the register cost outweighs it)
    constexpr bool PREF = N <= 5;
    constexpr int NFT = PREF ? (18 * N2 + NT - 1) / NT : 1; // face-trace tasks per thread (at most)
    double vnb[NFT][N];
#pragma unroll
    for (int k = 0; k < NFT; ++k) {
        const int t = tid + k * NT;
        if (PREF && t < 18 * N2) {
            const int f = t / (3 * N2), c = (t / N2) % 3, p = t % N2, a = p % N, bq = p / N;
            const double* nb = nbp(f);
#pragma unroll
            for (int j = 0; j < N; ++j) vnb[k][j] = nb ? __ldg(nb + c * N3 + pidx<N>(f >> 1, j, a, bq)) : 0.0;
        }
    }
    if constexpr (N == 4 && NT % 32 == 0) {
        // n = 4: a gradient sweep (c, e) has 16 lines = half a warp; pair half-warps of the same direction e
        // in one warp so that no warp runs two differently-specialised sweeps one after the other
        // (slots of 32 lanes: (0,3) (1,4) (2,5) 6 7 8 with ce = 3 c + e)
        constexpr int NSLOT = 6;
        for (int slot = tid >> 5; slot < NSLOT; slot += NT / 32) {
            const int h = (tid >> 4) & 1, l = tid & 15;
            const int ce = slot < 3 ? slot + 3 * h : (h ? -1 : slot + 3);
            if (ce < 0) continue;
            const int c = ce / 3, e = ce % 3;
            const double* in = U + c * L::NB;
            double* out = G + ce * L::NB;
            if (e == 0) sk::SwC<N, L::PS, 0, false>::line(in, out, T.eD, l);
            else if (e == 1) sk::SwC<N, L::PS, 1, false>::line(in, out, T.eD, l);
            else sk::SwC<N, L::PS, 2, false>::line(in, out, T.eD, l);
        }
    } else {
        for (int t = tid; t < 9 * N2; t += NT) {
            const int ce = t / N2, l = t % N2, c = ce / 3, e = ce % 3;
            const double* in = U + c * L::NB;
            double* out = G + ce * L::NB;
            if (e == 0) sk::SwC<N, L::PS, 0, false>::line(in, out, T.eD, l);
            else if (e == 1) sk::SwC<N, L::PS, 1, false>::line(in, out, T.eD, l);
            else sk::SwC<N, L::PS, 2, false>::line(in, out, T.eD, l);
        }
    }
    for (int t = tid; t < NP2; t += NT) qd::Sw3<NP, NP, NP, 2, N, false, false>::line(PR, TA, T.eAP, t);
    constexpr int NFL = PREF ? NFT : (18 * N2 + NT - 1) / NT;
#pragma unroll
    for (int k = 0; k < NFL; ++k) {
        const int t = tid + k * NT;
        if (t >= 18 * N2) break;
        const int f = t / (3 * N2), c = (t / N2) % 3, p = t % N2, a = p % N, bq = p / N;
        const int d = f >> 1, side = f & 1;
        const double* nb = PREF ? nullptr : nbp(f);
        const double* es = side ? T.e1 : T.e0;
        const double* ds = side ? T.d1 : T.d0;
        const double* en = side ? T.e0 : T.e1;
        const double* dn = side ? T.d0 : T.d1;
        double uo = 0, go = 0, un = 0, gn = 0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double vo = U[c * L::NB + sk::pad_pt<N, L::PS>(pidx<N>(d, j, a, bq))];
            uo = fma(es[j], vo, uo);
            go = fma(ds[j], vo, go);
            const double vn = PREF ? vnb[k][j] : (nb ? __ldg(nb + c * N3 + pidx<N>(d, j, a, bq)) : 0.0);
            un = fma(en[j], vn, un); // (zero on the boundary of the cube)
            gn = fma(dn[j], vn, gn);
        }
        double* TR = face(f) + L::TR + c * 4 * N2;
        TR[p] = uo;
        TR[N2 + p] = go;
        TR[2 * N2 + p] = un;
        TR[3 * N2 + p] = gn;
    }
    for (int t = tid; t < 6 * NP2; t += NT) {
        const int f = t / NP2, p = t % NP2, a = p % NP, bq = p / NP;
        const int d = f >> 1, side = f & 1;
        const double* nb = nbp(f);
        const double* es = side ? T.ep1 : T.ep0;
        const double* en = side ? T.ep0 : T.ep1;
        double po = 0, pn = 0;
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int P = pidx<NP>(d, j, a, bq);
            po = fma(es[j], PR[P], po);
            if (nb) pn = fma(en[j], __ldg(nb + 3 * N3 + P), pn);
        }
        double* PT = face(f) + L::PT;
        PT[p] = po;
        PT[NP2 + p] = pn;
    }
    __syncthreads();
    // ---------------- P2: pressure A_p along j1; face pressure A_p along t1 ----------------
    for (int t = tid; t < NP * N; t += NT) qd::Sw3<NP, NP, N, 1, N, false, false>::line(TA, TB, T.eAP, t);
    for (int t = tid; t < 12 * NP; t += NT) {
        const int f = t / (2 * NP), s = (t / NP) % 2, l = t % NP;
        double* Fb = face(f);
        qd::Sw2<NP, NP, 0, N, false, false>::line(Fb + L::PT + s * NP2, Fb + L::PF1 + s * N * NP, T.eAP, l);
    }
    __syncthreads();
    // ---------------- P3: pressure A_p along j0 (p at the N^3 points); face pressure along t2 ----------------
    for (int t = tid; t < N2; t += NT) qd::Sw3<NP, N, N, 0, N, false, false>::line(TB, PQ, T.eAP, t);
    for (int t = tid; t < 12 * N; t += NT) {
        const int f = t / (2 * N), s = (t / N) % 2, l = t % N;
        double* Fb = face(f);
        qd::Sw2<N, NP, 1, N, false, false>::line(Fb + L::PF1 + s * N * NP, Fb + L::PF2 + s * N2, T.eAP, l);
    }
    __syncthreads();
    // ---------------- P4: pointwise volume terms; face fluxes ----------------
    const double h0 = Ms.h[0], h1 = Ms.h[1], h2 = Ms.h[2];
    auto hsel = [&](int e) { return e == 0 ? h0 : (e == 1 ? h1 : h2); };
    // 1/h by multiplication (a double division is a ~20-instruction sequence with a slow-path branch)
    const double ih0 = 1.0 / h0, ih1 = 1.0 / h1, ih2 = 1.0 / h2;
    auto ihsel = [&](int e) { return e == 0 ? ih0 : (e == 1 ? ih1 : ih2); };
    for (int P = tid; P < N3; P += NT) {
        const int q0 = P % N, q1 = (P / N) % N, q2 = P / N2;
        const double W = sW[q0] * sW[q1] * sW[q2] * h0 * h1 * h2;
        const double p = PQ[P];
        double div = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                double* g = G + (3 * c + e) * L::NB + sk::pad_pt<N, L::PS>(P);
                const double ihe = e == 0 ? ih0 : (e == 1 ? ih1 : ih2);
                const double ge = *g * ihe;            // physical d u_c / d x_e
                if (c == e) div += ge;
                double q = W * ge;                     // (grad u_c, grad v): . d v / d x_e
                if (c == e) q -= W * p;                // -(p, div v)
                *g = q * ihe;                          // coefficient of the reference derivative
            }
        }
        PQ[P] = -W * div;                              // -(div u, q)
    }
    for (int t = tid; t < 6 * N2; t += NT) {
        const int f = t / N2, p = t % N2, a = p % N, bq = p / N;
        const int d = f >> 1, side = f & 1;
        const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
        double* Fb = face(f);
        double* TR = Fb + L::TR;
        const bool bnd = on_bnd(d, side);
        const double W = sW[a] * sW[bq] * hsel(t1) * hsel(t2);
        const double ihd = ihsel(d);
        const double gam = d == 0 ? Ms.gamma[0] : (d == 1 ? Ms.gamma[1] : Ms.gamma[2]);
        double Cv[3], Cn[3], Cq;
        if (bnd && d == 0 && side == 1) {
            // Gamma_N (x_0 = 1): no face terms
            Cv[0] = Cv[1] = Cv[2] = Cn[0] = Cn[1] = Cn[2] = Cq = 0.0;
        } else if (bnd) {
            // Dirichlet face: [u] -> u - g, one-sided flux, outer normal sn e_d
            const double sn = side ? 1.0 : -1.0;
            const double xi1 = d == 1 ? (double)side : (t1 == 1 ? sXi[a] : sXi[bq]);
            const double X1 = (ig1 + xi1) * h1;
            const double po = Fb[L::PF2 + p];
            double jd = 0.0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double g = c == 0 ? 4.0 * X1 * (1.0 - X1) : 0.0;
                const double jmp = TR[c * 4 * N2 + p] - g;
                const double dun = sn * TR[c * 4 * N2 + N2 + p] * ihd;
                Cv[c] = W * (-dun + gam * jmp + (c == d ? sn * po : 0.0));
                Cn[c] = -W * jmp * sn * ihd;           // theta (u - g, grad v . n), theta = -1
                if (c == d) jd = jmp;
            }
            Cq = W * sn * jd;                          // ((u - g) . n, q)
        } else {
            const double sv = side ? 1.0 : -1.0;       // [v] = sv v (this cell is T- iff side = 1)
            const double pavg = 0.5 * (Fb[L::PF2 + p] + Fb[L::PF2 + N2 + p]);
            double jd = 0.0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double uo = TR[c * 4 * N2 + p], go = TR[c * 4 * N2 + N2 + p];
                const double un = TR[c * 4 * N2 + 2 * N2 + p], gn = TR[c * 4 * N2 + 3 * N2 + p];
                const double jump = side ? uo - un : un - uo;
                const double avg = 0.5 * (go + gn) * ihd;
                Cv[c] = sv * W * (-avg + gam * jump + (c == d ? pavg : 0.0));
                Cn[c] = -0.5 * W * jump * ihd;         // theta ([u], {grad v} n)
                if (c == d) jd = jump;
            }
            Cq = 0.5 * W * jd;                         // ([u] . n, {q})
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            TR[c * 4 * N2 + p] = Cv[c];
            TR[c * 4 * N2 + N2 + p] = Cn[c];
        }
        Fb[L::PF2 + p] = Cq;
    }
    __syncthreads();
    // ---------------- P5: stage 3 (D^T per direction into RU, A_p^T for the pressure), face A_p^T ----------------
    for (int t = tid; t < 3 * N2; t += NT) {
        const int c = t / N2, l = t % N2;
        sk::SwC<N, L::PS, 0, false>::line(G + (3 * c) * L::NB, U + c * L::NB, T.eDt, l);
    }
    for (int t = tid; t < N2; t += NT) qd::Sw3<N, N, N, 0, NP, true, false>::line(PQ, TB, T.eAPt, t);
    for (int t = tid; t < 6 * N; t += NT) {
        const int f = t / N, l = t % N;
        double* Fb = face(f);
        qd::Sw2<N, N, 1, NP, true, false>::line(Fb + L::PF2, Fb + L::PF1, T.eAPt, l);
    }
    __syncthreads();
    for (int t = tid; t < 3 * N2; t += NT) {
        const int c = t / N2, l = t % N2;
        sk::SwC<N, L::PS, 1, true>::line(G + (3 * c + 1) * L::NB, U + c * L::NB, T.eDt, l);
    }
    for (int t = tid; t < NP * N; t += NT) qd::Sw3<NP, N, N, 1, NP, true, false>::line(TB, TA, T.eAPt, t);
    for (int t = tid; t < 6 * NP; t += NT) {
        const int f = t / NP, l = t % NP;
        double* Fb = face(f);
        qd::Sw2<N, NP, 0, NP, true, false>::line(Fb + L::PF1, Fb + L::PT, T.eAPt, l);
    }
    __syncthreads();
    for (int t = tid; t < 3 * N2; t += NT) {
        const int c = t / N2, l = t % N2;
        sk::SwC<N, L::PS, 2, true>::line(G + (3 * c + 2) * L::NB, U + c * L::NB, T.eDt, l);
    }
    for (int t = tid; t < NP2; t += NT) qd::Sw3<NP, NP, N, 2, NP, true, false>::line(TA, PR, T.eAPt, t);
    __syncthreads();
    // ---------------- P6: add the face back-projections along the normals, write the block once ----------------
    for (int i = tid; i < B; i += NT) {
        double v = i < 3 * N3 ? U[(i / N3) * L::NB + sk::pad_pt<N, L::PS>(i % N3)] : PR[i - 3 * N3];
        if (i < 3 * N3) {
            const int c = i / N3, P = i % N3;
            const int j[3] = {P % N, (P / N) % N, P / N2};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
                const int p = j[t1] + N * j[t2];
#pragma unroll
                for (int side = 0; side < 2; ++side) {
                    const double* TR = face(2 * d + side) + L::TR + c * 4 * N2;
                    const double e = side ? sE1[j[d]] : sE0[j[d]], dd = side ? sD1[j[d]] : sD0[j[d]];
                    v = fma(e, TR[p], fma(dd, TR[N2 + p], v));
                }
            }
        } else {
            const int P = i - 3 * N3;
            const int j[3] = {P % NP, (P / NP) % NP, P / NP2};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
                const int p = j[t1] + NP * j[t2];
#pragma unroll
                for (int side = 0; side < 2; ++side) {
                    const double e = side ? sEp1[j[d]] : sEp0[j[d]];
                    v = fma(e, face(2 * d + side)[L::PT + p], v);
                }
            }
        }
        r[lc * B + i] = v;
    }
}

} // namespace dg
