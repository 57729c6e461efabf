// K_quadw: the general-quadrature operator (M = n + 1 points, A != I) and the paper's
// diffusion-reaction problem (DR) with ONE WARP PER CELL — the same mathematics and the
// same 1D sweeps as k_quad (kernel_quad.cuh: stage 1 d0 = D0 A1 A2 X ..., stage 3 transposes, faces by
// traces along the normal then A / D on the face), but every dependency is
// inside one warp (__syncwarp), so the warps of an SM progress independently instead of meeting at
// ~9 CTA barriers per cell group (the first profile of k_quad: 42 % of the stall samples at barriers).
// Per warp: X, R and the stage buffers of one cell in shared memory; the six faces are evaluated one
// after the other with buffers aliasing the (then dead) stage-1/2 buffers. Used for n = 5, where it measured
// faster than k_quad (cfg4 size with 6 points: 410 vs 490 ms); for n <= 4 a warp phase has too few lines.
#pragma once

#include "kernel_quad.cuh"

namespace dg {

namespace qw {

template <int N, int M>
struct WLay {
    static constexpr int N2 = N * N, N3 = N * N * N, M2 = M * M, M3 = M * M * M, NM = N * M;
    static constexpr int WPB = (N <= 3) ? 8 : 4; // warps per CTA
    // per warp (doubles)
    static constexpr int X = 0, R = X + N3, GEO = R + N3;           // GEO: cell 14 + face 16
    static constexpr int Y2 = GEO + 30 + (N3 % 2), Y2d = Y2 + N2 * M; // stage 1a / 3b
    static constexpr int Z = Y2d + N2 * M, Zd1 = Z + N * M2, Zd2 = Zd1 + N * M2; // stage 1b / 3a
    static constexpr int G0 = Zd2 + N * M2, G1 = G0 + M3, G2 = G1 + M3, GU = G2 + M3; // points
    static constexpr int VOL_END = GU + M3;
    // face buffers alias Y2 .. (dead after stage 3c): FT [4][N2], F1 [6][NM], F2 [8][M2]
    static constexpr int FT = Y2, F1 = FT + 4 * N2, F2 = F1 + 6 * NM, FACE_END = F2 + 8 * M2;
    static constexpr int WARP = ((VOL_END > FACE_END ? VOL_END : FACE_END) + 1) / 2 * 2;
    static constexpr int BYTES = WPB * WARP * 8;
};

} // namespace qw

// grid: enough CTAs for one pass over the cells (each warp takes cells c = (blockIdx * WPB + warp) + k stride)
template <int N, int M, bool AFFINE, bool COEFF, bool DR = false>
__global__ void __launch_bounds__(qw::WLay<N, M>::WPB * 32)
k_quadw(const double* __restrict__ x, const double* __restrict__ xb, const double* __restrict__ xa, double* __restrict__ r,
        long long c_begin, long long c_end, const __grid_constant__ QTab<N, M> T, const MeshArgs Ms)
{
    using L = qw::WLay<N, M>;
    constexpr int N2 = L::N2, N3 = L::N3, M2 = L::M2, M3 = L::M3, NM = L::NM, WPB = L::WPB;
    extern __shared__ __align__(16) double sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* const b = sm + warp * L::WARP;
    const long long ncell = c_end - c_begin;

    for (long long lc = (long long)blockIdx.x * WPB + warp; lc < ncell; lc += (long long)gridDim.x * WPB) {
        const long long cg = c_begin + lc; // local cell index
        const int lp = (int)(cg / Ms.plane_cells), rem = (int)(cg - (long long)lp * Ms.plane_cells);
        const int ig[3] = {(Ms.plane_begin + lp) % Ms.N0, rem / Ms.N2, rem % Ms.N2};
        for (int i = lane; i < N3; i += 32) b[L::X + i] = __ldg(x + cg * N3 + i);
        // cell geometry: G~ = |det J| J^-1 J^-T, J rows 0-1, origin (lane 0)
        if (lane == 0) {
            double J[9], Ji[9];
            if (AFFINE) {
                const double* jp = Ms.jac + ((long long)(lp + 1) * Ms.plane_cells + rem) * 9;
                for (int i = 0; i < 9; ++i) J[i] = __ldg(jp + i);
            } else {
                for (int i = 0; i < 9; ++i) J[i] = 0.0;
                J[0] = Ms.h[0]; J[4] = Ms.h[1]; J[8] = Ms.h[2];
            }
            const double ad = fabs(inv3(J, Ji));
            double* g = b + L::GEO;
            auto gg = [&](int a, int c) { return ad * (Ji[3 * a] * Ji[3 * c] + Ji[3 * a + 1] * Ji[3 * c + 1] + Ji[3 * a + 2] * Ji[3 * c + 2]); };
            g[0] = gg(0, 0); g[1] = gg(1, 1); g[2] = gg(2, 2); g[3] = gg(0, 1); g[4] = gg(0, 2); g[5] = gg(1, 2);
            for (int i = 0; i < 6; ++i) g[6 + i] = J[i];
            g[12] = (double)ig[0] / Ms.N0;
            g[13] = (double)ig[1] / Ms.N1;
        }
        __syncwarp();
        // ---------------- stage 1: d0 = D0 A1 A2 X, d1 = A0 D1 A2 X, d2 = A0 A1 D2 X (+ u = A0 A1 A2 X) ----
        {
            using S = qd::Sw3<N, N, N, 2, M, false, false>;
            for (int t = lane; t < 2 * S::NL; t += 32) {
                if (t < S::NL) S::line(b + L::X, b + L::Y2, T.A, t);
                else S::line(b + L::X, b + L::Y2d, T.Dq, t - S::NL);
            }
        }
        __syncwarp();
        {
            using S = qd::Sw3<N, N, M, 1, M, false, false>;
            for (int t = lane; t < 3 * S::NL; t += 32) {
                const int k = t / S::NL, l = t - k * S::NL;
                if (k == 0) S::line(b + L::Y2, b + L::Z, T.A, l);
                else if (k == 1) S::line(b + L::Y2, b + L::Zd1, T.Dq, l);
                else S::line(b + L::Y2d, b + L::Zd2, T.A, l);
            }
        }
        __syncwarp();
        {
            using S = qd::Sw3<N, M, M, 0, M, false, false>;
            constexpr int NQ = DR ? 4 : 3;
            for (int t = lane; t < NQ * S::NL; t += 32) {
                const int k = t / S::NL, l = t - k * S::NL;
                if (k == 0) S::line(b + L::Z, b + L::G0, T.Dq, l);
                else if (k == 1) S::line(b + L::Zd1, b + L::G1, T.A, l);
                else if (k == 2) S::line(b + L::Zd2, b + L::G2, T.A, l);
                else S::line(b + L::Z, b + L::GU, T.A, l);
            }
        }
        __syncwarp();
        // ---------------- stage 2 at the M^3 points ----------------
        {
            const double* g = b + L::GEO;
            for (int P = lane; P < M3; P += 32) {
                const int q0 = P % M, q1 = (P / M) % M, q2 = P / M2;
                const double a0 = b[L::G0 + P], a1 = b[L::G1 + P], a2 = b[L::G2 + P];
                if (DR) {
                    const double h0 = Ms.h[0], h1 = Ms.h[1], h2 = Ms.h[2];
                    const double W = T.wq[q0] * T.wq[q1] * T.wq[q2] * h0 * h1 * h2;
                    const double x0 = (ig[0] + T.xq[q0]) * h0, x1 = (ig[1] + T.xq[q1]) * h1, x2 = (ig[2] + T.xq[q2]) * h2;
                    const double p0 = a0 / h0, p1 = a1 / h1, p2 = a2 / h2;
                    const double xg = x0 * p0 + x1 * p1 + x2 * p2; // K grad u = x (x . grad u) + grad u
                    b[L::G0 + P] = W * fma(x0, xg, p0) / h0;
                    b[L::G1 + P] = W * fma(x1, xg, p1) / h1;
                    b[L::G2 + P] = W * fma(x2, xg, p2) / h2;
                    b[L::GU + P] = W * (10.0 * b[L::GU + P] + 6.0);
                } else {
                    double cW = T.wq[q0] * T.wq[q1] * T.wq[q2];
                    if (COEFF) {
                        const double xi0 = T.xq[q0], xi1 = T.xq[q1], xi2 = T.xq[q2];
                        cW *= coeff_sincos(g[12] + g[6] * xi0 + g[7] * xi1 + g[8] * xi2, g[13] + g[9] * xi0 + g[10] * xi1 + g[11] * xi2);
                    }
                    b[L::G0 + P] = cW * fma(g[0], a0, fma(g[3], a1, g[4] * a2));
                    b[L::G1 + P] = cW * fma(g[3], a0, fma(g[1], a1, g[5] * a2));
                    b[L::G2 + P] = cW * fma(g[4], a0, fma(g[5], a1, g[2] * a2));
                }
            }
        }
        __syncwarp();
        // ---------------- stage 3 (transposes in reverse order) into R ----------------
        {
            using S = qd::Sw3<M, M, M, 0, N, true, false>;
            using Sa = qd::Sw3<M, M, M, 0, N, true, true>;
            for (int t = lane; t < 3 * S::NL; t += 32) {
                const int k = t / S::NL, l = t - k * S::NL;
                if (k == 0) {
                    S::line(b + L::G0, b + L::Z, T.Dq, l);
                    if (DR) Sa::line(b + L::GU, b + L::Z, T.A, l);
                } else if (k == 1) S::line(b + L::G1, b + L::Zd1, T.A, l);
                else S::line(b + L::G2, b + L::Zd2, T.A, l);
            }
        }
        __syncwarp();
        {
            using S = qd::Sw3<N, M, M, 1, N, true, false>;
            using Sa = qd::Sw3<N, M, M, 1, N, true, true>;
            for (int t = lane; t < 2 * S::NL; t += 32) {
                if (t < S::NL) { S::line(b + L::Z, b + L::Y2, T.A, t); Sa::line(b + L::Zd1, b + L::Y2, T.Dq, t); }
                else S::line(b + L::Zd2, b + L::Y2d, T.A, t - S::NL);
            }
        }
        __syncwarp();
        {
            using S = qd::Sw3<N, N, M, 2, N, true, false>;
            using Sa = qd::Sw3<N, N, M, 2, N, true, true>;
            for (int t = lane; t < S::NL; t += 32) {
                S::line(b + L::Y2, b + L::R, T.A, t);
                Sa::line(b + L::Y2d, b + L::R, T.Dq, t);
            }
        }
        __syncwarp();
        // ---------------- the six faces, one after the other ----------------
        for (int f = 0; f < 6; ++f) {
            const int d = f >> 1, side = f & 1;
            const int t1 = d == 0 ? 1 : 0, t2 = d == 2 ? 1 : 2;
            const int Nd = d == 0 ? Ms.N0 : (d == 1 ? Ms.N1 : Ms.N2);
            const bool bnd = DR && (side ? ig[d] == Nd - 1 : ig[d] == 0);
            // neighbour across the face
            int nlp = lp, nrem = rem, nig1 = ig[1], nig2 = ig[2];
            if (d == 0) nlp = lp + (side ? 1 : -1);
            else {
                if (d == 1) nig1 = (ig[1] + (side ? 1 : Ms.N1 - 1)) % Ms.N1;
                else nig2 = (ig[2] + (side ? 1 : Ms.N2 - 1)) % Ms.N2;
                nrem = nig1 * Ms.N2 + nig2;
            }
            // face geometry (lane 0): dS, a-, a+, J_- rows 0-1, T- origin
            double* fg = b + L::GEO + 14;
            if (lane == 0) {
                double J[9], Ji[9], Jn[9], Jni[9];
                if (AFFINE) {
                    const double* jp = Ms.jac + ((long long)(lp + 1) * Ms.plane_cells + rem) * 9;
                    const double* jn = Ms.jac + ((long long)(nlp + 1) * Ms.plane_cells + (d == 0 ? rem : nrem)) * 9;
                    for (int i = 0; i < 9; ++i) { J[i] = __ldg(jp + i); Jn[i] = __ldg(jn + i); }
                } else {
                    for (int i = 0; i < 9; ++i) J[i] = Jn[i] = 0.0;
                    J[0] = Jn[0] = Ms.h[0]; J[4] = Jn[4] = Ms.h[1]; J[8] = Jn[8] = Ms.h[2];
                }
                const double det = inv3(J, Ji), detn = inv3(Jn, Jni);
                const double* Jm = side ? J : Jn;
                const double* Jmi = side ? Ji : Jni;
                const double* Jpi = side ? Jni : Ji;
                const double nu0 = Jmi[3 * d], nu1 = Jmi[3 * d + 1], nu2 = Jmi[3 * d + 2];
                const double nn = sqrt(nu0 * nu0 + nu1 * nu1 + nu2 * nu2);
                const double n0 = nu0 / nn, n1 = nu1 / nn, n2 = nu2 / nn;
                fg[0] = fabs(side ? det : detn) * nn;
                for (int e = 0; e < 3; ++e) {
                    fg[1 + e] = Jmi[3 * e] * n0 + Jmi[3 * e + 1] * n1 + Jmi[3 * e + 2] * n2;
                    fg[4 + e] = Jpi[3 * e] * n0 + Jpi[3 * e + 1] * n1 + Jpi[3 * e + 2] * n2;
                }
                for (int i = 0; i < 6; ++i) fg[7 + i] = Jm[i];
                const int mi0 = (d == 0 && !side) ? (ig[0] + Ms.N0 - 1) % Ms.N0 : ig[0];
                const int mi1 = (d == 1 && !side) ? nig1 : ig[1];
                fg[13] = (double)mi0 / Ms.N0;
                fg[14] = (double)mi1 / Ms.N1;
            }
            const double* nbx;
            if (d == 0) nbx = nlp < 0 ? xb + (long long)rem * N3 : (nlp >= Ms.L ? xa + (long long)rem * N3 : x + ((long long)nlp * Ms.plane_cells + rem) * N3);
            else nbx = x + ((long long)lp * Ms.plane_cells + nrem) * N3;
            // traces along the normal (own from smem, neighbour from L2)
            for (int p = lane; p < N2; p += 32) {
                const int a = p % N, bq = p / N;
                double uo = 0, go = 0, un = 0, gn = 0;
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    const double vo = b[L::X + pidx<N>(d, j, a, bq)];
                    const double vn = bnd ? 0.0 : __ldg(nbx + pidx<N>(d, j, a, bq));
                    uo = fma(side ? T.e1[j] : T.e0[j], vo, uo);
                    go = fma(side ? T.d1[j] : T.d0[j], vo, go);
                    un = fma(side ? T.e0[j] : T.e1[j], vn, un);
                    gn = fma(side ? T.d0[j] : T.d1[j], vn, gn);
                }
                b[L::FT + p] = uo;
                b[L::FT + N2 + p] = go;
                b[L::FT + 2 * N2 + p] = un;
                b[L::FT + 3 * N2 + p] = gn;
            }
            __syncwarp();
            {
                using F = qd::Sw2<N, N, 0, M, false, false>; // along t1: N x N -> M x N
                for (int t = lane; t < 6 * F::NL; t += 32) {
                    const int k = t / F::NL, l = t - k * F::NL;
                    const double* src = b + L::FT + ((k < 3) ? (k == 2 ? N2 : 0) : (k == 5 ? 3 * N2 : 2 * N2));
                    if (k % 3 == 1) F::line(src, b + L::F1 + k * NM, T.Dq, l);
                    else F::line(src, b + L::F1 + k * NM, T.A, l);
                }
            }
            __syncwarp();
            {
                using F = qd::Sw2<M, N, 1, M, false, false>; // along t2: M x N -> M x M
                for (int t = lane; t < 8 * F::NL; t += 32) {
                    const int k = t / F::NL, l = t - k * F::NL;
                    const int s = k & 1, q = k >> 1;
                    const double* src = b + L::F1 + (3 * s + (q == 0 || q == 3 ? 0 : (q == 1 ? 2 : 1))) * NM;
                    if (q == 3) F::line(src, b + L::F2 + k * M2, T.Dq, l);
                    else F::line(src, b + L::F2 + k * M2, T.A, l);
                }
            }
            __syncwarp();
            // flux at the M^2 points -> this cell's coefficients (Cv, Ct1, Ct2, Cn) in place of F2[0..3]
            for (int p = lane; p < M2; p += 32) {
                const int a = p % M, bq = p / M;
                double* F2 = b + L::F2;
                const double Uo = F2[p], Un = F2[M2 + p], Gno = F2[2 * M2 + p], Gnn = F2[3 * M2 + p];
                const double T1o = F2[4 * M2 + p], T1n = F2[5 * M2 + p], T2o = F2[6 * M2 + p], T2n = F2[7 * M2 + p];
                double Cv, C1, C2, Cn;
                if (DR) {
                    const double xa_ = T.xq[a], xb_ = T.xq[bq];
                    const double xi0 = d == 0 ? (double)side : xa_;
                    const double xi1 = d == 1 ? (double)side : (d == 0 ? xa_ : xb_);
                    const double xi2 = d == 2 ? (double)side : xb_;
                    const double X0 = (ig[0] + xi0) * Ms.h[0], X1 = (ig[1] + xi1) * Ms.h[1], X2 = (ig[2] + xi2) * Ms.h[2];
                    const double Xd = d == 0 ? X0 : (d == 1 ? X1 : X2);
                    const double Xt1 = d == 0 ? X1 : X0, Xt2 = d == 2 ? X1 : X2;
                    const double hd = Ms.h[d], ht1 = Ms.h[t1], ht2 = Ms.h[t2];
                    const double kd = (Xd * Xd + 1.0) / hd, kt1 = Xd * Xt1 / ht1, kt2 = Xd * Xt2 / ht2;
                    const double W = T.wq[a] * T.wq[bq] * ht1 * ht2;
                    const double gam = d == 0 ? Ms.gamma[0] : (d == 1 ? Ms.gamma[1] : Ms.gamma[2]);
                    const double Kgo = kd * Gno + kt1 * T1o + kt2 * T2o;
                    double s;
                    if (bnd) {
                        const double sn = side ? 1.0 : -1.0;
                        const double jmp = Uo - (X0 * X0 + X1 * X1 + X2 * X2);
                        Cv = W * (-sn * Kgo + gam * jmp);
                        s = -W * jmp * sn;
                    } else {
                        const double Kgn = kd * Gnn + kt1 * T1n + kt2 * T2n;
                        const double jmp = side ? Uo - Un : Un - Uo;
                        const double Cvm = W * (-0.5 * (Kgo + Kgn) + gam * jmp);
                        Cv = side ? Cvm : -Cvm;
                        s = -0.5 * W * jmp;
                    }
                    C1 = s * kt1;
                    C2 = s * kt2;
                    Cn = s * kd;
                } else {
                    const double um = side ? Uo : Un, up = side ? Un : Uo;
                    const double gnm = side ? Gno : Gnn, gnp = side ? Gnn : Gno;
                    const double t1m = side ? T1o : T1n, t1p = side ? T1n : T1o;
                    const double t2m = side ? T2o : T2n, t2p = side ? T2n : T2o;
                    const double* am = fg + 1;
                    const double* ap = fg + 4;
                    double cF = 1.0;
                    if (COEFF) {
                        const double xa_ = T.xq[a], xb_ = T.xq[bq];
                        const double xi0 = d == 0 ? 1.0 : xa_;
                        const double xi1 = d == 1 ? 1.0 : (d == 0 ? xa_ : xb_);
                        const double xi2 = d == 2 ? 1.0 : xb_;
                        cF = coeff_sincos(fg[13] + fg[7] * xi0 + fg[8] * xi1 + fg[9] * xi2,
                                          fg[14] + fg[10] * xi0 + fg[11] * xi1 + fg[12] * xi2);
                    }
                    const double amd = d == 0 ? am[0] : (d == 1 ? am[1] : am[2]);
                    const double amt1 = t1 == 0 ? am[0] : am[1], amt2 = t2 == 1 ? am[1] : am[2];
                    const double apd = d == 0 ? ap[0] : (d == 1 ? ap[1] : ap[2]);
                    const double apt1 = t1 == 0 ? ap[0] : ap[1], apt2 = t2 == 1 ? ap[1] : ap[2];
                    const double gm = cF * (amd * gnm + amt1 * t1m + amt2 * t2m);
                    const double gp = cF * (apd * gnp + apt1 * t1p + apt2 * t2p);
                    const double W = T.wq[a] * T.wq[bq] * fg[0];
                    const double jump = um - up;
                    const double gam = d == 0 ? Ms.gamma[0] : (d == 1 ? Ms.gamma[1] : Ms.gamma[2]);
                    const double Cvm = W * (-0.5 * (gm + gp) + gam * jump);
                    const double Cg = -0.5 * W * jump * cF;
                    Cv = side ? Cvm : -Cvm;
                    C1 = (side ? amt1 : apt1) * Cg;
                    C2 = (side ? amt2 : apt2) * Cg;
                    Cn = (side ? amd : apd) * Cg;
                }
                F2[p] = Cv;
                F2[M2 + p] = C1;
                F2[2 * M2 + p] = C2;
                F2[3 * M2 + p] = Cn;
            }
            __syncwarp();
            {
                // back along t2: Pv = A^T Cv + D^T C2, Pt = A^T C1, Pn = A^T Cn  -> F1 [t1 = M][t2 = N]
                using F = qd::Sw2<M, M, 1, N, true, false>;
                using FA = qd::Sw2<M, M, 1, N, true, true>;
                for (int t = lane; t < 3 * F::NL; t += 32) {
                    const int k = t / F::NL, l = t - k * F::NL;
                    const double* C = b + L::F2;
                    if (k == 0) { F::line(C, b + L::F1, T.A, l); FA::line(C + 2 * M2, b + L::F1, T.Dq, l); }
                    else if (k == 1) F::line(C + M2, b + L::F1 + NM, T.A, l);
                    else F::line(C + 3 * M2, b + L::F1 + 2 * NM, T.A, l);
                }
            }
            __syncwarp();
            {
                // back along t1: V2 = A^T Pv + D^T Pt, G2 = A^T Pn  -> FT [t1 = N][t2 = N]
                using F = qd::Sw2<M, N, 0, N, true, false>;
                using FA = qd::Sw2<M, N, 0, N, true, true>;
                for (int t = lane; t < 2 * F::NL; t += 32) {
                    const int k = t / F::NL, l = t - k * F::NL;
                    if (k == 0) { F::line(b + L::F1, b + L::FT, T.A, l); FA::line(b + L::F1 + NM, b + L::FT, T.Dq, l); }
                    else F::line(b + L::F1 + 2 * NM, b + L::FT + N2, T.A, l);
                }
            }
            __syncwarp();
            // R += e_side V2 + d_side G2 along the normal lines
            for (int p = lane; p < N2; p += 32) {
                const int a = p % N, bq = p / N;
                const double V = b[L::FT + p], G = b[L::FT + N2 + p];
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    const int P = pidx<N>(d, j, a, bq);
                    b[L::R + P] = fma(side ? T.e1[j] : T.e0[j], V, fma(side ? T.d1[j] : T.d0[j], G, b[L::R + P]));
                }
            }
            __syncwarp();
        }
        for (int i = lane; i < N3; i += 32) r[cg * N3 + i] = b[L::R + i];
        __syncwarp();
    }
}

} // namespace dg
