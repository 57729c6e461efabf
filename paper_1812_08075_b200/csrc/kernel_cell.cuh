// K1+K2 (general): one fused cell-centric kernel — volume (Alg. assembly) and the
// six faces of each cell — for any geometry (axis-aligned or per-cell affine)
// and coefficient (c = 1 or c(x)). Each cell's residual block is written exactly once.
//
// Mapping: CPB cells per CTA, N^2 threads per cell; thread (a, b) owns, for every direction
// d, the 1D line along d with tangential coordinates (a, b) — the unit of one sum-factorisation
// sweep (a 1D contraction with the n x n table D, Eq. lowcomplex). The cell block X,
// the gradient/flux tensors and the residual R live in shared memory.
//
//   stage 1: d_hat_d U = (D along d) X, d = 0,1,2. Under collocation
//            (Lagrange on the Gauss nodes) A = I so U = X and the value sweeps vanish.
//   stage 2: Q = w_q c(x_q) |det J| J^{-1} J^{-T} grad_hat U  (pointwise)
//   stage 3: R = sum_d (D^T along d) Q_d
//   faces  : for each of the 6 faces, traces u, d_hat_n u of the cell and of the neighbour
//            (1-point tables e0/e1/d0/d1 in the normal direction, contracting
//            the normal direction first), tangential derivatives by D on the face
//            (affine only), the SIPG flux (Eq. diffreac_weak, theta = -1), and
//            back-projection onto the cell's own block with the transposed face tables.
#pragma once

#include "common.cuh"

namespace dg {

template <int N>
struct CellCfg {
    static constexpr int CPB = (N == 2) ? 32 : (N == 3) ? 14 : (N == 4) ? 8 : (N == 5) ? 5 : (N == 6) ? 3 : 2;
    static constexpr int THREADS = CPB * N * N;
};

template <int N, bool AFFINE, bool COEFF>
__global__ void __launch_bounds__(CellCfg<N>::THREADS)
k_cell_general(const double* __restrict__ x, const double* __restrict__ xb, const double* __restrict__ xa,
               double* __restrict__ r, long long c_begin, long long c_end, Tab<N> T, MeshArgs M)
{
    constexpr int CPB = CellCfg<N>::CPB;
    constexpr int NN = N * N, N3 = N * N * N;
    __shared__ double sX[CPB][N3];
    __shared__ double sQ[CPB][3][N3];
    __shared__ double sR[CPB][N3];
    __shared__ double sD[N * N];

    const int s = threadIdx.x / NN;
    const int t = threadIdx.x % NN;
    const int ta = t % N, tb = t / N;
    const long long cfirst = c_begin + (long long)blockIdx.x * CPB;
    const long long lc = cfirst + s;
    const bool valid = lc < c_end;
    const int ncell_here = (int)min((long long)CPB, c_end - cfirst);

    for (int i = threadIdx.x; i < N * N; i += blockDim.x) sD[i] = T.D[i];
    {
        const double* src = x + cfirst * N3;
        double* dst = &sX[0][0];
        for (int i = threadIdx.x; i < ncell_here * N3; i += blockDim.x) dst[i] = __ldg(src + i);
    }

    // cell coordinates (local plane lp, in-plane index rem)
    const long long lcv = valid ? lc : c_begin;
    const int lp = (int)(lcv / M.plane_cells);
    const int rem = (int)(lcv % M.plane_cells);
    const int i1 = rem / M.N2, i2 = rem % M.N2;
    const int ig[3] = {(M.plane_begin + lp) % M.N0, i1, i2};

    // per-cell geometry
    double J[9], Jinv[9], adet = 1.0;
    double Gt[6]; // |det| J^{-1} J^{-T}: (00, 11, 22, 01, 02, 12)
    if (AFFINE) {
        const double* jp = M.jac + ((long long)(lp + 1) * M.plane_cells + rem) * 9;
#pragma unroll
        for (int i = 0; i < 9; ++i) J[i] = __ldg(jp + i);
        adet = fabs(inv3(J, Jinv));
        auto g = [&](int a, int b) {
            return adet * (Jinv[3 * a] * Jinv[3 * b] + Jinv[3 * a + 1] * Jinv[3 * b + 1] + Jinv[3 * a + 2] * Jinv[3 * b + 2]);
        };
        Gt[0] = g(0, 0); Gt[1] = g(1, 1); Gt[2] = g(2, 2); Gt[3] = g(0, 1); Gt[4] = g(0, 2); Gt[5] = g(1, 2);
    } else {
#pragma unroll
        for (int i = 0; i < 9; ++i) J[i] = 0.0;
        J[0] = M.h[0]; J[4] = M.h[1]; J[8] = M.h[2];
        adet = M.h[0] * M.h[1] * M.h[2];
        Gt[0] = adet / (M.h[0] * M.h[0]); Gt[1] = adet / (M.h[1] * M.h[1]); Gt[2] = adet / (M.h[2] * M.h[2]);
        Gt[3] = Gt[4] = Gt[5] = 0.0;
    }
    const double o[3] = {(double)ig[0] / M.N0, (double)ig[1] / M.N1, (double)ig[2] / M.N2};
    __syncthreads();

    // ---------------- stage 1: reference gradients (3 sweeps) ----------------
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double xl[N];
#pragma unroll
        for (int j = 0; j < N; ++j) xl[j] = sX[s][pidx<N>(d, j, ta, tb)];
#pragma unroll
        for (int q = 0; q < N; ++q) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) acc = fma(T.D[q * N + j], xl[j], acc);
            sQ[s][d][pidx<N>(d, q, ta, tb)] = acc;
        }
    }
    __syncthreads();

    // ---------------- stage 2: pointwise flux ----------------
#pragma unroll
    for (int m = 0; m < N; ++m) {
        const int P = t + NN * m; // q0 = ta, q1 = tb, q2 = m
        const double W = T.w[ta] * T.w[tb] * T.w[m];
        double cW = W;
        if (COEFF) {
            const double xi0 = T.xi[ta], xi1 = T.xi[tb], xi2 = T.xi[m];
            const double x0 = o[0] + J[0] * xi0 + J[1] * xi1 + J[2] * xi2;
            const double x1 = o[1] + J[3] * xi0 + J[4] * xi1 + J[5] * xi2;
            cW *= coeff_sincos(x0, x1);
        }
        const double g0 = sQ[s][0][P], g1 = sQ[s][1][P], g2 = sQ[s][2][P];
        if (AFFINE) {
            sQ[s][0][P] = cW * (Gt[0] * g0 + Gt[3] * g1 + Gt[4] * g2);
            sQ[s][1][P] = cW * (Gt[3] * g0 + Gt[1] * g1 + Gt[5] * g2);
            sQ[s][2][P] = cW * (Gt[4] * g0 + Gt[5] * g1 + Gt[2] * g2);
        } else {
            sQ[s][0][P] = cW * Gt[0] * g0;
            sQ[s][1][P] = cW * Gt[1] * g1;
            sQ[s][2][P] = cW * Gt[2] * g2;
        }
    }
    __syncthreads();

    // ---------------- stage 3: transposed sweeps into R ----------------
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double ql[N];
#pragma unroll
        for (int q = 0; q < N; ++q) ql[q] = sQ[s][d][pidx<N>(d, q, ta, tb)];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) acc = fma(T.D[q * N + i], ql[q], acc);
            const int P = pidx<N>(d, i, ta, tb);
            sR[s][P] = (d == 0) ? acc : sR[s][P] + acc;
        }
        __syncthreads();
    }

    // ---------------- faces ----------------
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const int t1 = (d == 0) ? 1 : 0;
        const int t2 = (d == 2) ? 1 : 2;
        double Rl[N];
#pragma unroll
        for (int i = 0; i < N; ++i) Rl[i] = sR[s][pidx<N>(d, i, ta, tb)];
        double xl[N];
#pragma unroll
        for (int j = 0; j < N; ++j) xl[j] = sX[s][pidx<N>(d, j, ta, tb)];

#pragma unroll
        for (int side = 0; side < 2; ++side) {
            // side 1: face at xi_d = 1, this cell is T-; side 0: face at xi_d = 0, this cell is T+.
            // own-side and neighbour-side 1-point face tables (compile-time side => constant operands)
            auto eo = [&](int j) { return side ? T.e1[j] : T.e0[j]; };
            auto dO = [&](int j) { return side ? T.d1[j] : T.d0[j]; };
            auto en = [&](int j) { return side ? T.e0[j] : T.e1[j]; };
            auto dN = [&](int j) { return side ? T.d0[j] : T.d1[j]; };
            // neighbour cell (local plane / in-plane index)
            int nlp = lp, nrem = rem;
            int nig[3] = {ig[0], ig[1], ig[2]};
            const int delta = side ? 1 : -1;
            nig[d] = (ig[d] + delta + (d == 0 ? M.N0 : d == 1 ? M.N1 : M.N2)) % (d == 0 ? M.N0 : d == 1 ? M.N1 : M.N2);
            const double* nbx;
            if (d == 0) {
                nlp = lp + delta;
                nbx = (nlp < 0) ? xb + (long long)rem * N3
                                : (nlp >= M.L ? xa + (long long)rem * N3 : x + ((long long)nlp * M.plane_cells + rem) * N3);
            } else {
                nrem = nig[1] * M.N2 + nig[2];
                nbx = x + ((long long)lp * M.plane_cells + nrem) * N3;
            }
            double uo = 0.0, go = 0.0, un = 0.0, gn = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                uo = fma(eo(j), xl[j], uo);
                go = fma(dO(j), xl[j], go);
            }
            if (valid) {
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    const double v = __ldg(nbx + pidx<N>(d, j, ta, tb));
                    un = fma(en(j), v, un);
                    gn = fma(dN(j), v, gn);
                }
            }
            const double um = side ? uo : un, up = side ? un : uo;
            const double gmd = side ? go : gn, gpd = side ? gn : go;
            // T- cell global coordinates (for the face quadrature points x_F and c_F)
            int mig[3] = {ig[0], ig[1], ig[2]};
            if (!side) mig[d] = nig[d];
            const double xi_a = T.xi[ta], xi_b = T.xi[tb];
            const double jump = um - up;
            double Cv, G, ct1 = 0.0, ct2 = 0.0;
            if (!AFFINE) {
                const double hd = M.h[d];
                const double W = T.w[ta] * T.w[tb] * (adet / hd);
                double cF = 1.0;
                if (COEFF) {
                    double xF[3];
                    xF[d] = (double)mig[d] / (d == 0 ? M.N0 : d == 1 ? M.N1 : M.N2) + M.h[d];
                    xF[t1] = (double)mig[t1] / (t1 == 0 ? M.N0 : M.N1) + M.h[t1] * xi_a;
                    xF[t2] = (double)mig[t2] / (t2 == 1 ? M.N1 : M.N2) + M.h[t2] * xi_b;
                    cF = coeff_sincos(xF[0], xF[1]);
                }
                const double avg = 0.5 * cF * (gmd + gpd) / hd;
                Cv = side ? W * (-avg + M.gamma[d] * jump) : W * (avg - M.gamma[d] * jump);
                G = -0.5 * W * jump * cF / hd;
            } else {
                // geometry of both sides
                double Jn[9], Jm[9], Jp[9], Jminv[9], Jpinv[9];
                {
                    const int gl = (d == 0) ? nlp : lp;
                    const double* jp = M.jac + ((long long)(gl + 1) * M.plane_cells + (d == 0 ? rem : nrem)) * 9;
#pragma unroll
                    for (int i = 0; i < 9; ++i) Jn[i] = __ldg(jp + i);
                }
#pragma unroll
                for (int i = 0; i < 9; ++i) { Jm[i] = side ? J[i] : Jn[i]; Jp[i] = side ? Jn[i] : J[i]; }
                const double detm = inv3(Jm, Jminv);
                inv3(Jp, Jpinv);
                // nu = J_-^{-T} e_d, n_F = nu/|nu|, dS = |det J_-| |nu|  (Nanson)
                const double nu0 = Jminv[3 * d], nu1 = Jminv[3 * d + 1], nu2 = Jminv[3 * d + 2];
                const double nn = sqrt(nu0 * nu0 + nu1 * nu1 + nu2 * nu2);
                const double nF[3] = {nu0 / nn, nu1 / nn, nu2 / nn};
                const double sF = fabs(detm) * nn;
                double am[3], ap[3]; // J^{-1} n_F per side: grad u . n_F = grad_hat u . (J^{-1} n_F)
#pragma unroll
                for (int e = 0; e < 3; ++e) {
                    am[e] = Jminv[3 * e] * nF[0] + Jminv[3 * e + 1] * nF[1] + Jminv[3 * e + 2] * nF[2];
                    ap[e] = Jpinv[3 * e] * nF[0] + Jpinv[3 * e + 1] * nF[1] + Jpinv[3 * e + 2] * nF[2];
                }
                // tangential derivatives of the u traces on the face (D along t1, t2)
                double* fm = &sQ[s][0][0];
                double* fp = &sQ[s][1][0];
                fm[t] = um;
                fp[t] = up;
                __syncthreads();
                double dm1 = 0.0, dm2 = 0.0, dp1 = 0.0, dp2 = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    const double Da = sD[ta * N + j], Db = sD[tb * N + j];
                    dm1 = fma(Da, fm[j + N * tb], dm1);
                    dp1 = fma(Da, fp[j + N * tb], dp1);
                    dm2 = fma(Db, fm[ta + N * j], dm2);
                    dp2 = fma(Db, fp[ta + N * j], dp2);
                }
                double xim[3];
                xim[d] = 1.0; xim[t1] = xi_a; xim[t2] = xi_b;
                double cF = 1.0;
                if (COEFF) {
                    const double om0 = (double)mig[0] / M.N0, om1 = (double)mig[1] / M.N1;
                    const double x0 = om0 + Jm[0] * xim[0] + Jm[1] * xim[1] + Jm[2] * xim[2];
                    const double x1 = om1 + Jm[3] * xim[0] + Jm[4] * xim[1] + Jm[5] * xim[2];
                    cF = coeff_sincos(x0, x1);
                }
                const double gm = cF * (am[d] * gmd + am[t1] * dm1 + am[t2] * dm2);
                const double gp = cF * (ap[d] * gpd + ap[t1] * dp1 + ap[t2] * dp2);
                const double avg = 0.5 * (gm + gp);
                const double W = T.w[ta] * T.w[tb] * sF;
                Cv = side ? W * (-avg + M.gamma[d] * jump) : W * (avg - M.gamma[d] * jump);
                const double Cg = -0.5 * W * jump * cF;
                const double* ao = side ? am : ap;
                G = ao[d] * Cg;
                ct1 = ao[t1] * Cg;
                ct2 = ao[t2] * Cg;
                __syncthreads();
                double* f1 = &sQ[s][2][0];
                double* f2 = &sQ[s][2][NN];
                f1[t] = ct1;
                f2[t] = ct2;
                __syncthreads();
                double v = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    v = fma(sD[j * N + ta], f1[j + N * tb], v);
                    v = fma(sD[j * N + tb], f2[ta + N * j], v);
                }
                Cv += v;
                __syncthreads();
            }
#pragma unroll
            for (int i = 0; i < N; ++i) Rl[i] = fma(eo(i), Cv, fma(dO(i), G, Rl[i]));
        }
#pragma unroll
        for (int i = 0; i < N; ++i) sR[s][pidx<N>(d, i, ta, tb)] = Rl[i];
        __syncthreads();
    }

    // ---------------- write r once ----------------
    {
        double* dst = r + cfirst * N3;
        const double* src = &sR[0][0];
        for (int i = threadIdx.x; i < ncell_here * N3; i += blockDim.x) dst[i] = src[i];
    }
}

} // namespace dg
