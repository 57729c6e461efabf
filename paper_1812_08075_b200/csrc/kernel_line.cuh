// K_line: axis-aligned Poisson (c = 1), any n, for meshes whose vectors are L2-resident (cfg0, cfg1).
//
// Same algebra as the line-operator form of k_gen / k_axis8: with J = diag(h), c = 1 and
// collocation, stage 1 -> 2 -> 3 of Alg. assembly along direction d collapses into the 1D SIPG line
// operator B^ applied to every line of the cell along d, with the face terms of Eq. diffreac_weak (P:L986-989,
// theta = -1) coupling each line to the facing traces (e1.x, d1.x) / (e0.x, d0.x) of the neighbours' lines
// (1-point tables, normal direction first P:L884):
//   r_line += S_ab [ B^ x_line + (neighbour couplings) ],  S_ab = w_a w_b h_t1 h_t2 / h_d.
//
// Why a second kernel: k_gen marches a tile along i0 with a TMA pipeline one plane ahead; on a 2M-DOF mesh
// whose vectors sit in L2 that pipeline's per-plane latency (TMA wait + 3 barriers per plane, 1400 CTAs) bounds
// the apply at ~19 us whatever the tile / chunk shape. Here there is no pipeline: one thread
// per (cell, line position (a, b)) loads its cell's three lines through it and the six neighbour lines facing it
// straight from L2 (read-only path), forms the three line operators in registers, and the d = 0 / 1 results
// meet the d = 2 one in shared memory (one barrier); r is written once, coalesced.
#pragma once

#include "common.cuh"
#include "kernel_gen.cuh"

namespace dg {

template <int N>
struct LineCfg {
    static constexpr int N2 = N * N, N3 = N * N * N;
    static constexpr int NT = 128;
    static constexpr int CPB = NT / N2 > 0 ? NT / N2 : 1; // cells per CTA
    static constexpr int ACT = CPB * N2;                  // active threads
    static constexpr int SMEM = 2 * CPB * N3 * 8;
};

// grid: ceil(ncells / CPB) over the cells of local planes [p_begin, p_end); halo_tr: bit 0 / 1 the halo plane
// below / above is given as face traces (dg_apply_planes_tr, per cell u[N2] then d_0 u[N2])
template <int N>
__global__ void __launch_bounds__(LineCfg<N>::NT) k_line(const double* __restrict__ x, const double* __restrict__ xb,
                                                        const double* __restrict__ xa, double* __restrict__ r, int p_begin,
                                                        int p_end, int halo_tr, const EOTab<N> E, const MeshArgs M)
{
    using C = LineCfg<N>;
    constexpr int N2 = C::N2, N3 = C::N3, CPB = C::CPB, H = EOTab<N>::H, HE = EOTab<N>::HE;
    __shared__ double s01[2][CPB][N3];
    const int tid = threadIdx.x;
    const int PC = M.plane_cells;
    const long long cbeg = (long long)p_begin * PC, cend = (long long)p_end * PC;
    const int lc = tid / N2, ab = tid - lc * N2, a = ab % N, b = ab / N;
    const long long cell = cbeg + (long long)blockIdx.x * CPB + lc;
    const bool act = tid < C::ACT && cell < cend;
    double y2[N];
    if (act) {
        const int lp = (int)(cell / PC), rem = (int)(cell - (long long)lp * PC), i1 = rem / M.N2, i2 = rem - i1 * M.N2;
        const double* xc = x + cell * N3;
        const double wab = E.w[a] * E.w[b];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            // own line and the two facing neighbour lines (traces: lower -> (e1.x, d1.x), upper -> (e0.x, d0.x))
            // a d = 0 line is N contiguous doubles: 16-B loads when N is even (blocks are 16-B aligned then)
            auto load_line = [&](const double* blk, double* w) {
                if (d == 0 && (N % 2) == 0) {
                    const double2* l2 = reinterpret_cast<const double2*>(blk + pidx<N>(0, 0, a, b));
#pragma unroll
                    for (int j = 0; j < N / 2; ++j) {
                        const double2 t = __ldg(l2 + j);
                        w[2 * j] = t.x;
                        w[2 * j + 1] = t.y;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < N; ++j) w[j] = __ldg(blk + pidx<N>(d, j, a, b));
                }
            };
            double v[N];
            load_line(xc, v);
            double uL, gL, uR, gR;
            auto nb_traces = [&](const double* blk, bool lower) {
                double w[N];
                load_line(blk, w);
                double xe[HE], xo[H > 0 ? H : 1];
                gn::split<N>(w, xe, xo);
                double ulo, glo, uhi, ghi;
                gn::traces<N>(E, xe, xo, ulo, glo, uhi, ghi);
                if (lower) { uL = uhi; gL = ghi; }
                else { uR = ulo; gR = glo; }
            };
            if (d == 0) {
                if (lp > 0) nb_traces(xc - (long long)PC * N3, true);
                else if (halo_tr & 1) { uL = __ldg(xb + (long long)rem * 2 * N2 + ab); gL = __ldg(xb + (long long)rem * 2 * N2 + N2 + ab); }
                else nb_traces(xb + (long long)rem * N3, true);
                if (lp < M.L - 1) nb_traces(xc + (long long)PC * N3, false);
                else if (halo_tr & 2) { uR = __ldg(xa + (long long)rem * 2 * N2 + ab); gR = __ldg(xa + (long long)rem * 2 * N2 + N2 + ab); }
                else nb_traces(xa + (long long)rem * N3, false);
            } else if (d == 1) {
                const long long row = (long long)lp * PC;
                nb_traces(x + (row + (long long)(i1 > 0 ? i1 - 1 : M.N1 - 1) * M.N2 + i2) * N3, true);
                nb_traces(x + (row + (long long)(i1 < M.N1 - 1 ? i1 + 1 : 0) * M.N2 + i2) * N3, false);
            } else {
                const long long row = (long long)lp * PC + (long long)i1 * M.N2;
                nb_traces(x + (row + (i2 > 0 ? i2 - 1 : M.N2 - 1)) * N3, true);
                nb_traces(x + (row + (i2 < M.N2 - 1 ? i2 + 1 : 0)) * N3, false);
            }
            double xe[HE], xo[H > 0 ? H : 1], y[N];
            gn::split<N>(v, xe, xo);
            gn::lineop<N>(E, xe, xo, y, uL, gL, uR, gR);
            const double S = wab * E.Sc[d];
            if (d < 2) {
#pragma unroll
                for (int j = 0; j < N; ++j) s01[d][lc][pidx<N>(d, j, a, b)] = S * y[j];
            } else {
#pragma unroll
                for (int j = 0; j < N; ++j) y2[j] = S * y[j];
            }
        }
    }
    __syncthreads();
    if (act) {
        double* dst = r + cell * N3;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const int p = pidx<N>(2, j, a, b);
            dst[p] = y2[j] + s01[0][lc][p] + s01[1][lc][p];
        }
    }
}

} // namespace dg
