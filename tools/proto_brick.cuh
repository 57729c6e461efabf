// Prototype (development, not part of libdg; measured and removed): the brick kernel for cfg1.
// K_brick: axis-aligned Poisson (c = 1) on whole, L2-resident meshes (cfg1), the line-operator algebra of k_line
// (DESIGN.md §4.1 / §4.2b; Alg. assembly P:L857-881 collapsed along each direction, face terms of Eq. diffreac_weak
// P:L986-989 through the 1-point traces P:L143-146, normal direction first P:L884) evaluated brick by brick:
//
//   * a CTA owns a 4 x 4 x 4 brick of cells: the 64 blocks are copied to shared memory once, fully coalesced (a
//     brick row of 4 cells along i2 is contiguous in the cell-blocked layout);
//   * a thread owns a PENCIL per direction d: the line (a, b) along d through the 4 cells of the brick that share
//     the other two brick coordinates. The traces of each line feed the line operators of its neighbours in the
//     same thread (registers), so a face inside the brick costs no exchange and no second trace evaluation; only
//     the two faces at the pencil's ends read the neighbour brick's line from L2 (k_line reads six neighbour lines
//     for every line it owns);
//   * directions 0 and 1 write their results to two shared buffers, direction 2 adds them and writes r once
//     (two CTA barriers per brick, no plane pipeline).
//
// The per-line arithmetic is k_line's (gn::split, gn::traces, gn::lineop; the same scale and summation order,
// y2 + y0 + y1), so the result is bitwise that of k_line (slab and host-pipeline paths keep k_line).
#pragma once

#include "common.cuh"
#include "kernel_gen.cuh"

namespace dg {

template <int N>
struct BrickCfg {
    static constexpr int B = 4;                     // cells per brick edge
    static constexpr int CELLS = B * B * B;
    static constexpr int N2 = N * N, N3 = N * N * N;
    static constexpr int NT = 256;
    static constexpr int PEN = N2 * B * B;          // pencils per direction
    static constexpr int SMEM = 3 * CELLS * N3 * 8; // x brick, R0, R1
};

// grid: (N0/4) (N1/4) (N2/4) CTAs (brick index i2 fastest), block BrickCfg::NT, dynamic smem BrickCfg::SMEM.
// Whole mesh only (periodic wrap inside x), L = N0.
template <int N>
__global__ void __launch_bounds__(BrickCfg<N>::NT, 2) k_brick(const double* __restrict__ x, double* __restrict__ r,
                                                               const EOTab<N> E, const MeshArgs M)
{
    using C = BrickCfg<N>;
    constexpr int B = C::B, N2 = C::N2, N3 = C::N3, H = EOTab<N>::H, HE = EOTab<N>::HE;
    extern __shared__ __align__(16) double sm[];
    double* const XB = sm;                 // [cell][N3], cell = (c0 B + c1) B + c2
    double* const R0 = sm + C::CELLS * N3; // direction 0 results (scaled)
    double* const R1 = R0 + C::CELLS * N3; // direction 1 results
    const int tid = threadIdx.x;
    const int nb2 = M.N2 / B, nb1 = M.N1 / B;
    const int bid = blockIdx.x;
    const int b2 = bid % nb2, b1 = (bid / nb2) % nb1, b0 = bid / (nb2 * nb1);
    auto gcell = [&](int i0, int i1, int i2) -> long long {
        i0 = i0 < 0 ? i0 + M.N0 : (i0 >= M.N0 ? i0 - M.N0 : i0);
        i1 = i1 < 0 ? i1 + M.N1 : (i1 >= M.N1 ? i1 - M.N1 : i1);
        i2 = i2 < 0 ? i2 + M.N2 : (i2 >= M.N2 ? i2 - M.N2 : i2);
        return ((long long)i0 * M.N1 + i1) * M.N2 + i2;
    };

    // ---- the brick's blocks into shared memory: B * B rows of B contiguous cells, 16-B loads when N3 is even ----
    {
        constexpr int ROW = B * N3; // doubles per brick row
        if constexpr ((N3 % 2) == 0) {
            constexpr int ROW2 = ROW / 2;
            for (int t = tid; t < B * B * ROW2; t += C::NT) {
                const int rw = t / ROW2, e = t - rw * ROW2;
                const int c0 = rw / B, c1 = rw % B;
                const double2* src = reinterpret_cast<const double2*>(x + gcell(b0 * B + c0, b1 * B + c1, b2 * B) * N3);
                reinterpret_cast<double2*>(XB + rw * ROW)[e] = __ldg(src + e);
            }
        } else {
            for (int t = tid; t < B * B * ROW; t += C::NT) {
                const int rw = t / ROW, e = t - rw * ROW;
                const int c0 = rw / B, c1 = rw % B;
                XB[rw * ROW + e] = __ldg(x + gcell(b0 * B + c0, b1 * B + c1, b2 * B) * N3 + e);
            }
        }
    }
    __syncthreads();

    // one pencil: direction d, line position (a, b), the brick coordinates (u, v) of the two other directions
    // (increasing order); the 4 cells along d at brick positions k = 0..3
    auto pencil = [&](auto DC, int pen, double* out, double yk[B][N]) {
        constexpr int d = decltype(DC)::value;
        const int ab = pen % N2, a = ab % N, b = ab / N, uv = pen / N2, u = uv % B, v = uv / B;
        auto bcell = [&](int k) { // brick cell index of position k along d
            const int c0 = d == 0 ? k : u, c1 = d == 1 ? k : (d == 0 ? u : v), c2 = d == 2 ? k : v;
            return (c0 * B + c1) * B + c2;
        };
        auto gnb = [&](int k) { // global cell of brick position k along d (k = -1, B: the neighbour bricks)
            const int c0 = d == 0 ? k : u, c1 = d == 1 ? k : (d == 0 ? u : v), c2 = d == 2 ? k : v;
            return gcell(b0 * B + c0, b1 * B + c1, b2 * B + c2);
        };
        double xe[B][HE], xo[B][H > 0 ? H : 1], ulo[B], glo[B], uhi[B], ghi[B];
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const double* blk = XB + bcell(k) * N3;
            double w[N];
#pragma unroll
            for (int j = 0; j < N; ++j) w[j] = blk[pidx<N>(d, j, a, b)];
            gn::split<N>(w, xe[k], xo[k]);
            gn::traces<N>(E, xe[k], xo[k], ulo[k], glo[k], uhi[k], ghi[k]);
        }
        // the neighbour bricks' lines facing the pencil's ends (L2)
        double uL0, gL0, uRB, gRB;
        {
            double w[N], te[HE], to[H > 0 ? H : 1], u0, g0, u1, g1;
            const double* lo = x + gnb(-1) * N3;
#pragma unroll
            for (int j = 0; j < N; ++j) w[j] = __ldg(lo + pidx<N>(d, j, a, b));
            gn::split<N>(w, te, to);
            gn::traces<N>(E, te, to, u0, g0, u1, g1);
            uL0 = u1;
            gL0 = g1;
            const double* hi = x + gnb(B) * N3;
#pragma unroll
            for (int j = 0; j < N; ++j) w[j] = __ldg(hi + pidx<N>(d, j, a, b));
            gn::split<N>(w, te, to);
            gn::traces<N>(E, te, to, u0, g0, u1, g1);
            uRB = u0;
            gRB = g0;
        }
        const double S = (E.w[a] * E.w[b]) * E.Sc[d];
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const double uL = k > 0 ? uhi[k - 1] : uL0, gL = k > 0 ? ghi[k - 1] : gL0;
            const double uR = k < B - 1 ? ulo[k + 1] : uRB, gR = k < B - 1 ? glo[k + 1] : gRB;
            double y[N];
            gn::lineop<N>(E, xe[k], xo[k], y, uL, gL, uR, gR);
            if (out) {
                double* o = out + bcell(k) * N3;
#pragma unroll
                for (int j = 0; j < N; ++j) o[pidx<N>(d, j, a, b)] = S * y[j];
            } else {
#pragma unroll
                for (int j = 0; j < N; ++j) yk[k][j] = S * y[j];
            }
        }
    };

    double yk[B][N];
    for (int p = tid; p < C::PEN; p += C::NT) pencil(std::integral_constant<int, 0>{}, p, R0, yk);
    for (int p = tid; p < C::PEN; p += C::NT) pencil(std::integral_constant<int, 1>{}, p, R1, yk);
    __syncthreads();
    for (int p = tid; p < C::PEN; p += C::NT) {
        pencil(std::integral_constant<int, 2>{}, p, nullptr, yk);
        const int ab = p % N2, a = ab % N, b = ab / N, uv = p / N2, u = uv % B, v = uv / B;
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const int bc = (u * B + v) * B + k;
            double* dst = r + gcell(b0 * B + u, b1 * B + v, b2 * B + k) * N3;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const int q = pidx<N>(2, j, a, b);
                dst[q] = yk[k][j] + R0[bc * N3 + q] + R1[bc * N3 + q];
            }
        }
    }
}

} // namespace dg
