// K_axis8: axis-aligned Poisson (c = 1), n = 8 (Q7, cfg3) — the benchmark kernel.
//
// Algebra (exact reordering of Alg. assembly, for J = diag(h), c = 1):
// with collocation (A = I) the flux of stage 2 is diagonal, so stage 1 -> 2 -> 3 along one
// direction d collapses into the 1D stiffness  (1/h_d) D^T W D  applied to every line of the
// cell along d, scaled by the tangential weights w_a w_b h_t1 h_t2. The face terms of
// Eq. diffreac_weak (theta = -1) on faces normal to d only touch the same lines
// (tangential basis functions are nodal at the face quadrature points), so per line
//
//   r_line += S_ab [ B^ x_line + a^_L u_L + b^_L g_L + a^_R u_R + b^_R g_R ],  S_ab = w_a w_b h_t1 h_t2 / h_d
//   B^   = D^T W D + 1/2 (e0 d0^T + d0 e0^T - e1 d1^T - d1 e1^T) + P (e0 e0^T + e1 e1^T),  P = penalty_scale k(k+1)
//   u_L = e1.x_L, g_L = d1.x_L  (traces of the lower neighbour along d; 1-point tables)
//   u_R = e0.x_R, g_R = d0.x_R  (upper neighbour),  a^_L = -d0/2 - P e0, b^_L = e0/2, a^_R = d1/2 - P e1, b^_R = -e1/2.
// This is the sum-factorised operator with the face contraction done first in the normal
// direction. B^ is centro-symmetric (symmetric Gauss nodes), so every line product
// runs in even/odd form: 2 (4x4) products instead of one 8x8.
//
// Mapping (B200): one CTA owns a T1 x T2 tile of cells in (i1, i2) (2x4 with 256 threads and
// 97 KB smem, 2 CTAs per SM; or 4x4 / 512 threads / 193 KB) and MARCHES along i0 through the
// planes [p_begin, p_end):
//   * each plane's 16 blocks (64 KB) arrive by TMA (cp.async.bulk.tensor, 128B swizzle) into a
//     double buffer one plane ahead of use;
//   * pass d=1 and pass d=2: a thread owns one line position across up to 2 cells of a tile row
//     (and its partner lane, lane ^ 16, the other 2 of a 4-cell row), so the neighbour traces
//     inside the tile stay in registers (one shuffle pair per pass); the ring cells outside the
//     tile are read from L2 (their owner CTAs stream them concurrently);
//   * pass d=0 (the marching direction): the lower neighbour's traces are carried in registers
//     from the previous plane, the upper neighbour's come from the prefetched next plane;
//   * partial sums of the three passes meet in a swizzled smem buffer; the d=0 pass adds them
//     and writes r straight to global memory, once, with 64-byte coalesced rows.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace dg {

struct AxisTab8 {
    // Even/odd halves of the volume stiffness K = D^T W D (symmetric: the kernels read [min(i,j)][max(i,j)]).
    // The face part of B^ and the neighbour couplings are rank-2 per parity in the trace vectors, so the line
    // operator needs only K, the trace vectors and P (37 distinct doubles in the hot loop instead of 80: sm_100a
    // DFMA takes table operands from uniform registers, and 31 doubles fit there; see line_eo):
    double Ke[4][4], Ko[4][4];
    double te[4], to[4], qe[4], qo[4];   // e0 and d0 in even/odd form: e0.x = TE + TO, e1.x = TE - TO, ...
    double P;                            // penalty_scale k (k+1)
    double w[8];
    double c[3];                         // h_t1 h_t2 / h_d
};

namespace ax8 {

constexpr int N = 8;
constexpr int CELL_BYTES = N * N * N * 8; // 4096

// tile T1 x T2 cells in (i1, i2), NT threads
template <int T1, int T2, int NT>
struct Cfg {
    static constexpr int CELLS = T1 * T2;
    static constexpr int BUF_BYTES = CELLS * CELL_BYTES;
    static constexpr int SMEM_BYTES = 3 * BUF_BYTES + 1024; // X0, X1, R (+ barriers, alignment slack)
    static constexpr int WARPS = NT / 32;
    static constexpr int LPT = 64 * CELLS / NT; // pass d=0: lines per thread (1 or 2)
    static constexpr int WPC = 2 / LPT;         // pass d=0: warps per cell
    static_assert(LPT * NT == 64 * CELLS && (LPT == 1 || LPT == 2), "pass d=0 mapping");
    static constexpr int MINB = (SMEM_BYTES <= 56 * 1024) ? 4 : (SMEM_BYTES <= 113 * 1024) ? 2 : 1;
};

__device__ __forceinline__ uint32_t swz(uint32_t off) { return off ^ (((off >> 7) & 7u) << 4); }

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ double lds(uint32_t a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void lds2(uint32_t a, double& x, double& y)
{
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ void sts(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

// Trace sums of a line in even/odd form: TE = te.xe, TO = to.xo, QE = qe.xe, QO = qo.xo, so that
// e0.x = TE + TO, e1.x = TE - TO, d0.x = QE + QO, d1.x = QO - QE (1-point tables).
struct Sums {
    double TE, TO, QE, QO;
};
__host__ __device__ __forceinline__ Sums sums_eo(const AxisTab8& A, const double xe[4], const double xo[4])
{
    Sums t{0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        t.TE = fma(A.te[j], xe[j], t.TE);
        t.TO = fma(A.to[j], xo[j], t.TO);
        t.QE = fma(A.qe[j], xe[j], t.QE);
        t.QO = fma(A.qo[j], xo[j], t.QO);
    }
    return t;
}
__host__ __device__ __forceinline__ void split8(const double v[8], double xe[4], double xo[4])
{
#pragma unroll
    for (int j = 0; j < 4; ++j) { xe[j] = v[j] + v[7 - j]; xo[j] = v[j] - v[7 - j]; }
}

// Even/odd line kernel: y = B^ x + a^_L uL + b^_L gL + a^_R uR + b^_R gR in the halves ye (y_i + y_{7-i} parts), yo.
// With B^ = K + 1/2 (e0 d0^T + d0 e0^T - e1 d1^T - d1 e1^T) + P (e0 e0^T + e1 e1^T) (header) and the couplings
// a^_L = -d0/2 - P e0, b^_L = e0/2, a^_R = d1/2 - P e1, b^_R = -e1/2, the even half is
//   ye_i = (Ke xe)_i + te_i (2P TE + QE + dg/2 - P su) + qe_i (TE - su/2)
// and the odd half
//   yo_i = (Ko xo)_i + to_i (2P TO + QO + sg/2 - P du) + qo_i (TO - du/2)
// (su = uL + uR, du = uL - uR, sg = gL + gR, dg = gL - gR): the same FMAs per output as a full B^ table, from
// the trace sums the caller forms anyway.
__host__ __device__ __forceinline__ void line_eo(const AxisTab8& A, const double xe[4], const double xo[4], const Sums& t,
                                        double uL, double gL, double uR, double gR, double ye[4], double yo[4])
{
    const double su = uL + uR, du = uL - uR, sg = gL + gR, dg = gL - gR;
    const double ae = fma(A.P, fma(2.0, t.TE, -su), fma(0.5, dg, t.QE)), be = fma(-0.5, su, t.TE);
    const double ao = fma(A.P, fma(2.0, t.TO, -du), fma(0.5, sg, t.QO)), bo = fma(-0.5, du, t.TO);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        double e = fma(A.te[i], ae, A.qe[i] * be);
        double o = fma(A.to[i], ao, A.qo[i] * bo);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            e = fma(A.Ke[i < j ? i : j][i < j ? j : i], xe[j], e);
            o = fma(A.Ko[i < j ? i : j][i < j ? j : i], xo[j], o);
        }
        ye[i] = e;
        yo[i] = o;
    }
}

// In-plane pass (pd = 1: lines along j1 / neighbours along i1; pd = 2: along j2 / i2).
// TL = tile cells along the pass direction, TW = across. G = threads per tile row (1 or 2).
template <int pd, int TL, int TW, int NT>
__device__ __forceinline__ void inplane_pass(const AxisTab8& A, const MeshArgs& M, const double* __restrict__ x, uint32_t X,
                                             uint32_t R, int lp, int ti1, int ti2, int tid, double S)
{
    constexpr int G = (64 * TW * TL / NT == TL) ? 1 : 2; // cells per thread == TL -> one thread per row
    constexpr int CPT = TL / G;
    static_assert(G * CPT == TL && 64 * TW * G == NT, "pass mapping");
    constexpr int T1 = (pd == 1) ? TL : TW, T2 = (pd == 1) ? TW : TL;
    const int j0 = tid & 7, jb = (tid >> 3) & 1, hb = (tid >> 4) & 1, rest = tid >> 5;
    int half, jt, tw;
    if (G == 2) { half = hb; jt = jb + 2 * (rest & 3); tw = rest >> 2; }
    else        { half = 0;  jt = jb + 2 * hb + 4 * (rest & 1); tw = rest >> 1; }
    auto eoff = [&](int j) { return pd == 1 ? j0 + 8 * j + 64 * jt : j0 + 8 * jt + 64 * j; };
    auto bcell = [&](int cc) { const int a = half * CPT + cc; return pd == 1 ? a * T2 + tw : tw * T2 + a; };
    auto cidx = [&](int i1, int i2) -> long long { return (long long)lp * M.plane_cells + (long long)i1 * M.N2 + i2; };
    // ring cells (tile neighbours along the pass direction)
    long long rlo, rhi;
    if (pd == 1) {
        rlo = cidx((ti1 * T1 - 1 + M.N1) % M.N1, ti2 * T2 + tw);
        rhi = cidx((ti1 * T1 + T1) % M.N1, ti2 * T2 + tw);
    } else {
        rlo = cidx(ti1 * T1 + tw, (ti2 * T2 - 1 + M.N2) % M.N2);
        rhi = cidx(ti1 * T1 + tw, (ti2 * T2 + T2) % M.N2);
    }
    constexpr int NR = (G == 1) ? 2 : 1;
#ifndef DG_AX8_NO_RING_PREFETCH
    // the next plane's ring lines into L2 (evict_last) one plane ahead: about 40 % of the ring-line reads missed
    // L2 (ncu: 1.14 GB of DRAM reads above the algorithmic 7.25 GB per cfg3 launch) and stalled the pass
    if (lp + 1 < M.L) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const long long rc = (G == 1 ? (k ? rhi : rlo) : (half ? rhi : rlo)) + M.plane_cells;
            // thread j0 of each 8-lane group touches row j = j0: together they cover the whole line
            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(x + rc * 512 + eoff(j0)));
        }
    }
#endif
    DG_CHECK(lp >= 0 && lp < M.L && rlo >= 0 && rlo < (long long)M.L * M.plane_cells && rhi >= 0 &&
             rhi < (long long)M.L * M.plane_cells);
    double rv[NR][8];
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        const double* g = x + ((G == 1 ? (k ? rhi : rlo) : (half ? rhi : rlo))) * 512;
#pragma unroll
        for (int j = 0; j < 8; ++j) rv[k][j] = __ldg(g + eoff(j));
    }
    double xe[CPT][4], xo[CPT][4], u0[CPT], u1[CPT], g0[CPT], g1[CPT];
    Sums ts[CPT];
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) {
        const uint32_t cb = X + bcell(cc) * CELL_BYTES;
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = lds(cb + swz(8 * eoff(j)));
        split8(v, xe[cc], xo[cc]);
        ts[cc] = sums_eo(A, xe[cc], xo[cc]);
        u0[cc] = ts[cc].TE + ts[cc].TO;
        u1[cc] = ts[cc].TE - ts[cc].TO;
        g0[cc] = ts[cc].QE + ts[cc].QO;
        g1[cc] = ts[cc].QO - ts[cc].QE;
    }
    // ring traces: lower ring cell -> (e1.x, d1.x); upper -> (e0.x, d0.x) (the same even/odd sums)
    double loU = 0, loG = 0, hiU = 0, hiG = 0;
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        const bool up = (G == 1) ? (k == 1) : (half == 1);
        double re[4], ro[4];
        split8(rv[k], re, ro);
        const Sums t = sums_eo(A, re, ro);
        const double a = up ? t.TE + t.TO : t.TE - t.TO;
        const double b = up ? t.QE + t.QO : t.QO - t.QE;
        if (G == 1) { if (k) { hiU = a; hiG = b; } else { loU = a; loG = b; } }
        else { loU = hiU = a; loG = hiG = b; }
    }
    double recvU = 0.0, recvG = 0.0;
    if (G == 2) {
        const double sendU = half ? u0[0] : u1[CPT - 1];
        const double sendG = half ? g0[0] : g1[CPT - 1];
        recvU = __shfl_xor_sync(0xffffffffu, sendU, 16);
        recvG = __shfl_xor_sync(0xffffffffu, sendG, 16);
    }
#pragma unroll
    for (int cc = 0; cc < CPT; ++cc) {
        double uL, gL, uR, gR;
        if (cc > 0) { uL = u1[cc - 1]; gL = g1[cc - 1]; }
        else if (G == 2 && half) { uL = recvU; gL = recvG; }
        else { uL = loU; gL = loG; }
        if (cc < CPT - 1) { uR = u0[cc + 1]; gR = g0[cc + 1]; }
        else if (G == 2 && !half) { uR = recvU; gR = recvG; }
        else { uR = hiU; gR = hiG; }
        double ye[4], yo[4];
        line_eo(A, xe[cc], xo[cc], ts[cc], uL, gL, uR, gR, ye, yo);
        const uint32_t rb = R + bcell(cc) * CELL_BYTES;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t p0 = rb + swz(8 * eoff(i));
            const uint32_t p1 = rb + swz(8 * eoff(7 - i));
            if (pd == 1) {
                sts(p0, S * (ye[i] + yo[i]));
                sts(p1, S * (ye[i] - yo[i]));
            } else {
                sts(p0, fma(S, ye[i] + yo[i], lds(p0)));
                sts(p1, fma(S, ye[i] - yo[i], lds(p1)));
            }
        }
    }
}

// thread's tangential weights product for the in-plane passes (same decomposition as above)
template <int pd, int TL, int TW, int NT>
__device__ __forceinline__ double inplane_scale(const AxisTab8& A, int tid)
{
    constexpr int G = (64 * TW * TL / NT == TL) ? 1 : 2;
    const int j0 = tid & 7, jb = (tid >> 3) & 1, hb = (tid >> 4) & 1, rest = tid >> 5;
    const int jt = (G == 2) ? jb + 2 * (rest & 3) : jb + 2 * hb + 4 * (rest & 1);
    double wj0 = 0.0, wjt = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { // uniform-index table reads (no divergent constant loads)
        wj0 = (i == j0) ? A.w[i] : wj0;
        wjt = (i == jt) ? A.w[i] : wjt;
    }
    return wj0 * wjt * A.c[pd];
}

} // namespace ax8

// Halo traces of a slab for k_axis8 contexts (dg_pack_halo): lower-end (e0.x, d0.x) of the first plane's d = 0
// lines, upper-end (e1.x, d1.x) of the last plane's, with k_axis8's own even/odd trace algebra (bitwise the values
// its pass d = 0 computes from a block halo); per cell u[64] then d_0 u[64], line L = j1 + 8 j2.
__global__ void k_pack_traces8(const double* __restrict__ x, double* __restrict__ lo, double* __restrict__ hi,
                               int plane_cells, int L, const AxisTab8 A)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2LL * plane_cells * 64) return;
    const int side = (int)(t / ((long long)plane_cells * 64));
    const long long rem = t - (long long)side * plane_cells * 64;
    const long long c = rem / 64;
    const int l = (int)(rem - c * 64);
    const double* src = x + ((long long)(side ? L - 1 : 0) * plane_cells + c) * 512 + 8 * l;
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldg(src + j);
    double* o = (side ? hi : lo) + c * 128;
    double xe[4], xo[4];
    ax8::split8(v, xe, xo);
    const ax8::Sums ts = ax8::sums_eo(A, xe, xo);
    if (side) { // upper end (e1.x, d1.x)
        o[l] = ts.TE - ts.TO;
        o[64 + l] = ts.QO - ts.QE;
    } else {    // lower end (e0.x, d0.x)
        o[l] = ts.TE + ts.TO;
        o[64 + l] = ts.QE + ts.QO;
    }
}

// grid: (N1/T1) * (N2/T2) CTAs, block NT, dynamic smem Cfg::SMEM_BYTES
template <int T1, int T2, int NT, int MB = ax8::Cfg<T1, T2, NT>::MINB>
__global__ void __launch_bounds__(NT, MB)
k_axis8(const __grid_constant__ CUtensorMap tmx, const double* __restrict__ x, const double* __restrict__ xb,
        const double* __restrict__ xa, double* __restrict__ r, int p_begin, int p_end, int chunk_len, int halo_tr,
        const AxisTab8 A, const MeshArgs M, long long* __restrict__ dbg)
{
    using namespace ax8;
    using C = Cfg<T1, T2, NT>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 32-bit shared-window addresses (explicit ld/st.shared; 1024-aligned for the 128B swizzle)
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t bufX[2] = {sbase, sbase + C::BUF_BYTES};
    const uint32_t bufR = sbase + 2 * C::BUF_BYTES;
    const uint32_t bar0 = sbase + 3 * C::BUF_BYTES;
    auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ntile2 = M.N2 / T2;
    const int ntiles = (M.N1 / T1) * ntile2;
    // work item = (plane chunk, tile), chunk-major: concurrently resident CTAs march the same
    // planes, so their ring cells (each other's own cells) are L2 hits
    const int chunk = blockIdx.x / ntiles, tile = blockIdx.x % ntiles;
    const int ti1 = tile / ntile2, ti2 = tile % ntile2;
    {
        const int b = p_begin + chunk * chunk_len;
        p_end = min(p_end, b + chunk_len);
        p_begin = b;
    }
    const int PC = M.plane_cells;
    const int nsteps = p_end - p_begin;
    if (nsteps <= 0) return;

    auto cell_index = [&](int lp, int i1, int i2) -> long long { return (long long)lp * PC + (long long)i1 * M.N2 + i2; };

    // the TMA producer is lane 0 of the last warp (warp 0 carries the trace stamps)
    const bool producer = (tid == NT - 32);
    if (producer) {
        mbar_init(bar(0), 1);
        mbar_init(bar(1), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmx)) : "memory");
    }
    __syncthreads();

    auto issue = [&](int step) {
        // TMA the T1 x T2 blocks of plane p_begin + step into buffer (step & 1): one box per tile row
        const int lp = p_begin + step;
        const uint32_t b = bar(step & 1);
        DG_CHECK(lp >= 0 && lp < M.L && (ti1 + 1) * T1 <= M.N1 && (ti2 + 1) * T2 <= M.N2);
        mbar_expect_tx(b, C::BUF_BYTES);
#pragma unroll
        for (int c1 = 0; c1 < T1; ++c1) {
            const long long cell = cell_index(lp, ti1 * T1 + c1, ti2 * T2);
            tma_load_2d(bufX[step & 1] + c1 * T2 * CELL_BYTES, &tmx, 0, (int)(cell * (CELL_BYTES / 128)), b);
        }
    };
    if (producer) {
        issue(0);
        if (nsteps > 1) issue(1);
    }

    const double S1 = inplane_scale<1, T1, T2, NT>(A, tid);
    const double S2 = inplane_scale<2, T2, T1, NT>(A, tid);
    // d=0 mapping: warp w owns (part of) cell w / WPC (buffer order c1*T2+c2); lane owns lines
    // L = lane + 32 (q + LPT (w % WPC)), q < LPT
    constexpr int LPT = C::LPT, WPC = C::WPC;
    const int dcell = warp / WPC, lbase = 32 * LPT * (warp % WPC);
    const int dc1 = dcell / T2, dc2 = dcell % T2;
    const long long d0_inplane = (long long)(ti1 * T1 + dc1) * M.N2 + ti2 * T2 + dc2;
    double S0[LPT];
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
        const int L = lane + 32 * q + lbase;
        double wa = 0.0, wb = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            wa = ((L & 7) == i) ? A.w[i] : wa;
            wb = ((L >> 3) == i) ? A.w[i] : wb;
        }
        S0[q] = wa * wb * A.c[0];
    }

    double prevU[LPT], prevG[LPT]; // traces e1.x, d1.x of the lower x0-neighbour, per d=0 line
    if (p_begin == 0 && (halo_tr & 1)) {
        // halo below given as traces (dg_apply_planes_tr): per cell u[64] then d_0 u[64] at the d = 0 face points
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
            const int L = lane + 32 * q + lbase;
            prevU[q] = __ldg(xb + d0_inplane * 128 + L);
            prevG[q] = __ldg(xb + d0_inplane * 128 + 64 + L);
        }
    } else {
        const double* src = (p_begin == 0) ? xb + d0_inplane * 512 : x + (cell_index(p_begin - 1, 0, 0) + d0_inplane) * 512;
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
            const int L = lane + 32 * q + lbase;
            const double2* s2 = reinterpret_cast<const double2*>(src + 8 * L);
            double v[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                double2 t = __ldg(s2 + k);
                v[2 * k] = t.x;
                v[2 * k + 1] = t.y;
            }
            double xe[4], xo[4];
            ax8::split8(v, xe, xo);
            const ax8::Sums ts = ax8::sums_eo(A, xe, xo);
            prevU[q] = ts.TE - ts.TO;
            prevG[q] = ts.QO - ts.QE;
        }
    }

    // optional phase timestamps (DG_TRACE): dbg[block][step][phase], first 16 steps
    const bool trace = dbg != nullptr && tid == 0 && blockIdx.x < 1024;
    auto stamp = [&](int s, int ph) {
#ifdef DG_AX8_TRACE
        if (trace && s < 16) dbg[(blockIdx.x * 16 + s) * 8 + ph] = clock64();
#else
        (void)s; (void)ph; (void)trace;
#endif
    };
    for (int s = 0; s < nsteps; ++s) {
        const int lp = p_begin + s;
        const uint32_t X = bufX[s & 1];
        stamp(s, 0);
        mbar_wait(bar(s & 1), (s >> 1) & 1);
        stamp(s, 1);

        inplane_pass<1, T1, T2, NT>(A, M, x, X, bufR, lp, ti1, ti2, tid, S1);
        stamp(s, 2);
        __syncthreads();
        stamp(s, 3);
        inplane_pass<2, T2, T1, NT>(A, M, x, X, bufR, lp, ti1, ti2, tid, S2);
        stamp(s, 4);
        __syncthreads();
        stamp(s, 5);

        // ================= pass d = 0 (lines along j0; neighbours along i0: marching) =================
        {
            const bool last = (s == nsteps - 1);
            if (!last) mbar_wait(bar((s + 1) & 1), ((s + 1) >> 1) & 1);
            const uint32_t XN = bufX[(s + 1) & 1];
            const int cb = dcell;
            const double* nsrc = (p_end == M.L) ? xa + d0_inplane * 512 : x + (cell_index(p_end, 0, 0) + d0_inplane) * 512;
#pragma unroll
            for (int q = 0; q < LPT; ++q) {
                const int L = lane + 32 * q + lbase;
                // upper neighbour's traces e0.x, d0.x
                double uR = 0.0, gR = 0.0;
                if (last && p_end == M.L && (halo_tr & 2)) {
                    uR = __ldg(xa + d0_inplane * 128 + L); // halo above as traces (e0.x, d0.x)
                    gR = __ldg(xa + d0_inplane * 128 + 64 + L);
                } else {
                    double v[8];
                    if (!last) {
                        const uint32_t nb = XN + cb * CELL_BYTES;
#pragma unroll
                        for (int k = 0; k < 4; ++k) lds2(nb + swz(8 * (8 * L + 2 * k)), v[2 * k], v[2 * k + 1]);
                    } else {
                        const double2* s2 = reinterpret_cast<const double2*>(nsrc + 8 * L);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            double2 t = __ldg(s2 + k);
                            v[2 * k] = t.x;
                            v[2 * k + 1] = t.y;
                        }
                    }
                    double ne[4], no[4];
                    ax8::split8(v, ne, no);
                    const ax8::Sums tn = ax8::sums_eo(A, ne, no);
                    uR = tn.TE + tn.TO;
                    gR = tn.QE + tn.QO;
                }
                double v[8];
                const uint32_t xcb = X + cb * CELL_BYTES;
#pragma unroll
                for (int k = 0; k < 4; ++k) lds2(xcb + swz(8 * (8 * L + 2 * k)), v[2 * k], v[2 * k + 1]);
                double xe[4], xo[4];
                ax8::split8(v, xe, xo);
                const ax8::Sums ts = ax8::sums_eo(A, xe, xo);
                double ye[4], yo[4];
                ax8::line_eo(A, xe, xo, ts, prevU[q], prevG[q], uR, gR, ye, yo);
                prevU[q] = ts.TE - ts.TO;
                prevG[q] = ts.QO - ts.QE;
                const uint32_t rb = bufR + cb * CELL_BYTES;
                double o[8];
#pragma unroll
                for (int k = 0; k < 4; ++k) lds2(rb + swz(8 * (8 * L + 2 * k)), o[2 * k], o[2 * k + 1]);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    o[i] = fma(S0[q], ye[i] + yo[i], o[i]);
                    o[7 - i] = fma(S0[q], ye[i] - yo[i], o[7 - i]);
                }
                DG_CHECK(lp >= 0 && lp < M.L && d0_inplane < PC && L < 64);
                double2* dst = reinterpret_cast<double2*>(r + (cell_index(lp, 0, 0) + d0_inplane) * 512 + 8 * L);
#pragma unroll
                for (int k = 0; k < 4; ++k) dst[k] = make_double2(o[2 * k], o[2 * k + 1]);
            }
        }
        stamp(s, 6);
        __syncthreads();
        stamp(s, 7);
        if (producer && s + 2 < nsteps) issue(s + 2);
    }
}

} // namespace dg
