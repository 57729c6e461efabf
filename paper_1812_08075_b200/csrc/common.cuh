// Shared device-side definitions of the libdg kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

// Debug builds (-DDG_BOUNDS, `python -m paper_1812_08075_b200.build --bounds`): every global access and every
// bulk-copy destination of the marching-tile kernels is checked against the array / shared-memory extents
// derived from the launch arguments; a violation prints the site and traps (compute-sanitizer is not available
// on this GPU pool). Release builds compile the checks away.
#ifdef DG_BOUNDS
#define DG_CHECK(cond)                                                                                             \
    do {                                                                                                           \
        if (!(cond)) {                                                                                             \
            printf("DG_BOUNDS violation %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, blockIdx.x, \
                   threadIdx.x);                                                                                   \
            __trap();                                                                                              \
        }                                                                                                          \
    } while (0)
#else
#define DG_CHECK(cond) do { } while (0)
#endif

namespace dg {

// 1D tables passed by value as a kernel parameter (lives in the constant bank: table
// entries indexed by compile-time loop counters become DFMA constant operands).
template <int N>
struct Tab {
    double D[N * N]; // D[q*N + j] = l_j'(xi_q)
    double w[N];     // Gauss weights on [0,1]
    double xi[N];    // Gauss nodes on [0,1] (= Lagrange nodes)
    double e0[N], e1[N], d0[N], d1[N]; // l_j(0), l_j(1), l_j'(0), l_j'(1)
};

// Slab/mesh description for the kernels.
struct MeshArgs {
    int N0, N1, N2;       // global cells per direction
    int plane_begin;      // global index of local plane 0
    int L;                // local planes
    int plane_cells;      // N1 * N2
    double h[3];          // 1/N_d
    double gamma[3];      // penalty per face direction: penalty_scale k(k+1) N_d
    const double* jac;    // DEVICE (L+2) planes x plane_cells x 9 (affine only)
};

// Point index inside an n^3 block of the point at position j along direction d on the line
// with tangential coordinates (a, b) in the two other directions (increasing order).
// vec convention: P = i0 + N i1 + N^2 i2.
template <int N>
__device__ __forceinline__ constexpr int pidx(int d, int j, int a, int b)
{
    return d == 0 ? j + N * (a + N * b) : (d == 1 ? a + N * (j + N * b) : a + N * (b + N * j));
}

// c(x) = 1 + 0.5 sin(2 pi x0) cos(2 pi x1)  (BASELINE.json cfg2)
__device__ __forceinline__ double coeff_sincos(double x0, double x1)
{
    return 1.0 + 0.5 * sinpi(2.0 * x0) * cospi(2.0 * x1);
}

__device__ __forceinline__ double det3(const double* A)
{
    return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
           A[2] * (A[3] * A[7] - A[4] * A[6]);
}

// B = A^{-1}, returns det A
__device__ __forceinline__ double inv3(const double* A, double* B)
{
    const double c00 = A[4] * A[8] - A[5] * A[7];
    const double c01 = A[5] * A[6] - A[3] * A[8];
    const double c02 = A[3] * A[7] - A[4] * A[6];
    const double det = A[0] * c00 + A[1] * c01 + A[2] * c02;
    const double id = 1.0 / det;
    B[0] = c00 * id;
    B[1] = (A[2] * A[7] - A[1] * A[8]) * id;
    B[2] = (A[1] * A[5] - A[2] * A[4]) * id;
    B[3] = c01 * id;
    B[4] = (A[0] * A[8] - A[2] * A[6]) * id;
    B[5] = (A[2] * A[3] - A[0] * A[5]) * id;
    B[6] = c02 * id;
    B[7] = (A[1] * A[6] - A[0] * A[7]) * id;
    B[8] = (A[0] * A[4] - A[1] * A[3]) * id;
    return det;
}

} // namespace dg
