// Host-side construction of the 1D tables of the method (product path; independent of oracle/).
//   Gauss-Legendre rule on [0,1] with m points         P:L809-812 ("1D quadrature rules with maximum order")
//   Lagrange basis on the n Gauss-Legendre nodes        BASELINE.json cfg0 (reading R8: all configs)
//   D[q][j] = l_j'(xi_q)                                 P:L837 (matrix D^(j))
//   A[q][j] = l_j(xi_q) = delta_qj under collocation     P:L831 (so stage-1 value contractions vanish)
//   e0_j = l_j(0), e1_j = l_j(1), d0_j = l_j'(0), d1_j = l_j'(1)   P:L143-146 (1-point face matrices)
#pragma once

namespace dg {

constexpr int kMaxN = 9; // n <= 8 basis functions; Gauss rules up to m = 9 points (overintegration)

struct HostTables {
    int n;
    double xi[kMaxN], w[kMaxN];
    double D[kMaxN * kMaxN]; // row-major D[q * n + j]
    double e0[kMaxN], e1[kMaxN], d0[kMaxN], d1[kMaxN];
};

// Returns 0 on success, -1 if n is out of range.
int build_tables(int n, HostTables* t);

// The non-Gauss basis of SURVEY §8(f2): Lagrange polynomials on the n Gauss-Lobatto nodes (t = -1, the roots of
// P_{n-1}', +1 mapped to [0,1]); D at those nodes, e0 / e1 the unit vectors of the end nodes, d0 / d1 rows of D.
// Interpolated to Gauss points by fill_qtab: A = [l_j(xi_q)] != I even at m = n. n >= 2.
int build_tables_lobatto(int n, HostTables* t);
// The same for the n equidistant nodes j / (n - 1) (SPEC.md's CPU program's basis).
int build_tables_equidistant(int n, HostTables* t);

} // namespace dg
