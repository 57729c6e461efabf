// 1D tables for the sum-factorisation kernels, computed in long double on the host once per
// context (dg_setup). See tables.h for the paper passages.
#include "tables.h"

#include <cmath>

namespace dg {

namespace {

// Legendre P_n(t) and P_n'(t) by the Bonnet recurrence, long double.
void legendre(int n, long double t, long double* p, long double* dp)
{
    long double a = 1.0L, b = t; // P_0, P_1
    if (n == 0) { *p = 1.0L; *dp = 0.0L; return; }
    for (int k = 2; k <= n; ++k) {
        long double c = ((2 * k - 1) * t * b - (k - 1) * a) / k;
        a = b;
        b = c;
    }
    *p = b;
    *dp = n * (a - t * b) / (1.0L - t * t);
}

} // namespace

int build_tables(int n, HostTables* T)
{
    if (n < 1 || n > kMaxN) return -1;
    T->n = n;
    const long double pi = 3.141592653589793238462643383279502884L;
    long double x[kMaxN], w[kMaxN];
    // roots of P_n, ascending on [-1,1]; Tricomi initial guess, Newton to convergence
    for (int i = 0; i < n; ++i) {
        long double t = -std::cos(pi * (4.0L * i + 3.0L) / (4.0L * n + 2.0L));
        for (int it = 0; it < 64; ++it) {
            long double p, dp;
            legendre(n, t, &p, &dp);
            long double step = p / dp;
            t -= step;
            if (std::fabs(step) <= 1e-19L) break;
        }
        long double p, dp;
        legendre(n, t, &p, &dp);
        x[i] = 0.5L * (t + 1.0L);
        w[i] = 1.0L / ((1.0L - t * t) * dp * dp); // 2/((1-t^2)P'^2) on [-1,1], halved on [0,1]
    }
    // barycentric weights lambda_j = 1 / prod_{a != j} (x_j - x_a)
    long double lam[kMaxN];
    for (int j = 0; j < n; ++j) {
        long double p = 1.0L;
        for (int a = 0; a < n; ++a)
            if (a != j) p *= (x[j] - x[a]);
        lam[j] = 1.0L / p;
    }
    // collocation derivative matrix: D_qj = (lam_j/lam_q)/(x_q - x_j), D_qq = -sum_{j != q} D_qj
    for (int q = 0; q < n; ++q) {
        long double diag = 0.0L;
        for (int j = 0; j < n; ++j) {
            if (j == q) continue;
            long double v = (lam[j] / lam[q]) / (x[q] - x[j]);
            T->D[q * n + j] = (double)v;
            diag -= v;
        }
        T->D[q * n + q] = (double)diag;
    }
    // values and derivatives at s = 0 and s = 1 (not nodes): l_j(s) = lam_j prod_{a!=j}(s - x_a),
    // l_j'(s) = l_j(s) sum_{a != j} 1/(s - x_a)
    for (int side = 0; side < 2; ++side) {
        const long double s = side;
        for (int j = 0; j < n; ++j) {
            long double v = lam[j], sum = 0.0L;
            for (int a = 0; a < n; ++a)
                if (a != j) { v *= (s - x[a]); sum += 1.0L / (s - x[a]); }
            (side ? T->e1 : T->e0)[j] = (double)v;
            (side ? T->d1 : T->d0)[j] = (double)(v * sum);
        }
    }
    for (int i = 0; i < n; ++i) {
        T->xi[i] = (double)x[i];
        T->w[i] = (double)w[i];
    }
    return 0;
}

namespace {
// D, e0 / e1, d0 / d1 of the Lagrange basis on nodes x[0..n-1] that include both end points (x[0] = 0, x[n-1] = 1)
void endpoint_tables(int n, const long double* x, HostTables* T)
{
    long double lam[kMaxN];
    for (int j = 0; j < n; ++j) {
        long double p = 1.0L;
        for (int a = 0; a < n; ++a)
            if (a != j) p *= (x[j] - x[a]);
        lam[j] = 1.0L / p;
    }
    for (int q = 0; q < n; ++q) {
        long double diag = 0.0L;
        for (int j = 0; j < n; ++j) {
            if (j == q) continue;
            long double v = (lam[j] / lam[q]) / (x[q] - x[j]);
            T->D[q * n + j] = (double)v;
            diag -= v;
        }
        T->D[q * n + q] = (double)diag;
    }
    // the end points are nodes: l_j(0) = delta_j0, l_j(1) = delta_j,n-1, l_j'(0 / 1) = D rows 0 / n-1
    for (int j = 0; j < n; ++j) {
        T->e0[j] = j == 0 ? 1.0 : 0.0;
        T->e1[j] = j == n - 1 ? 1.0 : 0.0;
        T->d0[j] = T->D[0 * n + j];
        T->d1[j] = T->D[(n - 1) * n + j];
        T->xi[j] = (double)x[j];
    }
}
} // namespace

int build_tables_equidistant(int n, HostTables* T)
{
    if (n < 2 || n > kMaxN) return -1;
    T->n = n;
    long double x[kMaxN];
    for (int j = 0; j < n; ++j) x[j] = (long double)j / (n - 1);
    endpoint_tables(n, x, T);
    for (int j = 0; j < n; ++j) T->w[j] = 0.0; // no quadrature on these nodes
    return 0;
}

int build_tables_lobatto(int n, HostTables* T)
{
    if (n < 2 || n > kMaxN) return -1;
    T->n = n;
    const long double pi = 3.141592653589793238462643383279502884L;
    const int m = n - 1; // interior nodes: the roots of P_m'
    long double x[kMaxN], w[kMaxN];
    long double t_all[kMaxN];
    t_all[0] = -1.0L;
    t_all[n - 1] = 1.0L;
    for (int i = 1; i < n - 1; ++i) {
        // ascending; Chebyshev-Gauss-Lobatto initial guess, Newton on P_m' with P_m'' from Legendre's equation
        // (1 - t^2) P_m'' = 2 t P_m' - m (m + 1) P_m
        long double t = -std::cos(pi * i / m);
        for (int it = 0; it < 64; ++it) {
            long double p, dp;
            legendre(m, t, &p, &dp);
            const long double d2p = (2.0L * t * dp - m * (m + 1.0L) * p) / (1.0L - t * t);
            const long double step = dp / d2p;
            t -= step;
            if (std::fabs(step) <= 1e-19L) break;
        }
        t_all[i] = t;
    }
    for (int i = 0; i < n; ++i) {
        long double p, dp;
        legendre(m, t_all[i], &p, &dp);
        x[i] = 0.5L * (t_all[i] + 1.0L);
        w[i] = 1.0L / (n * (n - 1.0L) * p * p); // 2 / (n (n-1) P_{n-1}^2) on [-1,1], halved on [0,1]
    }
    endpoint_tables(n, x, T);
    for (int j = 0; j < n; ++j) T->w[j] = (double)w[j];
    return 0;
}

} // namespace dg
