/*
 * oracle/oracle.c — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library. The product path (paper_1812_08075_b200/) never links, imports or calls
 * it, and shares no code, header, table or constant generator with it.
 *
 * What it computes: one application r = A x of the symmetric interior penalty DG operator
 * for -div(c grad u) on a periodic hexahedral mesh, i.e. the residual R_I(x) = r(sum_J x_J phi_J,
 * phi_I) of PAPER.md Eq. diffreac_weak with f = 0, no boundary facets (periodic),
 * theta = -1, k(x) = c(x) I, no reaction term, and the penalty of BASELINE.json
 * (gamma = penalty_scale * k (k+1) / h_d, reading R2).
 *
 * How: the PLAIN DEFINITION — tensor-product Gauss quadrature of every volume and face
 * integral with the basis functions evaluated DIRECTLY at every quadrature point
 * as products of 1D Lagrange polynomials (the unfactorised form, Eq. highcomplex),
 * never sum factorisation. Cost O(n^3 m^3) per cell volume.
 *
 * Notation follows PAPER.md §2.1 and §5.2:
 *   n = k+1 basis functions per direction, Lagrange on the n Gauss-Legendre nodes of [0,1]
 *   (BASELINE.json cfg0; reading R8), or on the n Gauss-Lobatto nodes / the n equidistant nodes (the *_b entry
 *   points, basis 1 / 2: the non-Gauss bases of SURVEY §8(f2), A^(i) != I at the Gauss points); m quadrature
 *   points per direction.
 *   Cell T = (i0,i1,i2), canonical id c = (i0 N1 + i1) N2 + i2; local DOF J = j0 + n j1 + n^2 j2
 *   (vec convention, j0 fastest); global DOF g = c n^3 + J (reading R10).
 *   mu_T(xi) = o_T + J_T xi, o_T = (i0/N0, i1/N1, i2/N2) (reading R11).
 *   Interior face F between T- (lower index along d, periodic) and T+ = T- + e_d; n_F points
 *   from T- to T+ (P:L765). [v] = v|T- - v|T+ , {v} = (v|T- + v|T+)/2 (reading R4).
 *   Face geometry (normal, surface element, quadrature points, c_F) from T- (reading R11, R12).
 *
 * Parity pins (tests/test_oracle_pins.py): Gauss rule closed forms + numpy leggauss + monomial
 * exactness; Q1 table closed forms; independent Kronecker-sum SIPG matrix (oracle/brute.py,
 * exact polynomial integration) on tiny meshes; symmetry, A.1 = 0, PSD; linear and quadratic
 * consistency (exact special cases); c(x) reduction u = x2; uniform-shear affine consistency.
 * Gauss-Lobatto basis (tests/test_oracle_lobatto.py): node closed forms + numpy roots of P_{n-1}';
 * the change of basis r^L(x) = T^T r^G(T x), T_ij = l^L_j(xi^G_i) built with numpy, for every geometry
 * and coefficient with m = n and m = n + 1.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OMAX 16 /* max n and m */

static const double PI = 3.14159265358979323846264338327950288;

/* -------------------------------------------------------------------------------------- */
/* 1D Gauss-Legendre rule on [0,1] ("1D quadrature rules with maximum order").  */
/* Newton iteration on the Legendre polynomial P_m(t), t in [-1,1], evaluated with the      */
/* three-term recurrence (k+1) P_{k+1} = (2k+1) t P_k - k P_{k-1}; derivative                */
/* P_m'(t) = m (t P_m - P_{m-1}) / (t^2 - 1). Weights w = 2 / ((1 - t^2) P_m'(t)^2),        */
/* mapped to [0,1]: xi = (1 + t)/2, w01 = w/2.                                              */
/* -------------------------------------------------------------------------------------- */
int oracle_gauss_legendre(int m, double* xi, double* w)
{
    if (m < 1 || m > OMAX) return -1;
    for (int i = 0; i < m; ++i) {
        /* initial guess: Chebyshev-like (roots in descending t order, i-th largest) */
        double t = cos(PI * (i + 0.75) / (m + 0.5));
        double dp = 1.0;
        for (int it = 0; it < 100; ++it) {
            double pm1 = 1.0, pm = t; /* P_0 = 1, P_1 = t */
            for (int k = 1; k < m; ++k) {
                double pn = ((2.0 * k + 1.0) * t * pm - k * pm1) / (k + 1.0);
                pm1 = pm; pm = pn;
            }
            /* now pm = P_m(t), pm1 = P_{m-1}(t) */
            dp = m * (t * pm - pm1) / (t * t - 1.0);
            double dt = pm / dp;
            t -= dt;
            if (fabs(dt) < 1e-17) break;
        }
        /* recompute derivative at the converged root */
        {
            double pm1 = 1.0, pm = t;
            for (int k = 1; k < m; ++k) {
                double pn = ((2.0 * k + 1.0) * t * pm - k * pm1) / (k + 1.0);
                pm1 = pm; pm = pn;
            }
            dp = m * (t * pm - pm1) / (t * t - 1.0);
        }
        /* store ascending on [0,1]: t descending -> index m-1-i */
        xi[m - 1 - i] = 0.5 * (1.0 + t);
        w[m - 1 - i] = 0.5 * 2.0 / ((1.0 - t * t) * dp * dp);
    }
    return 0;
}

/* -------------------------------------------------------------------------------------- */
/* n-point Gauss-Lobatto nodes on [0,1] (the non-Gauss basis of SURVEY §8(f2): Lagrange     */
/* polynomials on these nodes, A = [l_j(xi_q)] != I at the Gauss points):       */
/* t = -1, the n-2 roots of P_{n-1}'(t), +1; Newton on P_{n-1}' with                         */
/* (1 - t^2) P_{n-1}'' = 2 t P_{n-1}' - (n-1) n P_{n-1} (Legendre's equation), P_{n-1} and   */
/* P_{n-1}' from the three-term recurrence and P' = m (t P_m - P_{m-1}) / (t^2 - 1).         */
/* -------------------------------------------------------------------------------------- */
static void legendre_pd(int m, double t, double* p, double* dp)
{
    double pm1 = 1.0, pm = t;
    if (m == 0) { *p = 1.0; *dp = 0.0; return; }
    for (int k = 1; k < m; ++k) {
        double pn = ((2.0 * k + 1.0) * t * pm - k * pm1) / (k + 1.0);
        pm1 = pm; pm = pn;
    }
    *p = pm;
    *dp = m * (t * pm - pm1) / (t * t - 1.0);
}

int oracle_gauss_lobatto(int n, double* xi)
{
    if (n < 2 || n > OMAX) return -1;
    const int m = n - 1; /* interior nodes: roots of P_m' */
    xi[0] = 0.0;
    xi[n - 1] = 1.0;
    for (int i = 1; i < n - 1; ++i) {
        /* initial guess: Chebyshev-Gauss-Lobatto point, descending in t */
        double t = cos(PI * i / m);
        for (int it = 0; it < 100; ++it) {
            double p, dp;
            legendre_pd(m, t, &p, &dp);
            const double d2p = (2.0 * t * dp - m * (m + 1.0) * p) / (1.0 - t * t);
            const double dt = dp / d2p;
            t -= dt;
            if (fabs(dt) < 1e-17) break;
        }
        xi[n - 1 - i] = 0.5 * (1.0 + t);
    }
    return 0;
}

/* Lagrange polynomial l_j on nodes[0..n-1] at s (product formula) and its derivative     */
/* (product rule: l_j'(s) = sum_{a != j} 1/(x_j - x_a) prod_{b != j, a} (s - x_b)/(x_j - x_b)). */
static void lagrange_1d(int n, const double* nodes, int j, double s, double* val, double* der)
{
    double v = 1.0;
    for (int a = 0; a < n; ++a)
        if (a != j) v *= (s - nodes[a]) / (nodes[j] - nodes[a]);
    double d = 0.0;
    for (int a = 0; a < n; ++a) {
        if (a == j) continue;
        double t = 1.0 / (nodes[j] - nodes[a]);
        for (int b = 0; b < n; ++b)
            if (b != j && b != a) t *= (s - nodes[b]) / (nodes[j] - nodes[b]);
        d += t;
    }
    *val = v;
    *der = d;
}

/* Basis nodes: basis 0 the n Gauss-Legendre nodes (reading R8), 1 the n Gauss-Lobatto nodes, 2 the n equidistant
 * nodes j / (n - 1) (SPEC.md's CPU program's choice). */
static int basis_nodes(int basis, int n, double* xi)
{
    double w[OMAX];
    if (basis == 0) return oracle_gauss_legendre(n, xi, w);
    if (basis == 1) return oracle_gauss_lobatto(n, xi);
    if (basis == 2) {
        if (n < 2 || n > OMAX) return -1;
        for (int j = 0; j < n; ++j) xi[j] = (double)j / (n - 1);
        return 0;
    }
    return -1;
}

/* Exported for pins: 1D tables of the basis (n nodes of the given kind) evaluated at arbitrary points. */
int oracle_basis_1d_b(int n, int basis, int npts, const double* pts, double* val, double* der)
{
    double xi[OMAX];
    if (basis_nodes(basis, n, xi)) return -1;
    for (int q = 0; q < npts; ++q)
        for (int j = 0; j < n; ++j)
            lagrange_1d(n, xi, j, pts[q], &val[q * n + j], &der[q * n + j]);
    return 0;
}

/* Exported for pins: 1D tables of the basis (n GL nodes) evaluated at arbitrary points.    */
int oracle_basis_1d(int n, int npts, const double* pts, double* val, double* der)
{
    double xi[OMAX], w[OMAX];
    if (oracle_gauss_legendre(n, xi, w)) return -1;
    for (int q = 0; q < npts; ++q)
        for (int j = 0; j < n; ++j)
            lagrange_1d(n, xi, j, pts[q], &val[q * n + j], &der[q * n + j]);
    return 0;
}

/* ---------------------------------------------------------------- 3x3 helpers (row-major) */
static double det3(const double* A)
{
    return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
           A[2] * (A[3] * A[7] - A[4] * A[6]);
}
static void inv3(const double* A, double* B)
{
    double d = det3(A);
    B[0] = (A[4] * A[8] - A[5] * A[7]) / d;
    B[1] = (A[2] * A[7] - A[1] * A[8]) / d;
    B[2] = (A[1] * A[5] - A[2] * A[4]) / d;
    B[3] = (A[5] * A[6] - A[3] * A[8]) / d;
    B[4] = (A[0] * A[8] - A[2] * A[6]) / d;
    B[5] = (A[2] * A[3] - A[0] * A[5]) / d;
    B[6] = (A[3] * A[7] - A[4] * A[6]) / d;
    B[7] = (A[1] * A[6] - A[0] * A[7]) / d;
    B[8] = (A[0] * A[4] - A[1] * A[3]) / d;
}
/* y = A^T x  (used as grad = J^{-T} grad_hat) */
static void mat_t_vec(const double* A, const double* x, double* y)
{
    for (int a = 0; a < 3; ++a) y[a] = A[0 + a] * x[0] + A[3 + a] * x[1] + A[6 + a] * x[2];
}

/* Coefficient c(x): kind 0 -> 1; kind 1 -> 1 + 0.5 sin(2 pi x0) cos(2 pi x1) (BASELINE.json cfg2). */
static double coeff(int kind, const double* x)
{
    if (kind == 0) return 1.0;
    return 1.0 + 0.5 * sin(2.0 * PI * x[0]) * cos(2.0 * PI * x[1]);
}

/* -------------------------------------------------------------------------------------- */
typedef struct {
    int n, m, k;
    int N[3];
    int coeff_kind;
    double penalty_scale;
    double bnodes[OMAX];           /* basis nodes: n-point GL nodes (basis 0) or GLL nodes (basis 1) */
    double qx[OMAX], qw[OMAX];     /* quadrature rule, m points */
    /* volume tables at all M = m^3 points for all n^3 basis functions: phi, dphi/dxi_0..2 */
    double* vphi;                  /* [M][n^3][4] */
    /* face tables: for d, side (0: xi_d = 0, 1: xi_d = 1), points (a,b) over m^2, [n^3][4] */
    double* fphi[3][2];
} otab;

static int point_index3(int m, int q0, int q1, int q2) { return q0 + m * (q1 + m * q2); }

/* Direct evaluation of phi_J and grad_hat phi_J at a reference point p (product of 1D values). */
static void eval_basis_point(const otab* T, const double p[3], double* out /* [n^3][4] */)
{
    const int n = T->n;
    double v[3][OMAX], d[3][OMAX];
    for (int dim = 0; dim < 3; ++dim)
        for (int j = 0; j < n; ++j) lagrange_1d(n, T->bnodes, j, p[dim], &v[dim][j], &d[dim][j]);
    for (int j2 = 0; j2 < n; ++j2)
        for (int j1 = 0; j1 < n; ++j1)
            for (int j0 = 0; j0 < n; ++j0) {
                int J = j0 + n * (j1 + n * j2);
                out[4 * J + 0] = v[0][j0] * v[1][j1] * v[2][j2];
                out[4 * J + 1] = d[0][j0] * v[1][j1] * v[2][j2];
                out[4 * J + 2] = v[0][j0] * d[1][j1] * v[2][j2];
                out[4 * J + 3] = v[0][j0] * v[1][j1] * d[2][j2];
            }
}

/* Tangential directions of a face with normal d (increasing order). */
static void tangential(int d, int* t1, int* t2)
{
    if (d == 0) { *t1 = 1; *t2 = 2; }
    else if (d == 1) { *t1 = 0; *t2 = 2; }
    else { *t1 = 0; *t2 = 1; }
}

static int otab_init_b(otab* T, int N0, int N1, int N2, int k, int m, int coeff_kind, double penalty_scale, int basis)
{
    memset(T, 0, sizeof(*T));
    T->k = k; T->n = k + 1; T->m = m;
    T->N[0] = N0; T->N[1] = N1; T->N[2] = N2;
    T->coeff_kind = coeff_kind;
    T->penalty_scale = penalty_scale;
    if (T->n > OMAX || m > OMAX || k < 1 || m < 1) return -1;
    if (basis_nodes(basis, T->n, T->bnodes)) return -1;
    if (oracle_gauss_legendre(m, T->qx, T->qw)) return -1;
    const int n3 = T->n * T->n * T->n, M = m * m * m;
    T->vphi = (double*)malloc(sizeof(double) * (size_t)M * n3 * 4);
    if (!T->vphi) return -1;
    for (int q2 = 0; q2 < m; ++q2)
        for (int q1 = 0; q1 < m; ++q1)
            for (int q0 = 0; q0 < m; ++q0) {
                double p[3] = {T->qx[q0], T->qx[q1], T->qx[q2]};
                eval_basis_point(T, p, T->vphi + (size_t)point_index3(m, q0, q1, q2) * n3 * 4);
            }
    for (int d = 0; d < 3; ++d) {
        int t1, t2;
        tangential(d, &t1, &t2);
        for (int side = 0; side < 2; ++side) {
            T->fphi[d][side] = (double*)malloc(sizeof(double) * (size_t)m * m * n3 * 4);
            if (!T->fphi[d][side]) return -1;
            for (int b = 0; b < m; ++b)
                for (int a = 0; a < m; ++a) {
                    double p[3];
                    p[d] = (double)side;
                    p[t1] = T->qx[a];
                    p[t2] = T->qx[b];
                    eval_basis_point(T, p, T->fphi[d][side] + (size_t)(a + m * b) * n3 * 4);
                }
        }
    }
    return 0;
}

static int otab_init(otab* T, int N0, int N1, int N2, int k, int m, int coeff_kind, double penalty_scale)
{
    return otab_init_b(T, N0, N1, N2, k, m, coeff_kind, penalty_scale, 0);
}

static void otab_free(otab* T)
{
    free(T->vphi);
    for (int d = 0; d < 3; ++d)
        for (int s = 0; s < 2; ++s) free(T->fphi[d][s]);
}

/* u and grad_hat u at a point from a DOF block and the point's basis table row. */
static void eval_u(int n3, const double* x, const double* tab, double* u, double gh[3])
{
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int J = 0; J < n3; ++J) {
        s0 += x[J] * tab[4 * J + 0];
        s1 += x[J] * tab[4 * J + 1];
        s2 += x[J] * tab[4 * J + 2];
        s3 += x[J] * tab[4 * J + 3];
    }
    *u = s0; gh[0] = s1; gh[1] = s2; gh[2] = s3;
}

/*
 * Residual rows of ONE cell T = (i0,i1,i2).
 *   xs[0] = x block of T, xs[1+2d] = block of T - e_d, xs[2+2d] = block of T + e_d (periodic)
 *   Js[.] = the matching row-major 3x3 Jacobians J_T of the affine maps mu_T.
 *   r    = n^3 output values (overwritten).
 */
static void cell_residual(const otab* T, int i0, int i1, int i2, const double* const xs[7],
                          const double* const Js[7], double* r)
{
    const int n = T->n, m = T->m, n3 = n * n * n;
    const int ic[3] = {i0, i1, i2};
    for (int I = 0; I < n3; ++I) r[I] = 0.0;

    /* ---------------- volume term (k grad u, grad v)_{0,T}, P:L982 ---------------- */
    {
        const double* J = Js[0];
        double Jinv[9];
        inv3(J, Jinv);
        const double adet = fabs(det3(J));
        double o[3];
        for (int a = 0; a < 3; ++a) o[a] = (double)ic[a] / T->N[a];
        for (int q2 = 0; q2 < m; ++q2)
            for (int q1 = 0; q1 < m; ++q1)
                for (int q0 = 0; q0 < m; ++q0) {
                    const double* tab = T->vphi + (size_t)point_index3(m, q0, q1, q2) * n3 * 4;
                    double u, gh[3], g[3];
                    eval_u(n3, xs[0], tab, &u, gh);
                    mat_t_vec(Jinv, gh, g);                 /* grad u = J^{-T} grad_hat u */
                    const double xi[3] = {T->qx[q0], T->qx[q1], T->qx[q2]};
                    double xp[3];
                    for (int a = 0; a < 3; ++a) xp[a] = o[a] + J[3 * a] * xi[0] + J[3 * a + 1] * xi[1] + J[3 * a + 2] * xi[2];
                    const double W = T->qw[q0] * T->qw[q1] * T->qw[q2] * adet;
                    const double cW = W * coeff(T->coeff_kind, xp);
                    for (int I = 0; I < n3; ++I) {
                        double gp[3];
                        mat_t_vec(Jinv, tab + 4 * I + 1, gp);  /* grad phi_I */
                        r[I] += cW * (g[0] * gp[0] + g[1] * gp[1] + g[2] * gp[2]);
                    }
                }
    }

    /* ---------------- face terms, P:L986-989 with theta = -1 ---------------- */
    for (int d = 0; d < 3; ++d) {
        int t1, t2;
        tangential(d, &t1, &t2);
        const double gamma = T->penalty_scale * T->k * (T->k + 1) * (double)T->N[d]; /* / h_d */
        for (int side = 0; side < 2; ++side) {
            /* side 1: face at xi_d = 1 of T; T is T-, neighbour T + e_d is T+.
               side 0: face at xi_d = 0 of T; T is T+, neighbour T - e_d is T-. */
            const int self_is_minus = (side == 1);
            const int im = self_is_minus ? 0 : 1 + 2 * d;
            const int ip = self_is_minus ? 2 + 2 * d : 0;
            int icm[3] = {ic[0], ic[1], ic[2]};
            if (!self_is_minus) icm[d] = (ic[d] - 1 + T->N[d]) % T->N[d];
            const double* Jm = Js[im];
            const double* Jp = Js[ip];
            double Jminv[9], Jpinv[9];
            inv3(Jm, Jminv);
            inv3(Jp, Jpinv);
            const double adetm = fabs(det3(Jm));
            /* nu = J_-^{-T} e_d (Nanson), n_F = nu/|nu|, dS = |det J_-| |nu| dS_hat */
            double ed[3] = {0, 0, 0}, nu[3];
            ed[d] = 1.0;
            mat_t_vec(Jminv, ed, nu);
            const double nnu = sqrt(nu[0] * nu[0] + nu[1] * nu[1] + nu[2] * nu[2]);
            const double nF[3] = {nu[0] / nnu, nu[1] / nnu, nu[2] / nnu};
            const double sF = adetm * nnu;
            double om[3];
            for (int a = 0; a < 3; ++a) om[a] = (double)icm[a] / T->N[a];
            const double* tabm = T->fphi[d][1]; /* T- evaluated at xi_d = 1 */
            const double* tabp = T->fphi[d][0]; /* T+ evaluated at xi_d = 0 */
            const double* tabself = self_is_minus ? tabm : tabp;
            const double* Jselfinv = self_is_minus ? Jminv : Jpinv;
            for (int b = 0; b < m; ++b)
                for (int a = 0; a < m; ++a) {
                    const size_t off = (size_t)(a + m * b) * n3 * 4;
                    double um, up, ghm[3], ghp[3], gm[3], gp[3];
                    eval_u(n3, xs[im], tabm + off, &um, ghm);
                    eval_u(n3, xs[ip], tabp + off, &up, ghp);
                    mat_t_vec(Jminv, ghm, gm);
                    mat_t_vec(Jpinv, ghp, gp);
                    double xim[3];
                    xim[d] = 1.0; xim[t1] = T->qx[a]; xim[t2] = T->qx[b];
                    double xF[3];
                    for (int c = 0; c < 3; ++c)
                        xF[c] = om[c] + Jm[3 * c] * xim[0] + Jm[3 * c + 1] * xim[1] + Jm[3 * c + 2] * xim[2];
                    const double cF = coeff(T->coeff_kind, xF);
                    const double W = T->qw[a] * T->qw[b] * sF;
                    const double jump = um - up;                                   /* [u] */
                    const double avg = 0.5 * cF * ((gm[0] + gp[0]) * nF[0] + (gm[1] + gp[1]) * nF[1] +
                                                   (gm[2] + gp[2]) * nF[2]);      /* n.{c grad u} */
                    /* test side: [v] = +phi (T-) or -phi (T+); n.{c grad v} = cF/2 grad phi . n */
                    const double sv = self_is_minus ? 1.0 : -1.0;
                    for (int I = 0; I < n3; ++I) {
                        const double phi = tabself[off + 4 * I];
                        double gphi[3];
                        mat_t_vec(Jselfinv, tabself + off + 4 * I + 1, gphi);
                        const double dphin = 0.5 * cF * (gphi[0] * nF[0] + gphi[1] * nF[1] + gphi[2] * nF[2]);
                        /* -(n.{c grad u}, [v]) + theta([u], n.{c grad v}) + gamma([u],[v]), theta = -1 */
                        r[I] += W * (-avg * sv * phi - jump * dphin + gamma * jump * sv * phi);
                    }
                }
        }
    }
}

/*
 * The paper's own problem (Eq. diffreac / diffreac_weak): on the
 * NON-periodic unit cube (0,1)^3 with an axiparallel mesh (h_d = 1/N_d),
 *   -div(K grad u) + c u = f,  u = g on the boundary,
 *   K(x) = x x^T + I, c = 10, f = -6, g = |x|^2 (g is a manufactured solution).
 * Residual R_I(x) = r_h(sum_J x_J phi_J, phi_I) of Eq. diffreac_weak with theta = -1:
 *   volume   (K grad u, grad v) + (c u, v) - (f, v)
 *   interior -(n.{K grad u}, [v]) + theta([u], n.{K grad v}) + gamma_F([u], [v])
 *   boundary the same with [v] = {v} = v|T and n the outer normal, plus
 *            -theta(g, n.(K grad v)) - gamma_F(g, v)
 *   gamma_F = alpha k (k+d-1) |F| / min(|T+|, |T-|) (interior), alpha k (k+d-1) |F| / |T| (boundary),
 *   d = 3; alpha = the `alpha` argument (the paper: 3).
 * Cell-centric like cell_residual; xs[1+2d] / xs[2+2d] may be NULL on boundary faces.
 */
static void Kmat(const double* x, double* K)
{
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) K[3 * a + b] = x[a] * x[b] + (a == b ? 1.0 : 0.0);
}

/*
 * mode 0: the paper's linear problem above.
 * mode 1: its nonlinear variant (reading R26): reaction c u^2 in place of c u, source
 *         f = c |x|^4 - 10 |x|^2 - 6 so that u = |x|^2 stays the exact solution (-div(K grad |x|^2) = -10|x|^2 - 6);
 *         residual R(x) with the volume term (c u^2 - f, v).
 * mode 2: the action of its Jacobian at the linearization point u0:
 *         J(u0) z = d/de R(u0 + e z) at e = 0: volume (K grad z, grad v) + (2 c u0 z, v); the face terms
 *         are those of R with z in place of u and g = 0 (they are affine in u; g does not depend on it).
 *         xs[] hold z; u0s is the cell's block of u0 (the linearization point, evaluated with the same
 *         basis at the same quadrature points).
 */
static void cell_residual_dr(const otab* T, int i0, int i1, int i2, const double* const xs[7], double alpha, double* r,
                             int mode, const double* u0s)
{
    const int n = T->n, m = T->m, n3 = n * n * n;
    const int ic[3] = {i0, i1, i2};
    const double h[3] = {1.0 / T->N[0], 1.0 / T->N[1], 1.0 / T->N[2]};
    const double vol = h[0] * h[1] * h[2];
    const double cr = 10.0, f = -6.0;
    for (int I = 0; I < n3; ++I) r[I] = 0.0;
    /* volume: grad u = J^{-T} grad_hat u = grad_hat u / h componentwise */
    for (int q2 = 0; q2 < m; ++q2)
        for (int q1 = 0; q1 < m; ++q1)
            for (int q0 = 0; q0 < m; ++q0) {
                const double* tab = T->vphi + (size_t)point_index3(m, q0, q1, q2) * n3 * 4;
                double u, gh[3], g[3], K[9], Kg[3];
                eval_u(n3, xs[0], tab, &u, gh);
                for (int a = 0; a < 3; ++a) g[a] = gh[a] / h[a];
                const double xq[3] = {(ic[0] + T->qx[q0]) * h[0], (ic[1] + T->qx[q1]) * h[1], (ic[2] + T->qx[q2]) * h[2]};
                Kmat(xq, K);
                for (int a = 0; a < 3; ++a) Kg[a] = K[3 * a] * g[0] + K[3 * a + 1] * g[1] + K[3 * a + 2] * g[2];
                const double W = T->qw[q0] * T->qw[q1] * T->qw[q2] * vol;
                /* the zeroth-order term q(u) - f, multiplied by v */
                double react;
                if (mode == 0) {
                    react = cr * u - f;
                } else if (mode == 1) {
                    const double s = xq[0] * xq[0] + xq[1] * xq[1] + xq[2] * xq[2];
                    const double fnl = cr * s * s - 10.0 * s - 6.0;
                    react = cr * u * u - fnl;
                } else {
                    double u0, gh0[3];
                    eval_u(n3, u0s, tab, &u0, gh0);
                    react = 2.0 * cr * u0 * u;
                }
                for (int I = 0; I < n3; ++I) {
                    const double* ti = tab + 4 * I;
                    const double gp0 = ti[1] / h[0], gp1 = ti[2] / h[1], gp2 = ti[3] / h[2];
                    r[I] += W * (Kg[0] * gp0 + Kg[1] * gp1 + Kg[2] * gp2 + react * ti[0]);
                }
            }
    /* faces */
    const double kk = (double)T->k * (T->k + 3 - 1);
    for (int d = 0; d < 3; ++d) {
        int t1, t2;
        tangential(d, &t1, &t2);
        const double area = h[t1] * h[t2];
        const double gamma = alpha * kk * area / vol; /* |F| / |T| (all cells have the same volume) */
        for (int side = 0; side < 2; ++side) {
            const int boundary = side ? (ic[d] == T->N[d] - 1) : (ic[d] == 0);
            const double* tabself = T->fphi[d][side];
            for (int b = 0; b < m; ++b)
                for (int a = 0; a < m; ++a) {
                    const size_t off = (size_t)(a + m * b) * n3 * 4;
                    double xi[3];
                    xi[d] = (double)side; xi[t1] = T->qx[a]; xi[t2] = T->qx[b];
                    double xF[3], K[9];
                    for (int c = 0; c < 3; ++c) xF[c] = (ic[c] + xi[c]) * h[c];
                    Kmat(xF, K);
                    const double W = T->qw[a] * T->qw[b] * area;
                    double us, ghs[3], gs[3];
                    eval_u(n3, xs[0], tabself + off, &us, ghs);
                    for (int c = 0; c < 3; ++c) gs[c] = ghs[c] / h[c];
                    if (boundary) {
                        /* outer normal n = +-e_d; [u] = u, {K grad u} = K grad u (one-sided) */
                        const double sn = side ? 1.0 : -1.0;
                        const double Kgn = sn * (K[3 * d] * gs[0] + K[3 * d + 1] * gs[1] + K[3 * d + 2] * gs[2]);
                        const double g = (mode == 2) ? 0.0 : xF[0] * xF[0] + xF[1] * xF[1] + xF[2] * xF[2];
                        for (int I = 0; I < n3; ++I) {
                            const double* ti = tabself + off + 4 * I;
                            const double gp[3] = {ti[1] / h[0], ti[2] / h[1], ti[3] / h[2]};
                            const double Kvn = sn * (K[3 * d] * gp[0] + K[3 * d + 1] * gp[1] + K[3 * d + 2] * gp[2]);
                            /* -(n.K grad u) v + theta u (n.K grad v) + gamma u v - theta g (n.K grad v) - gamma g v */
                            r[I] += W * (-Kgn * ti[0] - (us - g) * Kvn + gamma * (us - g) * ti[0]);
                        }
                    } else {
                        const int self_is_minus = (side == 1);
                        const double* xo = xs[self_is_minus ? 2 + 2 * d : 1 + 2 * d];
                        const double* tabo = T->fphi[d][self_is_minus ? 0 : 1];
                        double uo, gho[3], go[3];
                        eval_u(n3, xo, tabo + off, &uo, gho);
                        for (int c = 0; c < 3; ++c) go[c] = gho[c] / h[c];
                        const double um = self_is_minus ? us : uo, up = self_is_minus ? uo : us;
                        /* n = +e_d (T- -> T+): n.{K grad u} = 1/2 (K (grad u- + grad u+))_d */
                        double gsum[3];
                        for (int c = 0; c < 3; ++c) gsum[c] = (self_is_minus ? gs[c] + go[c] : go[c] + gs[c]);
                        const double avg = 0.5 * (K[3 * d] * gsum[0] + K[3 * d + 1] * gsum[1] + K[3 * d + 2] * gsum[2]);
                        const double jump = um - up;
                        const double sv = self_is_minus ? 1.0 : -1.0;
                        for (int I = 0; I < n3; ++I) {
                            const double* ti = tabself + off + 4 * I;
                            const double gp[3] = {ti[1] / h[0], ti[2] / h[1], ti[3] / h[2]};
                            const double dphin = 0.5 * (K[3 * d] * gp[0] + K[3 * d + 1] * gp[1] + K[3 * d + 2] * gp[2]);
                            r[I] += W * (-avg * sv * ti[0] - jump * dphin + gamma * jump * sv * ti[0]);
                        }
                    }
                }
        }
    }
}

/*
 * The paper's diffusion-reaction residual (cell_residual_dr) on the non-periodic unit cube; x, r global
 * canonical vectors; cells == NULL => all cells. Returns 0 or -1.
 */
static int apply_dr(int N0, int N1, int N2, int k, int m, double alpha, int mode, const double* u0, const double* x,
                    double* r, const int64_t* cells, int64_t ncells)
{
    otab T;
    if (N0 < 1 || N1 < 1 || N2 < 1) return -1;
    if (otab_init(&T, N0, N1, N2, k, m, 0, alpha)) { otab_free(&T); return -1; }
    const int n = k + 1;
    const int64_t n3 = (int64_t)n * n * n;
    const int64_t total = (int64_t)N0 * N1 * N2;
    const int64_t cnt = cells ? ncells : total;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t s = 0; s < cnt; ++s) {
        const int64_t c = cells ? cells[s] : s;
        const int i2 = (int)(c % N2), i1 = (int)((c / N2) % N1), i0 = (int)(c / ((int64_t)N1 * N2));
        const int ic[3] = {i0, i1, i2};
        const double* xs[7];
        xs[0] = x + c * n3;
        for (int d = 0; d < 3; ++d)
            for (int sgn = 0; sgn < 2; ++sgn) {
                int jc[3] = {ic[0], ic[1], ic[2]};
                jc[d] = ic[d] + (sgn ? 1 : -1);
                xs[1 + 2 * d + sgn] = (jc[d] < 0 || jc[d] >= T.N[d]) ? NULL
                                                                     : x + (((int64_t)jc[0] * N1 + jc[1]) * N2 + jc[2]) * n3;
            }
        cell_residual_dr(&T, i0, i1, i2, xs, alpha, r + c * n3, mode, u0 ? u0 + c * n3 : NULL);
    }
    otab_free(&T);
    return 0;
}

int oracle_apply_diffreac(int N0, int N1, int N2, int k, int m, double alpha, const double* x, double* r,
                          const int64_t* cells, int64_t ncells)
{
    return apply_dr(N0, N1, N2, k, m, alpha, 0, NULL, x, r, cells, ncells);
}

/*
 * The nonlinear variant (cell_residual_dr modes 1 and 2): jacobian == 0 -> R(x); jacobian == 1 -> J(u0) x.
 * u0: global canonical vector (jacobian == 1 only, else may be NULL). Returns 0 or -1.
 */
int oracle_apply_nlreac(int N0, int N1, int N2, int k, int m, double alpha, int jacobian, const double* u0,
                        const double* x, double* r, const int64_t* cells, int64_t ncells)
{
    if (jacobian && !u0) return -1;
    return apply_dr(N0, N1, N2, k, m, alpha, jacobian ? 2 : 1, jacobian ? u0 : NULL, x, r, cells, ncells);
}

/* Geometry of a canonical cell: row-major J_T. geom_kind 0: diag(1/N); 1: from jac[9 c ..]. */
static void cell_jac(int geom_kind, const int N[3], const double* jac, int64_t c, double* J)
{
    if (geom_kind == 0) {
        memset(J, 0, 9 * sizeof(double));
        J[0] = 1.0 / N[0]; J[4] = 1.0 / N[1]; J[8] = 1.0 / N[2];
    } else {
        memcpy(J, jac + 9 * c, 9 * sizeof(double));
    }
}

/*
 * Full (or sampled) operator application on a global vector.
 *   x, r: host arrays of N0 N1 N2 n^3 doubles in canonical order (r rows of unlisted cells untouched)
 *   jac : host array of 9 doubles per canonical cell (geom_kind 1), else NULL
 *   cells: list of canonical cell ids to compute (NULL => all cells)
 * Returns 0, or -1 on invalid arguments.
 */
int oracle_apply_b(int N0, int N1, int N2, int k, int m, int geom_kind, const double* jac, int coeff_kind,
                   double penalty_scale, int basis, const double* x, double* r, const int64_t* cells, int64_t ncells)
{
    otab T;
    if (N0 < 1 || N1 < 1 || N2 < 1 || (geom_kind == 1 && !jac)) return -1;
    if (otab_init_b(&T, N0, N1, N2, k, m, coeff_kind, penalty_scale, basis)) { otab_free(&T); return -1; }
    const int n = k + 1;
    const int64_t n3 = (int64_t)n * n * n;
    const int64_t total = (int64_t)N0 * N1 * N2;
    const int64_t cnt = cells ? ncells : total;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t s = 0; s < cnt; ++s) {
        const int64_t c = cells ? cells[s] : s;
        const int i2 = (int)(c % N2), i1 = (int)((c / N2) % N1), i0 = (int)(c / ((int64_t)N1 * N2));
        const int ic[3] = {i0, i1, i2};
        int64_t nb[7];
        nb[0] = c;
        for (int d = 0; d < 3; ++d)
            for (int sgn = 0; sgn < 2; ++sgn) {
                int jc[3] = {ic[0], ic[1], ic[2]};
                jc[d] = (ic[d] + (sgn ? 1 : -1) + T.N[d]) % T.N[d];
                nb[1 + 2 * d + sgn] = ((int64_t)jc[0] * N1 + jc[1]) * N2 + jc[2];
            }
        const double* xs[7];
        double Jbuf[7][9];
        const double* Js[7];
        for (int t = 0; t < 7; ++t) {
            xs[t] = x + nb[t] * n3;
            cell_jac(geom_kind, T.N, jac, nb[t], Jbuf[t]);
            Js[t] = Jbuf[t];
        }
        cell_residual(&T, i0, i1, i2, xs, Js, r + c * n3);
    }
    otab_free(&T);
    return 0;
}

int oracle_apply(int N0, int N1, int N2, int k, int m, int geom_kind, const double* jac, int coeff_kind,
                 double penalty_scale, const double* x, double* r, const int64_t* cells, int64_t ncells)
{
    return oracle_apply_b(N0, N1, N2, k, m, geom_kind, jac, coeff_kind, penalty_scale, 0, x, r, cells, ncells);
}

/*
 * Cell-local form used for sampled verification of meshes too large to hold on the host:
 *   cells[s]       canonical id of target cell s
 *   x7[s][7][n^3]  blocks of the target and its 6 face neighbours (order: self, -e0, +e0, -e1, +e1, -e2, +e2)
 *   j7[s][7][9]    matching Jacobians (ignored for geom_kind 0)
 *   r[s][n^3]      output rows
 */
int oracle_apply_cells_local_b(int N0, int N1, int N2, int k, int m, int geom_kind, int coeff_kind,
                               double penalty_scale, int basis, const int64_t* cells, int64_t ncells, const double* x7,
                               const double* j7, double* r)
{
    otab T;
    if (otab_init_b(&T, N0, N1, N2, k, m, coeff_kind, penalty_scale, basis)) { otab_free(&T); return -1; }
    const int n = k + 1;
    const int64_t n3 = (int64_t)n * n * n;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t s = 0; s < ncells; ++s) {
        const int64_t c = cells[s];
        const int i2 = (int)(c % N2), i1 = (int)((c / N2) % N1), i0 = (int)(c / ((int64_t)N1 * N2));
        const double* xs[7];
        double Jbuf[7][9];
        const double* Js[7];
        for (int t = 0; t < 7; ++t) {
            xs[t] = x7 + (s * 7 + t) * n3;
            if (geom_kind == 0) cell_jac(0, T.N, NULL, 0, Jbuf[t]);
            else memcpy(Jbuf[t], j7 + (s * 7 + t) * 9, 9 * sizeof(double));
            Js[t] = Jbuf[t];
        }
        cell_residual(&T, i0, i1, i2, xs, Js, r + s * n3);
    }
    otab_free(&T);
    return 0;
}

int oracle_apply_cells_local(int N0, int N1, int N2, int k, int m, int geom_kind, int coeff_kind,
                             double penalty_scale, const int64_t* cells, int64_t ncells, const double* x7,
                             const double* j7, double* r)
{
    return oracle_apply_cells_local_b(N0, N1, N2, k, m, geom_kind, coeff_kind, penalty_scale, 0, cells, ncells, x7, j7, r);
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the OpenMP loops (timing only: bench.py's 1-thread oracle time). */
void oracle_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ====================================================================================== */
/* Stokes (Eq. stokes_strong / stokes_weak).                 */
/*   -mu Lap u + grad p = f, div u = 0 on (0,1)^3, u = g on Gamma_D, mu grad u n - p n = 0  */
/*   on Gamma_N; mu = 1, f = 0 (g is the solution: reading R27),                          */
/*   Gamma_D = the boundary without the face x_0 = 1 (the paper's "x_1 < 1" with 1-based   */
/*   coordinates, R27), g = (4 x_1 (1 - x_1), 0, 0), exact pressure 8 (1 - x_0).           */
/* Residual r(u_h, p_h; v_h, q_h) of Eq. stokes_weak, theta = -1, gamma_F as for the       */
/* diffusion-reaction problem (alpha k (k+2) |F| / |T|, alpha = the argument):    */
/*   volume      (grad u, grad v) - (p, div v) - (div u, q)                                 */
/*   F in F_i+D  -({grad u} n, [v]) + theta([u], {grad v} n) + gamma([u], [v])              */
/*               + ({p}, [v] . n) + ([u] . n, {q})                                          */
/*   F in F_D    -theta(g, grad v n) - gamma(g, v) - (g . n, q)                              */
/* Boundary faces: [w] = {w} = w|T, n the outer normal (R21). Velocity Q_k (n = k+1 GL      */
/* nodes per direction), pressure Q_{k-1} (k GL nodes, R27), quadrature with m = k+1 Gauss  */
/* points (R28). DOFs per cell: [u_0 (n^3) | u_1 (n^3) | u_2 (n^3) | p (k^3)], each block in */
/* j0-fastest order, cells canonical (R27). Axiparallel mesh h_d = 1/N_d, non-periodic.     */
/* Plain definition: every basis function evaluated directly (lagrange_1d products) at      */
/* every quadrature point.                                                                   */
/* ====================================================================================== */
typedef struct {
    int k, n, np, m, B;
    double vx[OMAX], px[OMAX], qx[OMAX], qw[OMAX];
} stab;

/* value of the velocity basis function J and its reference gradient at reference point s */
static void st_vbasis(const stab* S, int J, const double s[3], double* v, double g[3])
{
    const int n = S->n;
    const int j[3] = {J % n, (J / n) % n, J / (n * n)};
    double a[3], d[3];
    for (int e = 0; e < 3; ++e) lagrange_1d(n, S->vx, j[e], s[e], &a[e], &d[e]);
    *v = a[0] * a[1] * a[2];
    g[0] = d[0] * a[1] * a[2];
    g[1] = a[0] * d[1] * a[2];
    g[2] = a[0] * a[1] * d[2];
}
static double st_pbasis(const stab* S, int J, const double s[3])
{
    const int np = S->np;
    const int j[3] = {J % np, (J / np) % np, J / (np * np)};
    double v = 1.0;
    for (int e = 0; e < 3; ++e) {
        double a, d;
        lagrange_1d(np, S->px, j[e], s[e], &a, &d);
        v *= a;
    }
    return v;
}
/* u (3 components), reference gradients gu[c][e], p of the block X at reference point s */
static void st_eval(const stab* S, const double* X, const double s[3], double u[3], double gu[3][3], double* p)
{
    const int n3 = S->n * S->n * S->n, p3 = S->np * S->np * S->np;
    for (int c = 0; c < 3; ++c) {
        u[c] = 0.0;
        gu[c][0] = gu[c][1] = gu[c][2] = 0.0;
    }
    for (int J = 0; J < n3; ++J) {
        double v, g[3];
        st_vbasis(S, J, s, &v, g);
        for (int c = 0; c < 3; ++c) {
            const double xc = X[c * n3 + J];
            u[c] += xc * v;
            for (int e = 0; e < 3; ++e) gu[c][e] += xc * g[e];
        }
    }
    *p = 0.0;
    for (int J = 0; J < p3; ++J) *p += X[3 * n3 + J] * st_pbasis(S, J, s);
}

static void cell_residual_stokes(const stab* S, const int N[3], const int ic[3], const double* const xs[7], double alpha,
                                 double* r)
{
    const int n3 = S->n * S->n * S->n, p3 = S->np * S->np * S->np, m = S->m;
    const double h[3] = {1.0 / N[0], 1.0 / N[1], 1.0 / N[2]};
    const double vol = h[0] * h[1] * h[2];
    const double theta = -1.0;
    for (int I = 0; I < S->B; ++I) r[I] = 0.0;
    /* volume */
    for (int q2 = 0; q2 < m; ++q2)
        for (int q1 = 0; q1 < m; ++q1)
            for (int q0 = 0; q0 < m; ++q0) {
                const double s[3] = {S->qx[q0], S->qx[q1], S->qx[q2]};
                const double W = S->qw[q0] * S->qw[q1] * S->qw[q2] * vol;
                double u[3], gu[3][3], p;
                st_eval(S, xs[0], s, u, gu, &p);
                double G[3][3], div = 0.0; /* physical gradients G[c][e] = d u_c / d x_e */
                for (int c = 0; c < 3; ++c)
                    for (int e = 0; e < 3; ++e) G[c][e] = gu[c][e] / h[e];
                for (int c = 0; c < 3; ++c) div += G[c][c];
                for (int J = 0; J < n3; ++J) {
                    double v, g[3];
                    st_vbasis(S, J, s, &v, g);
                    for (int c = 0; c < 3; ++c) {
                        double a = 0.0;
                        for (int e = 0; e < 3; ++e) a += G[c][e] * g[e] / h[e];  /* (grad u_c, grad v) */
                        a -= p * g[c] / h[c];                                       /* -(p, div v) */
                        r[c * n3 + J] += W * a;
                    }
                }
                for (int J = 0; J < p3; ++J) r[3 * n3 + J] += W * (-div * st_pbasis(S, J, s)); /* -(div u, q) */
            }
    /* faces */
    const double kk = (double)S->k * (S->k + 2);
    for (int d = 0; d < 3; ++d) {
        int t1, t2;
        tangential(d, &t1, &t2);
        const double area = h[t1] * h[t2];
        const double gamma = alpha * kk * area / vol;
        for (int side = 0; side < 2; ++side) {
            const int boundary = side ? (ic[d] == N[d] - 1) : (ic[d] == 0);
            if (boundary && d == 0 && side == 1) continue; /* Gamma_N: x_0 = 1, no face terms */
            for (int b = 0; b < m; ++b)
                for (int a = 0; a < m; ++a) {
                    double s[3];
                    s[d] = (double)side; s[t1] = S->qx[a]; s[t2] = S->qx[b];
                    double xF[3];
                    for (int e = 0; e < 3; ++e) xF[e] = (ic[e] + s[e]) * h[e];
                    const double W = S->qw[a] * S->qw[b] * area;
                    double us[3], gus[3][3], ps;
                    st_eval(S, xs[0], s, us, gus, &ps);
                    if (boundary) {
                        const double sn = side ? 1.0 : -1.0;
                        const double g[3] = {4.0 * xF[1] * (1.0 - xF[1]), 0.0, 0.0};
                        double jmp[3];
                        for (int c = 0; c < 3; ++c) jmp[c] = us[c] - g[c];
                        for (int J = 0; J < n3; ++J) {
                            double v, gv[3];
                            st_vbasis(S, J, s, &v, gv);
                            const double dvn = sn * gv[d] / h[d]; /* grad v . n */
                            for (int c = 0; c < 3; ++c) {
                                const double dun = sn * gus[c][d] / h[d];
                                double t = -dun * v + theta * jmp[c] * dvn + gamma * jmp[c] * v;
                                if (c == d) t += ps * v * sn; /* ({p}, [v] . n) */
                                r[c * n3 + J] += W * t;
                            }
                        }
                        for (int J = 0; J < p3; ++J) r[3 * n3 + J] += W * sn * jmp[d] * st_pbasis(S, J, s);
                    } else {
                        const int self_is_minus = (side == 1);
                        const double* xo = xs[self_is_minus ? 2 + 2 * d : 1 + 2 * d];
                        double so[3];
                        so[d] = self_is_minus ? 0.0 : 1.0; so[t1] = s[t1]; so[t2] = s[t2];
                        double uo[3], guo[3][3], po;
                        st_eval(S, xo, so, uo, guo, &po);
                        const double sv = self_is_minus ? 1.0 : -1.0; /* [v] = sv v */
                        double jump[3], avg[3];
                        for (int c = 0; c < 3; ++c) {
                            const double um = self_is_minus ? us[c] : uo[c], up = self_is_minus ? uo[c] : us[c];
                            jump[c] = um - up;
                            avg[c] = 0.5 * (gus[c][d] + guo[c][d]) / h[d]; /* {grad u_c} . n_F, n_F = +e_d */
                        }
                        const double pavg = 0.5 * (ps + po);
                        for (int J = 0; J < n3; ++J) {
                            double v, gv[3];
                            st_vbasis(S, J, s, &v, gv);
                            const double dvn = 0.5 * gv[d] / h[d]; /* {grad v} . n_F (v lives on this side) */
                            for (int c = 0; c < 3; ++c) {
                                double t = -avg[c] * sv * v + theta * jump[c] * dvn + gamma * jump[c] * sv * v;
                                if (c == d) t += pavg * sv * v;
                                r[c * n3 + J] += W * t;
                            }
                        }
                        for (int J = 0; J < p3; ++J) r[3 * n3 + J] += W * jump[d] * 0.5 * st_pbasis(S, J, s);
                    }
                }
        }
    }
}

/*
 * Stokes residual on the whole mesh (or the rows of `cells`): x, r global vectors of N0 N1 N2 (3 n^3 + k^3)
 * doubles in the block layout above. k >= 1 (k = 1: piecewise-constant pressure). Returns 0 or -1.
 */
int oracle_apply_stokes(int N0, int N1, int N2, int k, double alpha, const double* x, double* r, const int64_t* cells,
                        int64_t ncells)
{
    stab S;
    if (N0 < 1 || N1 < 1 || N2 < 1 || k < 1 || k + 1 > OMAX) return -1;
    S.k = k; S.n = k + 1; S.np = k; S.m = k + 1;
    S.B = 3 * S.n * S.n * S.n + S.np * S.np * S.np;
    double w[OMAX];
    if (oracle_gauss_legendre(S.n, S.vx, w) || oracle_gauss_legendre(S.np, S.px, w) ||
        oracle_gauss_legendre(S.m, S.qx, S.qw))
        return -1;
    const int N[3] = {N0, N1, N2};
    const int64_t total = (int64_t)N0 * N1 * N2;
    const int64_t cnt = cells ? ncells : total;
#pragma omp parallel for schedule(dynamic, 2)
    for (int64_t s = 0; s < cnt; ++s) {
        const int64_t c = cells ? cells[s] : s;
        const int ic[3] = {(int)(c / ((int64_t)N1 * N2)), (int)((c / N2) % N1), (int)(c % N2)};
        const double* xs[7];
        xs[0] = x + c * S.B;
        for (int d = 0; d < 3; ++d)
            for (int sgn = 0; sgn < 2; ++sgn) {
                int jc[3] = {ic[0], ic[1], ic[2]};
                jc[d] = ic[d] + (sgn ? 1 : -1);
                xs[1 + 2 * d + sgn] = (jc[d] < 0 || jc[d] >= N[d]) ? NULL
                                                                   : x + (((int64_t)jc[0] * N1 + jc[1]) * N2 + jc[2]) * S.B;
            }
        cell_residual_stokes(&S, N, ic, xs, alpha, r + c * S.B);
    }
    return 0;
}
