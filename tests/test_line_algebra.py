"""CPU pins of the kernels' 1D line algebra (dg_line_ops: the even/odd code of kernel_gen.cuh compiled
for the host, with the tables dg_setup builds) against an independent numpy construction of the
tables of the method: Gauss-Legendre nodes (numpy leggauss), Lagrange derivative matrix
D[q][j] = l_j'(xi_q) and the 1-point face tables e0, e1, d0, d1 from numpy
polynomial fits of the Lagrange basis — no product or oracle code on the reference side."""
import numpy as np
import pytest
from numpy.polynomial import legendre as npleg
from numpy.polynomial import polynomial as P


def ref_tables(n):
    t, w = npleg.leggauss(n)
    xi, w = 0.5 * (t + 1.0), 0.5 * w
    V = np.vander(xi, n, increasing=True)                # V[q, m] = xi_q^m
    C = np.linalg.solve(V, np.eye(n))                    # column j: monomial coefficients of l_j
    dC = np.array([P.polyder(C[:, j]) for j in range(n)]).T if n > 1 else np.zeros((0, n))
    D = np.array([[P.polyval(xi[q], dC[:, j]) for j in range(n)] for q in range(n)])
    e0 = np.array([P.polyval(0.0, C[:, j]) for j in range(n)])
    e1 = np.array([P.polyval(1.0, C[:, j]) for j in range(n)])
    d0 = np.array([P.polyval(0.0, dC[:, j]) for j in range(n)])
    d1 = np.array([P.polyval(1.0, dC[:, j]) for j in range(n)])
    return xi, w, D, e0, e1, d0, d1


@pytest.mark.parametrize("k", range(1, 8))
def test_line_ops_match_plain_tables(k):
    from paper_1812_08075_b200 import dg
    n = k + 1
    xi, w, D, e0, e1, d0, d1 = ref_tables(n)
    Pn = 10.0 * k * (k + 1)
    B = D.T @ np.diag(w) @ D + 0.5 * (np.outer(e0, d0) + np.outer(d0, e0) - np.outer(e1, d1) - np.outer(d1, e1)) \
        + Pn * (np.outer(e0, e0) + np.outer(e1, e1))
    aL, bL, aR, bR = -0.5 * d0 - Pn * e0, 0.5 * e0, 0.5 * d1 - Pn * e1, -0.5 * e1
    rng = np.random.default_rng(k)
    for _ in range(5):
        x = rng.uniform(-1, 1, n)
        nb = rng.uniform(-1, 1, 4)
        out = dg.dg_line_ops(k, 10.0, x, nb)
        # tolerances: the numpy reference (Vandermonde solve) loses ~cond(V) eps at n = 8; the product
        # tables are built in long double
        scale = np.abs(D).max() * n
        np.testing.assert_allclose(out[:n], D @ x, rtol=0, atol=1e-12 * scale)
        np.testing.assert_allclose(out[n:2 * n], D.T @ x + e0 * nb[0] + d0 * nb[1] + e1 * nb[2] + d1 * nb[3],
                                   rtol=0, atol=1e-12 * scale)
        np.testing.assert_allclose(out[2 * n:3 * n], B @ x + aL * nb[0] + bL * nb[1] + aR * nb[2] + bR * nb[3],
                                   rtol=0, atol=1e-12 * np.abs(B).max() * n)
        np.testing.assert_allclose(out[3 * n:], [e0 @ x, d0 @ x, e1 @ x, d1 @ x], rtol=0, atol=1e-12 * scale)


@pytest.mark.parametrize("k", range(1, 8))
def test_line_ops_exact_on_polynomials(k):
    """D x is the exact derivative of the interpolant for polynomial data of degree <= k; traces are the
    exact end values (closed forms, no table on the reference side)."""
    from paper_1812_08075_b200 import dg
    n = k + 1
    t, _ = npleg.leggauss(n)
    xi = 0.5 * (t + 1.0)
    c = np.random.default_rng(10 + k).uniform(-1, 1, n)   # p(s) = sum c_m s^m, degree k
    x = P.polyval(xi, c)
    out = dg.dg_line_ops(k, 10.0, x, np.zeros(4))
    dc = P.polyder(c)
    np.testing.assert_allclose(out[:n], P.polyval(xi, dc), rtol=0, atol=1e-11)
    np.testing.assert_allclose(out[3 * n:], [P.polyval(0.0, c), P.polyval(0.0, dc), P.polyval(1.0, c),
                                             P.polyval(1.0, dc)], rtol=0, atol=1e-11)
    # the line operator annihilates constants up to the neighbour terms: B^ 1 = P (e0 + e1) (e.1 = 1, d.1 = 0)
    one = dg.dg_line_ops(k, 10.0, np.ones(n), np.zeros(4))[2 * n:3 * n]
    xi_, w, D, e0, e1, d0, d1 = ref_tables(n)
    np.testing.assert_allclose(one, 10.0 * k * (k + 1) * (e0 + e1) + 0.5 * (d0 - d1), rtol=1e-10, atol=1e-10)


@pytest.mark.parametrize("penalty", [10.0, 3.0, 0.0])
def test_axis8_line_operator_matches_plain_tables(penalty):
    """k_axis8's line operator (built from the volume stiffness K = D^T W D and rank-2 trace terms)
    equals the full B^ and neighbour couplings assembled here from the numpy tables."""
    from paper_1812_08075_b200 import dg
    k, n = 7, 8
    xi, w, D, e0, e1, d0, d1 = ref_tables(n)
    Pn = penalty * k * (k + 1)
    B = D.T @ np.diag(w) @ D + 0.5 * (np.outer(e0, d0) + np.outer(d0, e0) - np.outer(e1, d1) - np.outer(d1, e1)) \
        + Pn * (np.outer(e0, e0) + np.outer(e1, e1))
    aL, bL, aR, bR = -0.5 * d0 - Pn * e0, 0.5 * e0, 0.5 * d1 - Pn * e1, -0.5 * e1
    rng = np.random.default_rng(77)
    for _ in range(8):
        x = rng.uniform(-1, 1, n)
        nb = rng.uniform(-1, 1, 4)
        out = dg.dg_line_ops_axis8(penalty, x, nb)
        ref = B @ x + aL * nb[0] + bL * nb[1] + aR * nb[2] + bR * nb[3]
        np.testing.assert_allclose(out[:n], ref, rtol=0, atol=1e-12 * np.abs(B).max() * n)
        scale = np.abs(D).max() * n
        np.testing.assert_allclose(out[n:], [e0 @ x, d0 @ x, e1 @ x, d1 @ x], rtol=0, atol=1e-12 * scale)
