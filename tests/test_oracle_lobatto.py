"""Pins of the oracle's non-Gauss bases (Lagrange polynomials on the n Gauss-Lobatto nodes or on the n
equidistant nodes of SPEC.md's CPU program, so the
interpolation matrix A^(i) = [l_j(xi_q)] != I even with m = n Gauss points).

* nodes: closed forms (tests/golden/gauss_lobatto.txt) and, for larger n, numpy's roots of P_{n-1}';
* basis tables: Kronecker delta at the nodes, partition of unity, exact derivatives of polynomials of degree <= k;
* the whole operator: with the same m-point Gauss rule, the Gauss-Lobatto and the Gauss-Legendre bases span the same
  Q_k space, so the residuals are related by the change of basis exactly: u = sum_j x_j phi^L_j =
  sum_i (T x)_i phi^G_i with T_ij = l^L_j(xi^G_i) (per direction, Kronecker product in the vec order), and
  r^L_J = r_h(u, phi^L_J) = sum_I T_IJ r_h(u, phi^G_I) = (T^T r^G(T x))_J for every geometry and coefficient. T is
  built here with numpy from the golden / numpy nodes (not with the oracle's Lagrange routine); the Gauss-basis
  oracle on the right-hand side is pinned by tests/test_oracle_pins.py.
"""
import os

import numpy as np
import pytest

import oracle
import synth

HERE = os.path.dirname(os.path.abspath(__file__))


def golden_nodes():
    out = {}
    for line in open(os.path.join(HERE, "golden", "gauss_lobatto.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = line.split()
        out[int(v[0])] = np.array([float(t) for t in v[1:]])
    return out


def numpy_lobatto(n):
    """Gauss-Lobatto nodes on [0,1] from numpy: the roots of P_{n-1}' with the end points."""
    if n == 2:
        return np.array([0.0, 1.0])
    r = np.sort(np.polynomial.legendre.Legendre.basis(n - 1).deriv().roots().real)
    return np.concatenate([[0.0], 0.5 * (1.0 + r), [1.0]])


def test_lobatto_nodes_closed_forms():
    for n, ref in golden_nodes().items():
        np.testing.assert_allclose(oracle.gauss_lobatto(n), ref, rtol=0, atol=2e-16)


@pytest.mark.parametrize("n", range(2, 10))
def test_lobatto_nodes_numpy(n):
    np.testing.assert_allclose(oracle.gauss_lobatto(n), numpy_lobatto(n), rtol=0, atol=1e-14)


@pytest.mark.parametrize("n", range(2, 9))
def test_lobatto_basis_tables(n):
    nodes = numpy_lobatto(n)
    val, der = oracle.basis_1d(n, nodes, basis=1)
    np.testing.assert_allclose(val, np.eye(n), atol=1e-13)
    pts = np.linspace(-0.1, 1.1, 17)
    val, der = oracle.basis_1d(n, pts, basis=1)
    np.testing.assert_allclose(val.sum(axis=1), 1.0, atol=1e-12)
    np.testing.assert_allclose(der.sum(axis=1), 0.0, atol=1e-10)
    for p in range(n):  # derivative of x^p (degree <= n - 1) reproduced exactly from its nodal values
        np.testing.assert_allclose(der @ nodes ** p, p * pts ** max(p - 1, 0) if p else 0.0 * pts, atol=1e-10)


def lagrange_at(nodes, pts):
    """[len(pts), n] values of the Lagrange polynomials on `nodes` (numpy product formula)."""
    n = len(nodes)
    out = np.ones((len(pts), n))
    for j in range(n):
        for a in range(n):
            if a != j:
                out[:, j] *= (pts - nodes[a]) / (nodes[j] - nodes[a])
    return out


def kron3(T):
    """The per-direction matrix T applied along all three directions of a cell block (vec order, j0 fastest)."""
    return np.kron(T, np.kron(T, T))


def basis_nodes_np(basis, n):
    return numpy_lobatto(n) if basis == 1 else np.linspace(0.0, 1.0, n)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("geom,coeff", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("mq", [0, 1])
@pytest.mark.parametrize("basis", [1, 2])
def test_change_of_basis(k, geom, coeff, mq, basis):
    n = k + 1
    N = (3, 2, 3)
    wl = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=70 + k, quad=n + mq, basis=basis)
    wg = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=70 + k, quad=n + mq, basis=0)
    gx, _ = np.polynomial.legendre.leggauss(n)
    T = lagrange_at(basis_nodes_np(basis, n), 0.5 * (gx + 1.0))  # T[i, j] = l^L_j(xi^G_i)
    T3 = kron3(T)
    # kron(T, kron(T, T)) acts on the index j2 n^2 + j1 n + j0 with the FIRST factor on j2: the vec order of a block
    jac = synth.jac_cells_np(wl, np.arange(wl.ncells)) if geom else None
    x = synth.x_np(wl)
    rl = oracle.apply(wl, x, jac)
    xg = (x.reshape(-1, n ** 3) @ T3.T).reshape(-1)
    rg = oracle.apply(wg, xg, jac)
    rl_ref = (rg.reshape(-1, n ** 3) @ T3).reshape(-1)
    err = np.abs(rl - rl_ref).max() / np.abs(rl_ref).max()
    assert err <= 1e-12, err


def test_lobatto_differs_from_gauss_basis():
    """The two bases are different coordinates: the same coefficient vector gives different residuals (the change of
    basis above is not the identity)."""
    wl = synth.small(3, (2, 2, 2), seed=5, basis=1)
    wg = synth.small(3, (2, 2, 2), seed=5, basis=0)
    x = synth.x_np(wl)
    assert np.abs(oracle.apply(wl, x) - oracle.apply(wg, x)).max() > 1e-3
