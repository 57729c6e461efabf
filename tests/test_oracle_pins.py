"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage / closed form it checks. A plausible mistake in the oracle —
a dropped face term, a sign of the jump, a transposed J^{-T}, a wrong index direction,
a wrong penalty — fails at least one of them (see DESIGN.md §3 'Pins').
"""
import os
from math import sqrt  # noqa: F401  (used by golden-file expressions)

import numpy as np
import pytest

import oracle
import synth
from oracle import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append([s.strip() for s in line.split(";")])
    return rows


def _gl01(n):
    return brute.gl01(n)


def _dense_oracle(w, jac=None):
    n = w.ndofs
    A = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        A[:, j] = oracle.apply(w, e, jac)
    return A


def _interp(w, u, jac=None, virtual=None):
    """DOF vector interpolating u at the mapped GL nodes of every cell.
    virtual=None: x_T(xi) = o_T + J_T xi (the oracle's map).
    virtual=J:    positions J (i + xi) of a conforming sheared lattice (uniform-shear pin)."""
    n = w.n
    xi, _ = _gl01(n)
    N0, N1, N2 = w.N
    c = np.arange(w.ncells)
    i2, i1, i0 = c % N2, (c // N2) % N1, c // (N1 * N2)
    j = np.arange(n ** 3)
    j0, j1, j2 = j % n, (j // n) % n, j // (n * n)
    ref = np.stack([xi[j0], xi[j1], xi[j2]], axis=-1)            # [n^3, 3]
    if virtual is not None:
        lat = np.stack([i0, i1, i2], axis=-1).astype(float)       # [C, 3]
        P = (lat[:, None, :] + ref[None, :, :]) @ virtual.T       # J (i + xi)
    else:
        o = np.stack([i0 / N0, i1 / N1, i2 / N2], axis=-1)
        if jac is None:
            J = np.tile(np.diag([1.0 / N0, 1.0 / N1, 1.0 / N2]).reshape(1, 9), (w.ncells, 1))
        else:
            J = jac
        J = J.reshape(-1, 3, 3)
        P = o[:, None, :] + np.einsum("cab,jb->cja", J, ref)
    return u(P[..., 0], P[..., 1], P[..., 2]).reshape(-1)


def _interior_mask(w, dirs):
    N0, N1, N2 = w.N
    c = np.arange(w.ncells)
    ic = [c // (N1 * N2), (c // N2) % N1, c % N2]
    m = np.ones(w.ncells, bool)
    for d in dirs:
        m &= (ic[d] >= 1) & (ic[d] <= w.N[d] - 2)
    return np.repeat(m, w.n ** 3)


# ------------------------------------------------------------------ 1D rule and tables
def test_gauss_legendre_golden():
    """S:L60-61 closed forms (+ the m=3 roots of P_3)."""
    for m, pts, wts in _read_golden("gauss_legendre.txt"):
        xi, w = oracle.gauss_legendre(int(m))
        np.testing.assert_allclose(xi, eval(pts), rtol=0, atol=1e-15)
        np.testing.assert_allclose(w, eval(wts), rtol=0, atol=1e-15)


@pytest.mark.parametrize("m", range(1, 13))
def test_gauss_legendre_library_and_exactness(m):
    """numpy leggauss (library routine) and exactness for x^p, p <= 2m-1."""
    xi, w = oracle.gauss_legendre(m)
    t, wl = np.polynomial.legendre.leggauss(m)
    np.testing.assert_allclose(xi, 0.5 * (t + 1), rtol=0, atol=2e-15)
    np.testing.assert_allclose(w, 0.5 * wl, rtol=0, atol=2e-15)
    assert abs(w.sum() - 1.0) < 1e-14
    assert np.all(np.diff(xi) > 0) and xi[0] > 0 and xi[-1] < 1
    for p in range(2 * m):
        assert abs(np.dot(w, xi ** p) - 1.0 / (p + 1)) < 1e-14
    # not exact one degree higher (the rule really has order 2m-1)
    if m <= 7:
        assert abs(np.dot(w, xi ** (2 * m)) - 1.0 / (2 * m + 1)) > 1e-12


def test_q1_tables_golden():
    """Q1 on GL nodes: A = I, D = sqrt3[[-1,1],[-1,1]], e0/e1/d0/d1 closed forms."""
    xi, _ = oracle.gauss_legendre(2)
    val, der = oracle.basis_1d(2, xi)
    v01, d01 = oracle.basis_1d(2, np.array([0.0, 1.0]))
    got = {"A": val.ravel(), "D": der.ravel(), "e0": v01[0], "e1": v01[1], "d0": d01[0], "d1": d01[1]}
    for name, expr in _read_golden("q1_tables.txt"):
        np.testing.assert_allclose(got[name], eval(expr), rtol=0, atol=1e-14)


@pytest.mark.parametrize("n", range(2, 9))
def test_basis_tables(n):
    """A = I bitwise under collocation; D p(xi) = p'(xi) for deg p <= k; partition of unity."""
    xi, _ = oracle.gauss_legendre(n)
    val, der = oracle.basis_1d(n, xi)
    assert np.array_equal(val, np.eye(n))
    for p in range(n):
        np.testing.assert_allclose(der @ xi ** p, p * xi ** max(p - 1, 0) if p else 0 * xi, atol=1e-11)
    np.testing.assert_allclose(der.sum(1), 0, atol=1e-11)
    v01, d01 = oracle.basis_1d(n, np.array([0.0, 1.0]))
    np.testing.assert_allclose(v01.sum(1), 1, atol=1e-13)
    # boundary vectors reproduce polynomials and their derivatives at 0 and 1
    for p in range(n):
        np.testing.assert_allclose(v01 @ xi ** p, [0.0 ** p, 1.0], atol=1e-12)
        np.testing.assert_allclose(d01 @ xi ** p, [p * 0.0 ** max(p - 1, 0) if p else 0, p], atol=1e-10)


# ------------------------------------------------------------------ whole operator
@pytest.mark.parametrize("k,N", [(1, (1, 1, 1)), (1, (2, 2, 2)), (2, (3, 2, 1)), (1, (3, 4, 2)),
                                 (3, (2, 2, 2)), (2, (2, 3, 2))])
def test_oracle_equals_kronecker_sum(k, N):
    """Axis-aligned c=1: oracle matrix == independent Kronecker-sum SIPG matrix (oracle/brute.py)."""
    w = synth.small(k, N)
    A = brute.dense(w)
    B = _dense_oracle(w)
    assert np.abs(A - B).max() <= 1e-12 * np.abs(A).max()


@pytest.mark.parametrize("k,N", [(1, 8), (3, 6), (4, 3)])
def test_oracle_equals_kronecker_apply(k, N):
    w = synth.small(k, N, seed=3)
    x = synth.x_np(w)
    r1 = oracle.apply(w, x)
    r2 = brute.apply(w, x)
    assert np.abs(r1 - r2).max() <= 1e-12 * np.abs(r2).max()


def test_penalty_scale_enters_linearly():
    """gamma = penalty_scale k(k+1)/h: A(s) - A(0) is linear in s (pins the penalty term alone)."""
    import dataclasses
    w = synth.small(2, (2, 2, 2))
    A0 = _dense_oracle(dataclasses.replace(w, penalty_scale=0.0))
    A1 = _dense_oracle(dataclasses.replace(w, penalty_scale=1.0))
    A10 = _dense_oracle(w)
    np.testing.assert_allclose(A10 - A0, 10.0 * (A1 - A0), atol=1e-10 * np.abs(A10).max())
    assert np.abs(A1 - A0).max() > 0


@pytest.mark.parametrize("geom,coeff,k,N", [(0, 0, 2, 3), (1, 0, 2, 3), (0, 1, 2, 3), (1, 1, 1, (3, 2, 3)),
                                            (1, 1, 3, 2)])
def test_symmetry_nullspace_psd(geom, coeff, k, N):
    """SIPG (theta=-1) is symmetric; A.1 = 0 on the periodic mesh; PSD with a 1-dim null space
    (BASELINE.json north_star checks)."""
    w = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=11)
    jac = synth.jac_cells_np(w, np.arange(w.ncells)) if geom else None
    A = _dense_oracle(w, jac)
    s = np.abs(A).max()
    assert np.abs(A - A.T).max() <= 1e-12 * s
    assert np.abs(A @ np.ones(w.ndofs)).max() <= 1e-12 * s
    ev = np.linalg.eigvalsh(0.5 * (A + A.T))
    assert ev[0] > -1e-10 * s
    assert ev[1] > 1e-8 * s  # exactly one zero eigenvalue (constants)


@pytest.mark.parametrize("k,N", [(1, 6), (2, 5), (3, 4)])
def test_linear_consistency(k, N):
    """SIPG consistency: a(u_I, v) = int -Lap u v = 0 for u = a.x on cells away from the periodic wrap.
    Detects the sign/orientation of the jump (reading R4)."""
    w = synth.small(k, N)
    for a in ([1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0], [0.3, -0.7, 1.1]):
        x = _interp(w, lambda X, Y, Z: a[0] * X + a[1] * Y + a[2] * Z)
        r = oracle.apply(w, x)
        dirs = [d for d in range(3) if a[d] != 0]
        m = _interior_mask(w, dirs)
        assert np.abs(r[m]).max() < 1e-11, (a, np.abs(r[m]).max())
        assert np.abs(r[~m]).max() > 1e-3   # the wrap faces do see the non-periodic field


@pytest.mark.parametrize("k,N", [(2, 5), (3, 4), (4, 4)])
def test_quadratic_consistency(k, N):
    """u = (x0 - 1/2)^2 -> r_{T,J} = -2 h^3 w_J; u = |x - 1/2|^2 -> -6 h^3 w_J (exact GL mass)."""
    w = synth.small(k, N)
    h = 1.0 / N
    _, wq = _gl01(w.n)
    n = w.n
    j = np.arange(n ** 3)
    wJ = wq[j % n] * wq[(j // n) % n] * wq[j // (n * n)]
    wJ = np.tile(wJ, w.ncells)
    x = _interp(w, lambda X, Y, Z: (X - 0.5) ** 2)
    r = oracle.apply(w, x)
    m = _interior_mask(w, [0])
    np.testing.assert_allclose(r[m], -2 * h ** 3 * wJ[m], atol=1e-11)
    x = _interp(w, lambda X, Y, Z: (X - 0.5) ** 2 + (Y - 0.5) ** 2 + (Z - 0.5) ** 2)
    r = oracle.apply(w, x)
    m = _interior_mask(w, [0, 1, 2])
    np.testing.assert_allclose(r[m], -6 * h ** 3 * wJ[m], atol=1e-11)


@pytest.mark.parametrize("k,N", [(2, 5), (3, 4)])
def test_coefficient_reduction(k, N):
    """c(x) = 1 + 0.5 sin(2 pi x0) cos(2 pi x1) does not depend on x2: u = x2 gives r = 0 away from
    the x2 wrap (volume and x2-face points share (x0,x1)); u = x0 does not (c varies along x0)."""
    w = synth.small(k, N, coeff_kind=1)
    x = _interp(w, lambda X, Y, Z: Z)
    r = oracle.apply(w, x)
    m = _interior_mask(w, [2])
    assert np.abs(r[m]).max() < 1e-11
    x = _interp(w, lambda X, Y, Z: X)
    r = oracle.apply(w, x)
    m = _interior_mask(w, [0])
    assert np.abs(r[m]).max() > 1e-4
    # with c = 1 the same mesh gives the Poisson operator exactly
    w1 = synth.small(k, N, coeff_kind=0)
    xr = synth.x_np(w1)
    r_c1 = oracle.apply(w1, xr)
    np.testing.assert_allclose(r_c1, brute.apply(w1, xr), atol=1e-12 * np.abs(r_c1).max())


def test_coefficient_value_at_points():
    """The c(x) path integrates c exactly as defined: for u = x0 on a single interior column the
    volume residual of the x0-derivative test functions equals the GL quadrature of c(x) * dphi/dx0,
    computed here independently (one cell row, k = 1, numpy)."""
    k, N = 1, 4
    w = synth.small(k, N, coeff_kind=1)
    x = _interp(w, lambda X, Y, Z: X)
    r = oracle.apply(w, x).reshape(w.ncells, -1)
    # independent expectation: r_{T,I} = sum_q W_q c(x_q) dphi_I/dx0 (q)  (face terms vanish:
    # [u] = 0 everywhere off the wrap, and -{c du/dn}[v] on x0-faces is -c_F [v]; x1/x2 faces: du/dn = 0)
    xi, wq = _gl01(2)
    n = 2
    L = brute.lagrange_polys(n)
    dL = [p.deriv() for p in L]
    h = 1.0 / N
    c_of = lambda P: 1 + 0.5 * np.sin(2 * np.pi * P[0]) * np.cos(2 * np.pi * P[1])
    cell = synth.cell_id(w, 1, 2, 1)
    i0, i1, i2 = 1, 2, 1
    exp = np.zeros(n ** 3)
    for J in range(n ** 3):
        j0, j1, j2 = J % n, (J // n) % n, J // (n * n)
        s = 0.0
        for q0 in range(n):
            for q1 in range(n):
                for q2 in range(n):
                    P = (h * (i0 + xi[q0]), h * (i1 + xi[q1]), h * (i2 + xi[q2]))
                    Wq = wq[q0] * wq[q1] * wq[q2] * h ** 3
                    dphi0 = dL[j0](xi[q0]) / h * L[j1](xi[q1]) * L[j2](xi[q2])
                    s += Wq * c_of(P) * 1.0 * dphi0
        # x0 faces: lower face (T is T+): -(n.{c grad u})[v] = -(c_F)(-phi) ; upper face: -(c_F)(phi)
        for side, xi0, sgn in ((0, 0.0, -1.0), (1, 1.0, 1.0)):
            for q1 in range(n):
                for q2 in range(n):
                    P = (h * (i0 + xi0), h * (i1 + xi[q1]), h * (i2 + xi[q2]))
                    W = wq[q1] * wq[q2] * h * h
                    phi = L[j0](xi0) * L[j1](xi[q1]) * L[j2](xi[q2])
                    s += -W * c_of(P) * sgn * phi
        exp[J] = s
    np.testing.assert_allclose(r[cell], exp, atol=1e-13)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_uniform_shear_affine(k):
    """Every cell has the same non-symmetric J (conforming sheared lattice P = J (i + xi)), c = 1:
    u = a.P gives r = 0 on interior cells; u = |P|^2 gives r = -6 |det J| w_J (exact quadrature).
    Pins the affine path: J^{-T} gradients, Nanson normal/surface element, |det J| weights."""
    N = 5 if k < 3 else 4
    w = synth.small(k, N, geom_kind=1)
    h = 1.0 / N
    E = np.array([[0.08, -0.05, 0.03], [0.02, -0.09, 0.06], [-0.07, 0.04, 0.1]])
    J = h * (np.eye(3) + E)
    jac = np.tile(J.reshape(1, 9), (w.ncells, 1))
    m = _interior_mask(w, [0, 1, 2])
    x = _interp(w, lambda X, Y, Z: 0.4 * X - 1.3 * Y + 0.9 * Z, virtual=J)
    r = oracle.apply(w, x, jac)
    assert np.abs(r[m]).max() < 1e-11
    if k >= 2:
        x = _interp(w, lambda X, Y, Z: X ** 2 + Y ** 2 + Z ** 2, virtual=J)
        r = oracle.apply(w, x, jac)
        _, wq = _gl01(w.n)
        n = w.n
        j = np.arange(n ** 3)
        wJ = np.tile(wq[j % n] * wq[(j // n) % n] * wq[j // (n * n)], w.ncells)
        np.testing.assert_allclose(r[m], -6 * abs(np.linalg.det(J)) * wJ[m], atol=1e-11)


def test_cells_local_matches_full():
    """The cell-local entry (sampled verification) equals the full apply on the same cells."""
    w = synth.small(2, (3, 4, 3), geom_kind=1, coeff_kind=1, seed=5)
    jac = synth.jac_cells_np(w, np.arange(w.ncells))
    x = synth.x_np(w)
    r = oracle.apply(w, x, jac)
    cells = np.array([0, 5, 17, w.ncells - 1])
    rl = oracle.apply_sampled(w, cells, lambda ids: synth.x_cells_np(w, ids), lambda ids: synth.jac_cells_np(w, ids))
    np.testing.assert_array_equal(rl, r.reshape(w.ncells, -1)[cells])
    # the listed-cells mode of oracle_apply too
    rs = oracle.apply(w, x, jac, cells=cells)
    np.testing.assert_array_equal(rs.reshape(w.ncells, -1)[cells], rl)


@pytest.mark.parametrize("k,N,geom", [(1, (3, 2, 4), 0), (2, (2, 3, 3), 1), (3, (2, 2, 3), 1), (4, (2, 2, 2), 0)])
def test_overintegration_exact_for_polynomial_integrands(k, N, geom):
    """General quadrature m > k+1 (SURVEY §8(f2), P:L811 'quadrature with m points'): with c = 1 every
    volume and face integrand is a polynomial of degree <= 2k per direction (affine: constant metric), so
    the k+1- and k+2/k+3-point Gauss rules give the same operator to rounding — pins the oracle's
    general-m path (interpolation A != I at the quadrature points) against the pinned m = k+1 path."""
    w1 = synth.small(k, N, geom_kind=geom, coeff_kind=0, seed=9)
    jac = synth.jac_cells_np(w1, np.arange(w1.ncells)) if geom else None
    x = synth.x_np(w1)
    r1 = oracle.apply(w1, x, jac)
    for q in (k + 2, k + 3):
        wq = synth.small(k, N, geom_kind=geom, coeff_kind=0, seed=9, quad=q)
        rq = oracle.apply(wq, x, jac)
        assert np.abs(rq - r1).max() <= 1e-12 * np.abs(r1).max()


def test_overintegration_changes_nonpolynomial_coefficient():
    """With c(x) = 1 + 0.5 sin cos the integrand is not polynomial: k+2 points give a different (more
    accurate) operator, converging as m grows (the difference m = k+2 vs k+5 is below that of k+1 vs k+5)."""
    k, N = 2, (3, 3, 2)
    ws = [synth.small(k, N, geom_kind=1, coeff_kind=1, seed=4, quad=q) for q in (k + 1, k + 2, k + 5)]
    jac = synth.jac_cells_np(ws[0], np.arange(ws[0].ncells))
    x = synth.x_np(ws[0])
    r = [oracle.apply(w, x, jac) for w in ws]
    e1 = np.abs(r[0] - r[2]).max()
    e2 = np.abs(r[1] - r[2]).max()
    assert e1 > 1e-6 * np.abs(r[2]).max()
    assert e2 < e1


# ------------------------------------------------------------------ the paper's diffusion-reaction problem
def _interp_fn(w, fn):
    """DOF vector interpolating fn(x0, x1, x2) at the GL nodes of every cell of the unit-cube mesh."""
    n = w.n
    xi, _ = _gl01(n)
    N0, N1, N2 = w.N
    c = np.arange(w.ncells)
    i2, i1, i0 = c % N2, (c // N2) % N1, c // (N1 * N2)
    j = np.arange(n ** 3)
    j0, j1, j2 = j % n, (j // n) % n, j // (n * n)
    X0 = (i0[:, None] + xi[j0][None, :]) / N0
    X1 = (i1[:, None] + xi[j1][None, :]) / N1
    X2 = (i2[:, None] + xi[j2][None, :]) / N2
    return fn(X0, X1, X2).reshape(-1)


@pytest.mark.parametrize("k,N", [(2, (2, 3, 2)), (3, (2, 2, 3)), (4, (2, 2, 2))])
def test_diffreac_manufactured_solution(k, N):
    """g = |x|^2 solves -div((xx^T + I) grad u) + 10 u = -6 with u = g on the boundary, and it
    lies in Q_k for k >= 2; SIPG is consistent, so with quadrature exact for every term (m = k+2, SURVEY
    §8(f1)) the residual of its interpolant vanishes on every cell (boundary cells included)."""
    w = synth.diffreac(k, N, quad=k + 2)
    x = _interp_fn(w, lambda a, b, c: a * a + b * b + c * c)
    r = oracle.apply_diffreac(w, x)
    r0 = oracle.apply_diffreac(w, np.zeros_like(x))
    assert np.abs(r).max() <= 1e-11 * np.abs(r0).max()


def test_diffreac_detects_a_wrong_solution():
    """The same residual is far from zero for a perturbed solution (the pin above is not vacuous)."""
    k, N = 2, (2, 2, 2)
    w = synth.diffreac(k, N, quad=k + 2)
    x = _interp_fn(w, lambda a, b, c: a * a + b * b + c * c + 0.01 * a * b)
    r0 = oracle.apply_diffreac(w, np.zeros_like(x))
    assert np.abs(oracle.apply_diffreac(w, x)).max() > 1e-4 * np.abs(r0).max()


@pytest.mark.parametrize("k,N", [(1, (3, 2, 2)), (2, (2, 3, 2))])
def test_diffreac_bilinear_part_symmetric_positive(k, N):
    """a(u, v) = R(u) - R(0) is the SIPG bilinear form (theta = -1) plus the reaction mass: symmetric and
    positive definite with Dirichlet boundary faces (no null space, unlike the periodic operator)."""
    w = synth.diffreac(k, N, quad=k + 2)
    nd = w.ndofs
    r0 = oracle.apply_diffreac(w, np.zeros(nd))
    A = np.zeros((nd, nd))
    for j in range(nd):
        e = np.zeros(nd)
        e[j] = 1.0
        A[:, j] = oracle.apply_diffreac(w, e) - r0
    assert np.abs(A - A.T).max() <= 1e-12 * np.abs(A).max()
    assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > 0


def test_diffreac_rhs_terms():
    """R(0) = -(f, v) + boundary terms in g only: with alpha -> 2 alpha the penalty parts of R(0) and of a
    double (the g-penalty term -gamma (g, v) and gamma(u, v) are linear in alpha)."""
    k, N = 2, (2, 2, 2)
    w1 = synth.diffreac(k, N, quad=k + 2, alpha=3.0)
    w2 = synth.diffreac(k, N, quad=k + 2, alpha=6.0)
    w0 = synth.diffreac(k, N, quad=k + 2, alpha=0.0)
    z = np.zeros(w1.ndofs)
    p1 = oracle.apply_diffreac(w1, z) - oracle.apply_diffreac(w0, z)
    p2 = oracle.apply_diffreac(w2, z) - oracle.apply_diffreac(w0, z)
    assert np.abs(p2 - 2 * p1).max() <= 1e-12 * np.abs(p2).max()


# ---------------------------------------------------------------- the nonlinear variant
@pytest.mark.parametrize("k,N", [(2, (2, 3, 2)), (3, (2, 2, 3))])
def test_nlreac_manufactured_solution(k, N):
    """Reading R26: -div(K grad u) + c u^2 = f with f = c|x|^4 - 10|x|^2 - 6 is solved by u = |x|^2 = g
    (-div((xx^T + I) 2x) = -10|x|^2 - 6); every term is a polynomial the k+2 point rule integrates exactly
    (u^2 v: degree 4 + k <= 2k + 3 per direction), so the residual of the interpolant vanishes."""
    w = synth.nlreac(k, N)
    x = _interp_fn(w, lambda a, b, c: a * a + b * b + c * c)
    r = oracle.apply_nlreac(w, x)
    r0 = oracle.apply_nlreac(w, np.zeros_like(x))
    assert np.abs(r).max() <= 1e-11 * np.abs(r0).max()
    # not vacuous: a perturbed function has a residual far from zero
    y = _interp_fn(w, lambda a, b, c: a * a + b * b + c * c + 0.01 * a * b)
    assert np.abs(oracle.apply_nlreac(w, y)).max() > 1e-4 * np.abs(r0).max()


@pytest.mark.parametrize("k,N", [(1, (3, 2, 2)), (2, (2, 2, 3)), (3, (2, 2, 2))])
def test_nlreac_jacobian_is_the_exact_derivative(k, N):
    """R is quadratic in x, so the central difference is exact for any step:
    J(u) z = (R(u + s z) - R(u - s z)) / (2 s) (the action of dR/dc on z). A dropped factor 2 in
    the reaction term, a g-term left in the Jacobian or a wrong linearization point fails it."""
    w = synth.nlreac(k, N)
    rng = np.random.default_rng(5)
    u = rng.standard_normal(w.ndofs)
    z = rng.standard_normal(w.ndofs)
    J = oracle.apply_nlreac(w, z, u0=u)
    for s in (1.0, 0.37):
        fd = (oracle.apply_nlreac(w, u + s * z) - oracle.apply_nlreac(w, u - s * z)) / (2 * s)
        assert np.abs(J - fd).max() <= 1e-11 * np.abs(J).max()


def test_nlreac_jacobian_at_constant_half_is_the_linear_operator():
    """At u0 = 1/2 the reaction derivative 2 c u0 = c: J(1/2) z = a(z, .) of the paper's linear problem, i.e.
    apply_diffreac(z) - apply_diffreac(0) (itself pinned by its manufactured solution)."""
    k, N = 2, (3, 2, 2)
    wn = synth.nlreac(k, N)
    wl = synth.diffreac(k, N, quad=k + 2)
    z = np.random.default_rng(9).standard_normal(wn.ndofs)
    J = oracle.apply_nlreac(wn, z, u0=np.full(wn.ndofs, 0.5))
    A = oracle.apply_diffreac(wl, z) - oracle.apply_diffreac(wl, np.zeros_like(z))
    assert np.abs(J - A).max() <= 1e-12 * np.abs(A).max()


def test_nlreac_jacobian_symmetric():
    """J(u0) = SIPG (theta = -1) + the mass matrix weighted by 2 c u0: symmetric for any u0."""
    k, N = 1, (2, 2, 3)
    w = synth.nlreac(k, N)
    u0 = np.random.default_rng(3).standard_normal(w.ndofs)
    nd = w.ndofs
    J = np.zeros((nd, nd))
    for j in range(nd):
        e = np.zeros(nd)
        e[j] = 1.0
        J[:, j] = oracle.apply_nlreac(w, e, u0=u0)
    assert np.abs(J - J.T).max() <= 1e-12 * np.abs(J).max()


# ---------------------------------------------------------------- Stokes
def _stokes_exact(w):
    """Interpolant of the paper's solution: u = g = (4 x_1 (1 - x_1), 0, 0), p = 8 (1 - x_0)
    (0-based coordinates, R27), in the block layout [u_0 | u_1 | u_2 | p]."""
    n, k = w.n, w.k
    N0, N1, N2 = w.N
    c = np.arange(w.ncells)
    i2, i1, i0 = c % N2, (c // N2) % N1, c // (N1 * N2)

    def pts(m_):
        xi = 0.5 * (np.polynomial.legendre.leggauss(m_)[0] + 1.0) if m_ > 1 else np.array([0.5])
        j = np.arange(m_ ** 3)
        j0, j1, j2 = j % m_, (j // m_) % m_, j // (m_ * m_)
        return ((i0[:, None] + xi[j0][None, :]) / N0, (i1[:, None] + xi[j1][None, :]) / N1,
                (i2[:, None] + xi[j2][None, :]) / N2)
    X0, X1, X2 = pts(n)
    P0, _, _ = pts(k)
    u0 = 4.0 * X1 * (1.0 - X1)
    z = np.zeros_like(u0)
    p = 8.0 * (1.0 - P0)
    return np.concatenate([u0, z, z, p], axis=1).reshape(-1)


@pytest.mark.parametrize("k,N", [(2, (2, 3, 2)), (3, (2, 2, 2)), (4, (2, 1, 2))])
def test_stokes_manufactured_solution(k, N):
    """with mu = 1, f = 0, g = (4 x_1 (1 - x_1), 0, 0) the exact solution is u = g,
    p = 8 (1 - x_0), in (Q_k)^3 x Q_{k-1} for k >= 2; the DG form is consistent and the k+1 point rule
    integrates every term exactly, so the residual of the interpolant vanishes (every row: momentum and
    continuity, Dirichlet and Neumann boundary cells)."""
    w = synth.stokes(k, N)
    x = _stokes_exact(w)
    r = oracle.apply_stokes(w, x)
    r0 = oracle.apply_stokes(w, np.zeros_like(x))
    assert np.abs(r).max() <= 1e-11 * np.abs(r0).max()
    # not vacuous: a wrong pressure level violates the Neumann condition p = 0 at x_0 = 1
    y = x.copy().reshape(w.ncells, -1)
    y[:, 3 * w.n ** 3:] += 0.1
    assert np.abs(oracle.apply_stokes(w, y.reshape(-1))).max() > 1e-4 * np.abs(r0).max()


@pytest.mark.parametrize("k,N", [(1, (2, 2, 3)), (2, (2, 2, 2)), (3, (2, 1, 2))])
def test_stokes_bilinear_part_equals_kronecker_assembly(k, N):
    """R(x) - R(0) == the independent Kronecker assembly of Eq. stokes_weak (oracle/brute.py: 1D SIPG, 1D
    pressure-velocity coupling and mixed masses by exact polynomial integration, Dirichlet / Neumann ends of
    the cube), dense on tiny meshes; also symmetric (b(p, v) and b(q, u) are the same form)."""
    w = synth.stokes(k, N)
    K = brute.stokes_dense(w)
    assert np.abs(K - K.T).max() <= 1e-12 * np.abs(K).max()
    rng = np.random.default_rng(21)
    r0 = oracle.apply_stokes(w, np.zeros(w.ndofs))
    for _ in range(3):
        x = rng.standard_normal(w.ndofs)
        got = oracle.apply_stokes(w, x) - r0
        ref = K @ x
        assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max()


def test_stokes_penalty_linear():
    """The alpha-dependence of R is gamma([u] - g, [v]): linear in alpha."""
    k, N = 2, (2, 2, 2)
    ws = [synth.stokes(k, N, alpha=a) for a in (0.0, 3.0, 6.0)]
    x = np.random.default_rng(4).standard_normal(ws[0].ndofs)
    r = [oracle.apply_stokes(w, x) for w in ws]
    assert np.abs((r[2] - r[0]) - 2 * (r[1] - r[0])).max() <= 1e-12 * np.abs(r[2]).max()
