"""Pin of the oracle's per-side Jacobian face terms on a conforming mesh whose Jacobians differ across
every face (the T-/T+ branch of oracle.c's face loop was unpinned).

P:L760-769 (§2.1: the maps mu_T, n_F oriented T- -> T+) and P:L986-989 (Eq. diffreac_weak: the average
{c grad u} . n takes each side's gradient, the test term n.{c grad v} the test side's): on a conforming
affinely mapped mesh SIPG is consistent, so with exact quadrature
  u = a . x  ->  r = 0  and  u = |x|^2  ->  r_{T,J} = -6 |det J_T| w_J   on cells away from the wrap
whatever the per-cell J. A plausible slip in the face branch — the two sides' J^{-T} swapped for the
trial gradients, or the test function differentiated with the neighbour's J — keeps symmetry and
A 1 = 0 but breaks these identities; the mutation tests below compile such variants of oracle.c and
show the pins reject them.
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import oracle
import synth
from oracle import brute
import varjac

ORACLE_SRC = os.path.join(os.path.dirname(oracle.__file__), "oracle.c")


def _run(lib, w, x, jac):
    dp = ctypes.POINTER(ctypes.c_double)
    x = np.ascontiguousarray(x, dtype=np.float64)
    jac = np.ascontiguousarray(jac, dtype=np.float64)
    r = np.full(w.ndofs, np.nan)
    rc = lib.oracle_apply(w.N[0], w.N[1], w.N[2], w.k, w.m, 1, jac.ctypes.data_as(dp), 0, ctypes.c_double(w.penalty_scale),
                          x.ctypes.data_as(dp), r.ctypes.data_as(dp), None, ctypes.c_int64(0))
    assert rc == 0
    return r


def _setup_lib(L):
    dp = ctypes.POINTER(ctypes.c_double)
    L.oracle_apply.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp,
                               ctypes.c_int, ctypes.c_double, dp, dp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64]
    return L


def _pins(lib, k, N):
    """(max |r| on interior cells for u = a.x, max |r - (-6 |det J| w_J)| for u = |x|^2, scale)."""
    w = synth.small(k, N, geom_kind=1, coeff_kind=0, seed=3)
    n = w.n
    xi, wq = brute.gl01(n)
    jac = varjac.jac_cells(N, np.arange(w.ncells))
    P = varjac.node_positions(N, n, xi)
    m = varjac.interior_mask(N, n)
    x_lin = (0.7 * P[..., 0] - 1.1 * P[..., 1] + 0.4 * P[..., 2]).reshape(-1)
    r_lin = _run(lib, w, x_lin, jac)
    x_q = (P ** 2).sum(-1).reshape(-1)
    r_q = _run(lib, w, x_q, jac)
    j = np.arange(n ** 3)
    wJ = wq[j % n] * wq[(j // n) % n] * wq[j // (n * n)]
    adet = np.abs(np.linalg.det(jac.reshape(-1, 3, 3)))
    expect = (-6.0 * adet[:, None] * wJ[None, :]).reshape(-1)
    return np.abs(r_lin[m]).max(), np.abs(r_q[m] - expect[m]).max(), np.abs(expect[m]).max()


def _asym(lib, k, N):
    """|y.Ax - x.Ay| / (|y||Ax|) for two seeded random vectors (SIPG with theta = -1 is symmetric)."""
    w = synth.small(k, N, geom_kind=1, coeff_kind=0, seed=3)
    jac = varjac.jac_cells(N, np.arange(w.ncells))
    rng = np.random.default_rng(7)
    x, y = rng.uniform(-1, 1, w.ndofs), rng.uniform(-1, 1, w.ndofs)
    ax, ay = _run(lib, w, x, jac), _run(lib, w, y, jac)
    return abs(y @ ax - x @ ay) / (np.linalg.norm(y) * np.linalg.norm(ax))


def test_mesh_is_conforming_and_jacobians_differ():
    """The helper's geometry: shared faces coincide, J differs across every interior face."""
    N = (4, 5, 4)
    n = 3
    xi = np.array([0.0, 0.5, 1.0])  # include the end points: face nodes
    P = varjac.node_positions(N, n, xi)
    J = varjac.jac_cells(N, np.arange(np.prod(N))).reshape(-1, 3, 3)
    cid = lambda a, b, c: (a * N[1] + b) * N[2] + c
    j = np.arange(n ** 3)
    jj = [j % n, (j // n) % n, j // (n * n)]
    for d in range(3):
        lo = [0, 0, 0]
        hi = [0, 0, 0]
        hi[d] = 1
        a, b = cid(*[1 + lo[0], 1 + lo[1], 1 + lo[2]]), cid(*[1 + hi[0], 1 + hi[1], 1 + hi[2]])
        up = P[a][jj[d] == n - 1]
        dn = P[b][jj[d] == 0]
        np.testing.assert_allclose(up, dn, atol=1e-15)
        assert np.abs(J[a] - J[b]).max() > 1e-3


@pytest.mark.parametrize("k,N", [(1, (5, 4, 5)), (2, (5, 5, 4)), (3, (4, 5, 5)), (4, (4, 4, 5))])
def test_varjac_consistency(k, N):
    lin, quad, scale = _pins(oracle.lib(), k, N)
    assert lin < 1e-11
    if k >= 2:
        assert quad < 1e-11 * max(1.0, scale)
    assert _asym(oracle.lib(), k, N) < 1e-13


# ------------------------------------------------------------------ mutation checks
MUTATIONS = {
    # the two sides' J^{-T} swapped for the trial gradients g- / g+
    "swap_trial_jinv": ("mat_t_vec(Jminv, ghm, gm);\n                    mat_t_vec(Jpinv, ghp, gp);",
                        "mat_t_vec(Jpinv, ghm, gm);\n                    mat_t_vec(Jminv, ghp, gp);"),
    # the test function's gradient taken with the neighbour's J^{-T}
    "swap_test_jinv": ("const double* Jselfinv = self_is_minus ? Jminv : Jpinv;",
                       "const double* Jselfinv = self_is_minus ? Jpinv : Jminv;"),
    # both sides' trial gradients with T-'s J^{-T}
    "trial_jinv_minus_both": ("mat_t_vec(Jpinv, ghp, gp);", "mat_t_vec(Jminv, ghp, gp);"),
}


@pytest.fixture(scope="module")
def mutants(tmp_path_factory):
    src = open(ORACLE_SRC).read()
    out = {}
    d = tmp_path_factory.mktemp("mutants")
    for name, (a, b) in MUTATIONS.items():
        assert src.count(a) == 1, f"mutation {name}: pattern not found exactly once in oracle.c"
        c = d / f"{name}.c"
        c.write_text(src.replace(a, b))
        so = d / f"lib{name}.so"
        subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", str(so), str(c), "-lm"], check=True)
        out[name] = _setup_lib(ctypes.CDLL(str(so)))
    return out


@pytest.mark.parametrize("name", sorted(MUTATIONS))
def test_mutant_fails_pins(mutants, name):
    """Each mutated face branch violates linear / quadratic consistency (a wrong trial gradient) or symmetry
    (a wrong test gradient: the theta term is multiplied by [u] = 0 for smooth u, but it is the transpose of
    the flux term) on the varying-J mesh."""
    lin, quad, scale = _pins(mutants[name], 2, (5, 5, 4))
    asym = _asym(mutants[name], 2, (5, 5, 4))
    assert lin > 1e-6 or quad > 1e-6 * scale or asym > 1e-6, (name, lin, quad, asym)


@pytest.mark.parametrize("name", sorted(MUTATIONS))
def test_mutant_passes_uniform_pins(mutants, name):
    """...while the round-1 pins (uniform J) could not see it: with one J for every cell the mutants
    agree with the oracle (why this mesh is needed)."""
    w = synth.small(2, (4, 4, 4), geom_kind=1, coeff_kind=0, seed=5)
    J = 0.25 * (np.eye(3) + np.array([[0.08, -0.05, 0.03], [0.02, -0.09, 0.06], [-0.07, 0.04, 0.1]]))
    jac = np.tile(J.reshape(1, 9), (w.ncells, 1))
    x = synth.x_np(w)
    r_ref = oracle.apply(w, x, jac)
    r_mut = _run(mutants[name], w, x, jac)
    assert np.abs(r_mut - r_ref).max() <= 1e-12 * np.abs(r_ref).max()
