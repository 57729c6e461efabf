"""CPU oracle for the SIPG operator — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg may
import this package. The product package `paper_1812_08075_b200` never imports it, and the two
share no code: this side is plain C (oracle.c, the unfactorised quadrature definition) plus
numpy (brute.py, an independent Kronecker-sum assembly used to pin the C oracle).

`build()` compiles oracle.c with gcc -O2 -fopenmp (no -ffast-math, reading R15) into
oracle/liboracle.so.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.oracle_gauss_legendre.argtypes = [ctypes.c_int, dp, dp]
        L.oracle_basis_1d.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, dp]
        L.oracle_basis_1d_b.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp]
        L.oracle_gauss_lobatto.argtypes = [ctypes.c_int, dp]
        L.oracle_apply_b.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, dp, ctypes.c_int, ctypes.c_double, ctypes.c_int, dp, dp, i64p,
                                     ctypes.c_int64]
        L.oracle_apply_cells_local_b.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                                 ctypes.c_int, i64p, ctypes.c_int64, dp, dp, dp]
        L.oracle_apply.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, dp, ctypes.c_int, ctypes.c_double, dp, dp, i64p, ctypes.c_int64]
        L.oracle_apply_cells_local.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                               i64p, ctypes.c_int64, dp, dp, dp]
        L.oracle_apply_diffreac.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_double, dp, dp, i64p, ctypes.c_int64]
        L.oracle_apply_nlreac.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_int, dp, dp, dp, i64p, ctypes.c_int64]
        L.oracle_apply_stokes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                          dp, dp, i64p, ctypes.c_int64]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i64p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_threads(n: int) -> None:
    """OpenMP thread count of the oracle loops (timing only)."""
    lib().oracle_set_threads(int(n))


def gauss_legendre(m: int):
    """m-point Gauss-Legendre rule on [0,1] (oracle's own Newton iteration)."""
    xi = np.zeros(m)
    w = np.zeros(m)
    if lib().oracle_gauss_legendre(m, _dp(xi), _dp(w)) != 0:
        raise ValueError(f"invalid m={m}")
    return xi, w


def gauss_lobatto(n: int):
    """n Gauss-Lobatto nodes on [0,1] (oracle's own Newton iteration on P_{n-1}')."""
    xi = np.zeros(n)
    if lib().oracle_gauss_lobatto(n, _dp(xi)) != 0:
        raise ValueError(f"invalid n={n}")
    return xi


def basis_1d(n: int, pts, basis: int = 0):
    """Values and derivatives of the n Lagrange polynomials on the n GL nodes (basis 0) or the n Gauss-Lobatto
    nodes (basis 1) at `pts`: arrays [len(pts), n]."""
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    val = np.zeros((len(pts), n))
    der = np.zeros((len(pts), n))
    if lib().oracle_basis_1d_b(n, int(basis), len(pts), _dp(pts), _dp(val), _dp(der)) != 0:
        raise ValueError("invalid n / basis")
    return val, der


def apply(w, x: np.ndarray, jac: np.ndarray | None = None, cells=None) -> np.ndarray:
    """r = A x on the whole mesh of workload `w` (or only the rows of `cells`, others NaN)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    assert x.size == w.ndofs
    r = np.full(w.ndofs, np.nan)
    if w.geom_kind == 1:
        assert jac is not None and jac.shape == (w.ncells, 9)
        jac = np.ascontiguousarray(jac, dtype=np.float64)
        jp = _dp(jac)
    else:
        jp = None
    if cells is None:
        cp, nc = None, 0
    else:
        cells = np.ascontiguousarray(cells, dtype=np.int64)
        cp, nc = _i64p(cells), len(cells)
    rc = lib().oracle_apply_b(w.N[0], w.N[1], w.N[2], w.k, w.m, w.geom_kind, jp, w.coeff_kind,
                              float(w.penalty_scale), int(getattr(w, "basis", 0)), _dp(x), _dp(r), cp, nc)
    if rc != 0:
        raise ValueError("oracle_apply: invalid arguments")
    return r


def apply_diffreac(w, x: np.ndarray, cells=None) -> np.ndarray:
    """The paper's diffusion-reaction residual on the non-periodic unit cube of
    workload `w` (w.problem == 1; axiparallel, w.m Gauss points, alpha = w.penalty_scale): R(x), including the
    f and g terms (R(0) != 0)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    assert x.size == w.ndofs
    r = np.full(w.ndofs, np.nan)
    if cells is None:
        cp, nc = None, 0
    else:
        cells = np.ascontiguousarray(cells, dtype=np.int64)
        cp, nc = _i64p(cells), len(cells)
    rc = lib().oracle_apply_diffreac(w.N[0], w.N[1], w.N[2], w.k, w.m, float(w.penalty_scale), _dp(x), _dp(r),
                                     cp, nc)
    if rc != 0:
        raise ValueError("oracle_apply_diffreac: invalid arguments")
    return r


def apply_nlreac(w, x: np.ndarray, u0: np.ndarray | None = None, cells=None) -> np.ndarray:
    """The nonlinear variant of the paper's problem (reading R26: reaction c u^2, source
    f = c|x|^4 - 10|x|^2 - 6, same K, g, penalty as apply_diffreac). u0 is None: the residual R(x);
    else the Jacobian action J(u0) x at the linearization point u0."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    assert x.size == w.ndofs
    r = np.full(w.ndofs, np.nan)
    if u0 is not None:
        u0 = np.ascontiguousarray(u0, dtype=np.float64)
        assert u0.size == w.ndofs
    if cells is None:
        cp, nc = None, 0
    else:
        cells = np.ascontiguousarray(cells, dtype=np.int64)
        cp, nc = _i64p(cells), len(cells)
    rc = lib().oracle_apply_nlreac(w.N[0], w.N[1], w.N[2], w.k, w.m, float(w.penalty_scale), int(u0 is not None),
                                   None if u0 is None else _dp(u0), _dp(x), _dp(r), cp, nc)
    if rc != 0:
        raise ValueError("oracle_apply_nlreac: invalid arguments")
    return r


def apply_stokes(w, x: np.ndarray, cells=None) -> np.ndarray:
    """The paper's Stokes residual (Eq. stokes_weak; readings R27/R28) on the
    axiparallel unit-cube mesh of workload `w` (w.problem == 3): per cell [u_0 | u_1 | u_2 | p] blocks of
    3 n^3 + k^3 DOFs; alpha = w.penalty_scale."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    assert x.size == w.ndofs
    r = np.full(w.ndofs, np.nan)
    if cells is None:
        cp, nc = None, 0
    else:
        cells = np.ascontiguousarray(cells, dtype=np.int64)
        cp, nc = _i64p(cells), len(cells)
    rc = lib().oracle_apply_stokes(w.N[0], w.N[1], w.N[2], w.k, float(w.penalty_scale), _dp(x), _dp(r), cp, nc)
    if rc != 0:
        raise ValueError("oracle_apply_stokes: invalid arguments")
    return r


def neighbours(w, cells):
    """[len, 7] canonical ids: self, -e0, +e0, -e1, +e1, -e2, +e2 (periodic)."""
    cells = np.asarray(cells, dtype=np.int64)
    N0, N1, N2 = w.N
    i2 = cells % N2
    i1 = (cells // N2) % N1
    i0 = cells // (N1 * N2)
    out = np.zeros((len(cells), 7), dtype=np.int64)
    out[:, 0] = cells
    ic = [i0, i1, i2]
    for d in range(3):
        for s, delta in enumerate((-1, 1)):
            jc = [a.copy() for a in ic]
            jc[d] = (ic[d] + delta) % w.N[d]
            out[:, 1 + 2 * d + s] = (jc[0] * N1 + jc[1]) * N2 + jc[2]
    return out


def apply_cells_local(w, cells, x7: np.ndarray, j7: np.ndarray | None) -> np.ndarray:
    """Rows of r for `cells` from their own + 6 neighbour blocks x7 [len,7,n^3] and Jacobians
    j7 [len,7,9]. Returns [len, n^3]."""
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    n3 = w.n ** 3
    x7 = np.ascontiguousarray(x7, dtype=np.float64).reshape(len(cells), 7, n3)
    if j7 is None:
        j7 = np.zeros((len(cells), 7, 9))
    j7 = np.ascontiguousarray(j7, dtype=np.float64).reshape(len(cells), 7, 9)
    r = np.zeros((len(cells), n3))
    rc = lib().oracle_apply_cells_local_b(w.N[0], w.N[1], w.N[2], w.k, w.m, w.geom_kind, w.coeff_kind,
                                          float(w.penalty_scale), int(getattr(w, "basis", 0)), _i64p(cells),
                                          len(cells), _dp(x7), _dp(j7), _dp(r))
    if rc != 0:
        raise ValueError("oracle_apply_cells_local: invalid arguments")
    return r


def apply_sampled(w, cells, x_of_cells, jac_of_cells=None) -> np.ndarray:
    """Rows of r for `cells`, fetching blocks through callbacks
    x_of_cells(ids) -> [len, n^3] and jac_of_cells(ids) -> [len, 9]."""
    nb = neighbours(w, cells)
    flat = nb.reshape(-1)
    x7 = x_of_cells(flat).reshape(len(cells), 7, -1)
    j7 = None if (w.geom_kind == 0 or jac_of_cells is None) else jac_of_cells(flat).reshape(len(cells), 7, 9)
    return apply_cells_local(w, cells, x7, j7)
