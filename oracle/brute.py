"""Independent brute-force SIPG operator for AXIS-ALIGNED meshes with c = 1 — TEST INFRASTRUCTURE ONLY.

Pins the C oracle (oracle.c) with different arithmetic: on an axis-aligned periodic mesh
with c = 1 the SIPG operator of PAPER.md Eq. diffreac_weak (theta = -1) is the
Kronecker sum (DESIGN.md pin P-KRON)

    A_3D = A_1^(0) (x) M^(1) (x) M^(2) + M^(0) (x) A_1^(1) (x) M^(2) + M^(0) (x) M^(1) (x) A_1^(2)

in the per-direction global index I_d = i_d n + j_d, where
    * M^(d) = h_d diag(w)                the exact collocated 1D mass (n-point GL integrates
                                          l_i l_j, degree 2k <= 2n-1, exactly); checked here
                                          by exact polynomial integration;
    * A_1^(d)                            the 1D periodic SIPG matrix, assembled by hand:
          volume   (1/h) int_0^1 l_i' l_j'             (exact, numpy.polynomial.polyint)
          face     -{u'}[v] - [u]{v'} + gamma [u][v]    with [v] = v(T-) - v(T+),
                   {v'} = (v'(T-) + v'(T+))/2, gamma = penalty_scale k (k+1) / h.
Nodes come from numpy.polynomial.legendre.leggauss (a library routine), the Lagrange
polynomials from numpy.polynomial.Polynomial products — nothing from oracle.c.
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import Polynomial
from numpy.polynomial.legendre import leggauss


def gl01(n: int):
    t, w = leggauss(n)
    return 0.5 * (t + 1.0), 0.5 * w


def lagrange_polys(n: int):
    xi, _ = gl01(n)
    polys = []
    for j in range(n):
        p = Polynomial([1.0])
        for a in range(n):
            if a != j:
                p = p * Polynomial([-xi[a], 1.0]) / (xi[j] - xi[a])
        polys.append(p)
    return polys


def exact_int01(p: Polynomial) -> float:
    P = p.integ()
    return float(P(1.0) - P(0.0))


def one_d(k: int, N: int, penalty_scale: float = 10.0):
    """(A1, M1): the 1D periodic SIPG matrix and exact mass on N cells of size h = 1/N."""
    n = k + 1
    h = 1.0 / N
    L = lagrange_polys(n)
    dL = [p.deriv() for p in L]
    K = np.array([[exact_int01(dL[i] * dL[j]) for j in range(n)] for i in range(n)]) / h
    Mloc = np.array([[exact_int01(L[i] * L[j]) for j in range(n)] for i in range(n)]) * h
    e0 = np.array([p(0.0) for p in L])
    e1 = np.array([p(1.0) for p in L])
    d0 = np.array([p(0.0) for p in dL]) / h
    d1 = np.array([p(1.0) for p in dL]) / h
    gamma = penalty_scale * k * (k + 1) / h
    A = np.zeros((N * n, N * n))
    M = np.zeros((N * n, N * n))
    for c in range(N):
        s = slice(c * n, (c + 1) * n)
        A[s, s] += K
        M[s, s] += Mloc
    # face between cell c (T-) and c+1 (T+), periodic
    Jv = np.concatenate([e1, -e0])          # [v] = v(T-) - v(T+)
    Av = 0.5 * np.concatenate([d1, d0])     # {v'}
    B = -np.outer(Jv, Av) - np.outer(Av, Jv) + gamma * np.outer(Jv, Jv)
    for c in range(N):
        cp = (c + 1) % N
        idx = np.concatenate([np.arange(c * n, (c + 1) * n), np.arange(cp * n, (cp + 1) * n)])
        for a in range(2 * n):
            for b in range(2 * n):
                A[idx[a], idx[b]] += B[a, b]
    return A, M


def _perm(w):
    """perm[g] = I-space linear index (I0 n1 + I1) n2 + I2 of canonical DOF g."""
    n = w.n
    N0, N1, N2 = w.N
    g = np.arange(w.ndofs)
    J = g % (n ** 3)
    c = g // (n ** 3)
    j0, j1, j2 = J % n, (J // n) % n, J // (n * n)
    i2, i1, i0 = c % N2, (c // N2) % N1, c // (N1 * N2)
    I0, I1, I2 = i0 * n + j0, i1 * n + j1, i2 * n + j2
    return (I0 * (N1 * n) + I1) * (N2 * n) + I2


def dense(w) -> np.ndarray:
    """Dense A in canonical DOF order (tiny meshes only)."""
    assert w.geom_kind == 0 and w.coeff_kind == 0
    mats = [one_d(w.k, w.N[d], w.penalty_scale) for d in range(3)]
    A0, M0 = mats[0]
    A1, M1 = mats[1]
    A2, M2 = mats[2]
    AI = np.kron(A0, np.kron(M1, M2)) + np.kron(M0, np.kron(A1, M2)) + np.kron(M0, np.kron(M1, A2))
    p = _perm(w)
    return AI[np.ix_(p, p)]


def apply(w, x: np.ndarray) -> np.ndarray:
    """Matrix-free A x (canonical order) via the Kronecker sum with sparse 1D factors."""
    import scipy.sparse as sp
    assert w.geom_kind == 0 and w.coeff_kind == 0
    n = w.n
    N0, N1, N2 = w.N
    U = x.reshape(N0, N1, N2, n, n, n).transpose(0, 5, 1, 4, 2, 3).reshape(N0 * n, N1 * n, N2 * n)
    mats = [one_d(w.k, w.N[d], w.penalty_scale) for d in range(3)]
    m = [np.diag(mats[d][1]) for d in range(3)]
    A = [sp.csr_matrix(mats[d][0]) for d in range(3)]
    s0, s1, s2 = U.shape
    R = (A[0] @ U.reshape(s0, -1)).reshape(s0, s1, s2) * m[1][None, :, None] * m[2][None, None, :]
    R += (A[1] @ U.transpose(1, 0, 2).reshape(s1, -1)).reshape(s1, s0, s2).transpose(1, 0, 2) \
        * m[0][:, None, None] * m[2][None, None, :]
    R += (A[2] @ U.transpose(2, 0, 1).reshape(s2, -1)).reshape(s2, s0, s1).transpose(1, 2, 0) \
        * m[0][:, None, None] * m[1][None, :, None]
    return R.reshape(N0, n, N1, n, N2, n).transpose(0, 2, 4, 5, 3, 1).reshape(-1)
