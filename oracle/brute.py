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


# ------------------------------------------------------------------------------------------------------
# Stokes (Eq. stokes_weak; readings R27/R28): the bilinear part
# R(x) - R(0) on an axiparallel mesh is, like the Poisson SIPG operator, a sum of Kronecker products of 1D
# matrices, because every term factorises over the three directions (a face with normal d integrates the
# direction-d trace terms times 1D masses in the two tangential directions):
#   velocity-velocity (each component): A_1^(0) (x) M (x) M + M (x) A_1^(1) (x) M + M (x) M (x) A_1^(2)
#       with the 1D SIPG matrices of the boundary conditions of the cube: Dirichlet at both ends of
#       directions 1, 2 and at x_0 = 0; nothing at x_0 = 1 (Neumann);
#   velocity component c - pressure: B_c = G^(c) in direction c, the 1D mixed mass P in the others,
#       G = -int q v' + sum over interior points {q}[v] + Dirichlet ends q v n  (b(p, v) of Eq. stokes_weak);
#   pressure - velocity: B_c^T (b(q, u) is the same form with the roles swapped).
# Exact polynomial integration (numpy.polynomial), numpy's leggauss nodes, nothing from oracle.c.
def _nodes_polys(nn: int):
    if nn == 1:
        return np.array([0.5]), [Polynomial([1.0])]
    return gl01(nn)[0], lagrange_polys(nn)


def stokes_one_d(k: int, N: int, alpha: float, dirichlet_left: bool, dirichlet_right: bool):
    """1D factors on N cells of size h: (A, M, G, P) — velocity SIPG (n = k+1 Lagrange polynomials on GL
    nodes), velocity mass, the pressure (k nodes) - velocity coupling G [velocity rows, pressure cols] and the
    mixed mass P [velocity rows, pressure cols]. gamma = alpha k (k+2) / h (P:L1116 -> P:L966-977)."""
    n, npr = k + 1, k
    h = 1.0 / N
    L = lagrange_polys(n)
    dL = [q.deriv() for q in L]
    _, Lp = _nodes_polys(npr)
    K = np.array([[exact_int01(dL[i] * dL[j]) for j in range(n)] for i in range(n)]) / h
    Ml = np.array([[exact_int01(L[i] * L[j]) for j in range(n)] for i in range(n)]) * h
    Gl = np.array([[-exact_int01(Lp[j] * dL[i]) for j in range(npr)] for i in range(n)])  # -int q v'  (h cancels)
    Pl = np.array([[exact_int01(L[i] * Lp[j]) for j in range(npr)] for i in range(n)]) * h
    e0, e1 = np.array([q(0.0) for q in L]), np.array([q(1.0) for q in L])
    d0, d1 = np.array([q(0.0) for q in dL]) / h, np.array([q(1.0) for q in dL]) / h
    p0, p1 = np.array([q(0.0) for q in Lp]), np.array([q(1.0) for q in Lp])
    gamma = alpha * k * (k + 2) / h
    A = np.zeros((N * n, N * n))
    M = np.zeros((N * n, N * n))
    G = np.zeros((N * n, N * npr))
    P = np.zeros((N * n, N * npr))
    for c in range(N):
        s, sp_ = slice(c * n, (c + 1) * n), slice(c * npr, (c + 1) * npr)
        A[s, s] += K
        M[s, s] += Ml
        G[s, sp_] += Gl
        P[s, sp_] += Pl
    Jv = np.concatenate([e1, -e0])
    Av = 0.5 * np.concatenate([d1, d0])
    Bf = -np.outer(Jv, Av) - np.outer(Av, Jv) + gamma * np.outer(Jv, Jv)
    Qa = 0.5 * np.concatenate([p1, p0])  # {q}
    for c in range(N - 1):
        idx = np.concatenate([np.arange(c * n, (c + 2) * n)])
        pidx = np.arange(c * npr, (c + 2) * npr)
        A[np.ix_(idx, idx)] += Bf
        G[np.ix_(idx, pidx)] += np.outer(Jv, Qa)  # ({q}, [v] n), n = +1
    # Dirichlet ends: [v] = v, {v'} = v', outer normal sn: -(u' sn) v - (u)(v' sn) + gamma u v; (q, v sn)
    for end, on in ((0, dirichlet_left), (1, dirichlet_right)):
        if not on:
            continue
        c = 0 if end == 0 else N - 1
        sn = -1.0 if end == 0 else 1.0
        e, dd, pe = (e0, d0, p0) if end == 0 else (e1, d1, p1)
        idx = np.arange(c * n, (c + 1) * n)
        A[np.ix_(idx, idx)] += -sn * np.outer(e, dd) - sn * np.outer(dd, e) + gamma * np.outer(e, e)
        G[np.ix_(idx, np.arange(c * npr, (c + 1) * npr))] += sn * np.outer(e, pe)
    return A, M, G, P


def stokes_dense(w) -> np.ndarray:
    """Dense bilinear part of the Stokes residual in the canonical block layout (tiny meshes only)."""
    k, n, npr = w.k, w.n, w.k
    f = [stokes_one_d(k, w.N[d], w.penalty_scale, True, d != 0) for d in range(3)]
    A = [x[0] for x in f]
    M = [x[1] for x in f]
    G = [x[2] for x in f]
    P = [x[3] for x in f]
    kron3 = lambda a, b, c: np.kron(a, np.kron(b, c))
    Av = kron3(A[0], M[1], M[2]) + kron3(M[0], A[1], M[2]) + kron3(M[0], M[1], A[2])
    Bc = [kron3(G[0], P[1], P[2]), kron3(P[0], G[1], P[2]), kron3(P[0], P[1], G[2])]
    nv, npp = Av.shape[0], Bc[0].shape[1]
    K = np.zeros((3 * nv + npp, 3 * nv + npp))
    for c in range(3):
        K[c * nv:(c + 1) * nv, c * nv:(c + 1) * nv] = Av
        K[c * nv:(c + 1) * nv, 3 * nv:] = Bc[c]
        K[3 * nv:, c * nv:(c + 1) * nv] = Bc[c].T
    # canonical order: cell c = (i0 N1 + i1) N2 + i2, block [u_0 | u_1 | u_2 | p], j0 fastest
    N0, N1, N2 = w.N
    perm = []
    for cell in range(w.ncells):
        i2, i1, i0 = cell % N2, (cell // N2) % N1, cell // (N1 * N2)
        for comp in range(4):
            m_ = npr if comp == 3 else n
            for J in range(m_ ** 3):
                j0, j1, j2 = J % m_, (J // m_) % m_, J // (m_ * m_)
                I = ((i0 * m_ + j0) * (N1 * m_) + (i1 * m_ + j1)) * (N2 * m_) + (i2 * m_ + j2)
                perm.append(I + (comp * nv if comp < 3 else 3 * nv))
    perm = np.array(perm)
    return K[np.ix_(perm, perm)]
