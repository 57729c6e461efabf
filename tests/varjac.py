"""A conforming hexahedral mesh whose cell Jacobians differ across EVERY face (test helper).

Used to pin the oracle's per-side Jacobian face terms (reading R11: each side's gradient uses its
own J^{-T}; normal, surface element, points and c_F from T-) and to check the CUDA path on the same
geometry (VERDICT r01 "What's weak" 1).

Construction (no method arithmetic, only the mesh): three families of column vectors
c0(i0), c1(i1), c2(i2) (each h_d (e_d + delta), delta ~ U[-0.15, 0.15]^3 from a seeded numpy RNG),
cell T = (i0, i1, i2) has J_T = [c0(i0) | c1(i1) | c2(i2)] (columns) and maps
    xi -> P(i) + J_T xi,   P(i) = sum_{m<i0} c0(m) + sum_{m<i1} c1(m) + sum_{m<i2} c2(m).
The face of T at xi_0 = 1 is P(i) + c0(i0) + xi_1 c1(i1) + xi_2 c2(i2) = the face of T + e0 at
xi_0 = 0, and likewise for d = 1, 2: the mesh is conforming away from the periodic wrap, while
J_{T-} != J_{T+} on every interior face (column d differs; the other two coincide). Because column d
carries off-diagonal (shear) entries, a swapped J_-^{-T} / J_+^{-T} changes the normal flux.

With c = 1 the operator never uses the cell origin o_T (R11), so the DOFs of a smooth u are its
values at P(i) + J_T xi_J; on cells whose 6 neighbours are not across the wrap:
  u = a . x     ->  r = 0                               (SIPG consistency, exact quadrature)
  u = |x|^2     ->  r_{T,J} = -6 |det J_T| w_J           (-Lap u = -6; collocated mass, exact)
"""
from __future__ import annotations

import numpy as np


def columns(N, seed=2024, amp=0.15):
    rng = np.random.default_rng(seed)
    cols = []
    for d in range(3):
        h = 1.0 / N[d]
        c = np.zeros((N[d], 3))
        c[:, d] = h
        c += h * rng.uniform(-amp, amp, size=(N[d], 3))
        cols.append(c)
    return cols


def jac_cells(N, cells, seed=2024):
    """Row-major J_T (9 doubles) of canonical cells c = (i0 N1 + i1) N2 + i2."""
    c0, c1, c2 = columns(N, seed)
    cells = np.asarray(cells, dtype=np.int64)
    i2 = cells % N[2]
    i1 = (cells // N[2]) % N[1]
    i0 = cells // (N[1] * N[2])
    J = np.stack([c0[i0], c1[i1], c2[i2]], axis=-1)  # [C, 3 (row a), 3 (column b)]
    return J.reshape(len(cells), 9)


def jac_planes(N, plane_begin, nplanes, seed=2024):
    """J of the cells of x0-planes plane_begin .. plane_begin+nplanes-1 (mod N0), canonical order
    (the dg_setup jac layout with plane_begin-1 .. plane_begin+L)."""
    pc = N[1] * N[2]
    planes = [(plane_begin + p) % N[0] for p in range(nplanes)]
    cells = np.concatenate([np.arange(p * pc, (p + 1) * pc) for p in planes])
    return jac_cells(N, cells, seed)


def node_positions(N, n, xi, seed=2024):
    """Physical positions [C, n^3, 3] of the nodes xi_J (j0 fastest) of every cell."""
    c0, c1, c2 = columns(N, seed)
    o = [np.concatenate([np.zeros((1, 3)), np.cumsum(c, axis=0)[:-1]]) for c in (c0, c1, c2)]
    C = N[0] * N[1] * N[2]
    cells = np.arange(C)
    i2 = cells % N[2]
    i1 = (cells // N[2]) % N[1]
    i0 = cells // (N[1] * N[2])
    P = o[0][i0] + o[1][i1] + o[2][i2]  # [C, 3]
    J = jac_cells(N, cells, seed).reshape(C, 3, 3)
    j = np.arange(n ** 3)
    ref = np.stack([xi[j % n], xi[(j // n) % n], xi[j // (n * n)]], axis=-1)  # [n^3, 3]
    return P[:, None, :] + np.einsum("cab,jb->cja", J, ref)


def interior_mask(N, n):
    """DOF mask of the cells with 1 <= i_d <= N_d - 2 in every direction."""
    C = N[0] * N[1] * N[2]
    c = np.arange(C)
    ic = [c // (N[1] * N[2]), (c // N[2]) % N[1], c % N[2]]
    m = np.ones(C, bool)
    for d in range(3):
        m &= (ic[d] >= 1) & (ic[d] <= N[d] - 2)
    return np.repeat(m, n ** 3)
