"""Seeded synthetic inputs and workload definitions — shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no basis, quadrature, flux or geometry
derivation). It only:
  * defines the five BASELINE.json workloads (mesh size, degree, geometry/coefficient kind);
  * draws the random numbers the workloads call for — the DOF vector x ~ U[-1,1] and the
    per-cell Jacobian perturbation E_T ~ U[-0.1,0.1] — with a counter-based generator, so
    that any rank / any test can regenerate any slice without communication.

Generator (reading R14):
    u(seed, stream, i) = (splitmix64(seed ^ splitmix64(stream ^ splitmix64(i))) >> 11) * 2^-53
    x_g   = 2 u(seed, STREAM_X, g) - 1                         g = global DOF index
    E_ab  = 0.1 (2 u(seed, STREAM_J, 9 c + 3 a + b) - 1)         c = canonical cell id
    J_T   = diag(h) (I + E_T)     (row-major, J[a][b] at 3 a + b), h_d = 1 / N_d

Two implementations of the same generator: numpy uint64 (well-defined wraparound; the
reference used by tests) and torch int64 (wraparound two's-complement arithmetic, logical
shifts emulated with masks) so that full-size inputs can be drawn on the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

STREAM_X = 1
STREAM_J = 2

_M64 = (1 << 64) - 1
_C_ADD = 0x9E3779B97F4A7C15
_C_M1 = 0xBF58476D1CE4E5B9
_C_M2 = 0x94D049BB133111EB


def _s64(v: int) -> int:
    """Reinterpret an unsigned 64-bit constant as signed int64."""
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


# --------------------------------------------------------------------------- numpy (uint64)
def _splitmix64_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(_C_ADD)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_C_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_C_M2)
        return z ^ (z >> np.uint64(31))


def hash_uniform_np(seed: int, stream: int, index) -> np.ndarray:
    """u in [0,1) for every index (numpy reference implementation)."""
    i = np.asarray(index, dtype=np.uint64)
    s = _splitmix64_np(i)
    s = _splitmix64_np(np.uint64(stream & _M64) ^ s)
    s = _splitmix64_np(np.uint64(seed & _M64) ^ s)
    return (s >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


# --------------------------------------------------------------------------- torch (int64)
def _lsr(z, s: int):
    """Logical right shift of an int64 tensor (two's-complement bit pattern)."""
    import torch
    return (z >> s) & ((1 << (64 - s)) - 1)


def _splitmix64_t(z):
    z = z + _s64(_C_ADD)
    z = (z ^ _lsr(z, 30)) * _s64(_C_M1)
    z = (z ^ _lsr(z, 27)) * _s64(_C_M2)
    return z ^ _lsr(z, 31)


def hash_uniform_torch(seed: int, stream: int, index):
    """u in [0,1) for every entry of an int64 tensor `index` (any device)."""
    s = _splitmix64_t(index)
    s = _splitmix64_t(s ^ _s64(stream))
    s = _splitmix64_t(s ^ _s64(seed))
    return _lsr(s, 11).to(__import__("torch").float64) * (2.0 ** -53)


# --------------------------------------------------------------------------- workloads
@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config (0-indexed)."""
    name: str
    k: int                      # polynomial degree per direction; n = k + 1
    N: tuple                    # global cells per direction (periodic unit cube)
    geom_kind: int              # 0 = axis-aligned J = diag(h); 1 = per-cell affine J = diag(h)(I+E)
    coeff_kind: int             # 0 = c = 1; 1 = c(x) = 1 + 0.5 sin(2 pi x0) cos(2 pi x1)
    seed: int
    penalty_scale: float = 10.0  # gamma = penalty_scale * k (k+1) / h  (BASELINE.json configs)
    quad: int = -1              # Gauss points per direction; -1 -> k + 1
    gpus: tuple = (1,)
    problem: int = 0            # 0: periodic SIPG of the configs; 1: the paper's diffusion-reaction problem; 2: its nonlinear
                                #    variant (R26); 3: the paper's Stokes problem (R27, block 3 n^3 + k^3 per cell)
                                #    (non-periodic cube, Dirichlet g = |x|^2, K = xx^T + I, c = 10,
                                #    f = -6; penalty_scale = alpha = 3, gamma = alpha k(k+2) |F|/|T|)
    text: str = ""
    basis: int = 0              # 0: Lagrange on the n Gauss-Legendre nodes (reading R8); 1: on the n Gauss-Lobatto nodes;
                                #    2: on the n equidistant nodes (the non-Gauss bases of SURVEY §8(f2): A != I at m = n)

    @property
    def n(self) -> int:
        return self.k + 1

    @property
    def m(self) -> int:
        return self.k + 1 if self.quad < 0 else self.quad

    @property
    def ncells(self) -> int:
        return self.N[0] * self.N[1] * self.N[2]

    @property
    def block(self) -> int:
        """DOFs per cell: n^3, or 3 n^3 + k^3 for Stokes (problem 3: [u_0 | u_1 | u_2 | p], R27)."""
        return 3 * self.n ** 3 + self.k ** 3 if self.problem == 3 else self.n ** 3

    @property
    def ndofs(self) -> int:
        return self.ncells * self.block

    @property
    def plane_cells(self) -> int:
        return self.N[1] * self.N[2]


CONFIGS = [
    Workload("cfg0_poisson_q1_8", 1, (8, 8, 8), 0, 0, seed=0,
             text="Poisson SIPG, DG Q1 on GL nodes, 2 Gauss pts/dir, periodic 8^3 axis-aligned, fp64, 1 GPU"),
    Workload("cfg1_poisson_q3_32", 3, (32, 32, 32), 0, 0, seed=1,
             text="Poisson SIPG, DG Q3, 4 Gauss pts/dir, periodic 32^3 axis-aligned (2.1M DOFs), 1 GPU"),
    Workload("cfg2_diffusion_q5_64_affine", 5, (64, 64, 64), 1, 1, seed=2,
             text="diffusion -div(c grad u) SIPG, DG Q5, 64^3 periodic per-cell affine, c(x) at quad pts, 1 GPU"),
    Workload("cfg3_poisson_q7_96", 7, (96, 96, 96), 0, 0, seed=3, gpus=(1, 2, 4, 8),
             text="Poisson SIPG, DG Q7, 96^3 axis-aligned periodic (453M DOFs), x0 slabs over 1/2/4/8 GPUs"),
    Workload("cfg4_diffusion_q4_256_affine", 4, (256, 256, 256), 1, 1, seed=4, gpus=(1, 2, 4, 8),
             text="diffusion SIPG as cfg2 with DG Q4 on 256^3 affine-perturbed cells (2.1B DOFs), 2/4/8 GPUs"),
]


def diffreac(k: int, N, seed: int = 11, quad: int = -1, alpha: float = 3.0) -> Workload:
    """The paper's diffusion-reaction problem on an axiparallel N0 x N1 x N2 mesh of (0,1)^3."""
    if isinstance(N, int):
        N = (N, N, N)
    return Workload(f"diffreac_k{k}_N{N[0]}x{N[1]}x{N[2]}_m{k + 1 if quad < 0 else quad}", k, tuple(N), 0, 0,
                    seed=seed, penalty_scale=alpha, quad=quad, problem=1)


def nlreac(k: int, N, seed: int = 13, alpha: float = 3.0) -> Workload:
    """The nonlinear variant of the paper's problem (reading R26: reaction c u^2)
    on an axiparallel N0 x N1 x N2 mesh of (0,1)^3, k+2 Gauss points per direction."""
    if isinstance(N, int):
        N = (N, N, N)
    return Workload(f"nlreac_k{k}_N{N[0]}x{N[1]}x{N[2]}_m{k + 2}", k, tuple(N), 0, 0,
                    seed=seed, penalty_scale=alpha, quad=k + 2, problem=2)


def stokes(k: int, N, seed: int = 17, alpha: float = 3.0) -> Workload:
    """The paper's Stokes problem (readings R27/R28) on an axiparallel
    N0 x N1 x N2 mesh of (0,1)^3: velocity Q_k, pressure Q_{k-1}, k+1 Gauss points per direction."""
    if isinstance(N, int):
        N = (N, N, N)
    return Workload(f"stokes_k{k}_N{N[0]}x{N[1]}x{N[2]}", k, tuple(N), 0, 0, seed=seed, penalty_scale=alpha,
                    problem=3)


def small(k: int, N, geom_kind: int = 0, coeff_kind: int = 0, seed: int = 7, quad: int = -1, basis: int = 0) -> Workload:
    """A small ad-hoc workload for tests."""
    if isinstance(N, int):
        N = (N, N, N)
    return Workload(f"small_k{k}_N{N[0]}x{N[1]}x{N[2]}_g{geom_kind}c{coeff_kind}" + ("", "_gll", "_equi")[basis], k, tuple(N),
                    geom_kind, coeff_kind, seed=seed, quad=quad, basis=basis)


# --------------------------------------------------------------------------- draws
def x_np(w: Workload, start: int = 0, count: int | None = None) -> np.ndarray:
    """x_g = 2u - 1 for global DOF indices [start, start+count) (numpy)."""
    if count is None:
        count = w.ndofs - start
    idx = np.arange(start, start + count, dtype=np.uint64)
    return 2.0 * hash_uniform_np(w.seed, STREAM_X, idx) - 1.0


def x_torch(w: Workload, start: int = 0, count: int | None = None, device="cpu", chunk: int = 1 << 26):
    """Same draw as x_np, produced in chunks on `device` (GPU for full-size workloads)."""
    import torch
    if count is None:
        count = w.ndofs - start
    out = torch.empty(count, dtype=torch.float64, device=device)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        idx = torch.arange(start + s, start + e, dtype=torch.int64, device=device)
        out[s:e] = hash_uniform_torch(w.seed, STREAM_X, idx) * 2.0 - 1.0
    return out


def x_cells_np(w: Workload, cells) -> np.ndarray:
    """DOF blocks of the listed canonical cells, shape (len(cells), n^3)."""
    n3 = w.n ** 3
    cells = np.asarray(cells, dtype=np.uint64)
    idx = cells[:, None] * np.uint64(n3) + np.arange(n3, dtype=np.uint64)[None, :]
    return 2.0 * hash_uniform_np(w.seed, STREAM_X, idx) - 1.0


def jac_cells_np(w: Workload, cells) -> np.ndarray:
    """Per-cell Jacobians J_T (row-major 3x3) of the listed canonical cells, shape (len, 9).

    geom_kind 0: J = diag(h).  geom_kind 1: J = diag(h)(I + E_T), E_ab ~ U[-0.1, 0.1].
    """
    cells = np.asarray(cells, dtype=np.uint64)
    h = np.array([1.0 / w.N[0], 1.0 / w.N[1], 1.0 / w.N[2]])
    J = np.zeros((len(cells), 9))
    if w.geom_kind == 0:
        J[:, 0], J[:, 4], J[:, 8] = h[0], h[1], h[2]
        return J
    idx = cells[:, None] * np.uint64(9) + np.arange(9, dtype=np.uint64)[None, :]
    E = 0.1 * (2.0 * hash_uniform_np(w.seed, STREAM_J, idx) - 1.0)
    for a in range(3):
        for b in range(3):
            J[:, 3 * a + b] = h[a] * ((1.0 if a == b else 0.0) + E[:, 3 * a + b])
    return J


def jac_planes_torch(w: Workload, plane_begin: int, nplanes: int, device="cpu"):
    """Jacobians of the cells in x0-planes [plane_begin, plane_begin+nplanes) (periodic wrap),
    shape (nplanes * N1 * N2, 9), canonical order. torch implementation of jac_cells_np."""
    import torch
    pc = w.plane_cells
    planes = [(plane_begin + p) % w.N[0] for p in range(nplanes)]
    cells = torch.cat([torch.arange(p * pc, (p + 1) * pc, dtype=torch.int64, device=device) for p in planes])
    h = [1.0 / w.N[0], 1.0 / w.N[1], 1.0 / w.N[2]]
    J = torch.zeros(cells.numel(), 9, dtype=torch.float64, device=device)
    if w.geom_kind == 0:
        J[:, 0], J[:, 4], J[:, 8] = h[0], h[1], h[2]
        return J
    for ab in range(9):
        a, b = divmod(ab, 3)
        E = 0.1 * (2.0 * hash_uniform_torch(w.seed, STREAM_J, cells * 9 + ab) - 1.0)
        J[:, ab] = h[a] * ((1.0 if a == b else 0.0) + E)
    return J


def cell_coords(w: Workload, c):
    """Canonical cell id -> (i0, i1, i2); ordering c = (i0 N1 + i1) N2 + i2 (i0 slowest)."""
    i2 = c % w.N[2]
    i1 = (c // w.N[2]) % w.N[1]
    i0 = c // (w.N[1] * w.N[2])
    return i0, i1, i2


def cell_id(w: Workload, i0, i1, i2):
    return (i0 * w.N[1] + i1) * w.N[2] + i2


def sample_cells(w: Workload, nrandom: int = 10000, seed: int = 12345, slabs: int = 8,
                 wrap_plane_cells: int = 4096, plane_cap: int = 20000) -> np.ndarray:
    """Deterministic verification sample (SURVEY §8(c) 'Oracle vs GPU'):
    every cell (at most `plane_cap` per plane) in the first and last x0-plane of each of `slabs` slabs (covers the slab
    boundaries at 2/4/8 ranks and the periodic wrap), `wrap_plane_cells` cells from each of
    the i1 and i2 wrap planes, and `nrandom` uniform random cells."""
    rng = np.random.default_rng(seed)
    N0, N1, N2 = w.N
    pc = N1 * N2
    sel = []
    for s in range(slabs):
        lo = (s * N0) // slabs
        hi = ((s + 1) * N0) // slabs - 1
        for p in {lo, hi}:
            if pc <= plane_cap:
                sel.append(np.arange(p * pc, (p + 1) * pc))
            else:
                sel.append(p * pc + rng.choice(pc, plane_cap, replace=False))
    for i1 in (0, N1 - 1):
        i0 = rng.integers(0, N0, wrap_plane_cells)
        i2 = rng.integers(0, N2, wrap_plane_cells)
        sel.append(cell_id(w, i0, i1, i2))
    for i2 in (0, N2 - 1):
        i0 = rng.integers(0, N0, wrap_plane_cells)
        i1 = rng.integers(0, N1, wrap_plane_cells)
        sel.append(cell_id(w, i0, i1, i2))
    sel.append(rng.integers(0, w.ncells, nrandom))
    return np.unique(np.concatenate(sel).astype(np.int64))
