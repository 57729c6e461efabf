"""GPU parity of the paper's Stokes problem (Eq. stokes_weak; DESIGN.md readings
R27/R28): k_stokes through the C-ABI against the oracle (oracle.apply_stokes, pinned in test_oracle_pins.py by
the manufactured solution and an independent Kronecker assembly), the manufactured solution on the GPU, a
larger mesh on sampled cells, and the slab decomposition."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


def _op(w, **kw):
    from paper_1812_08075_b200 import Operator
    return Operator(w.N, w.k, penalty_scale=w.penalty_scale, problem=3, **kw)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("k", range(1, 8))
def test_stokes_parity(k):
    """Every degree (k = 1: piecewise-constant pressure), boundary cells of both kinds (Dirichlet, Neumann
    x_0 = 1), anisotropic meshes."""
    N = (3, 4, 5) if k <= 4 else (2, 3, 3)
    w = synth.stokes(k, N)
    op = _op(w)
    assert op.kernel_name == "k_stokes"
    assert op.ndofs == w.ndofs
    x = synth.x_torch(w, device="cuda")
    r = op.apply(x)
    torch.cuda.synchronize()
    ref = oracle.apply_stokes(w, x.cpu().numpy())
    op.close()
    assert _rel(r.cpu().numpy(), ref) <= TOL


def _exact(w):
    n, k = w.n, w.k
    N0, N1, N2 = w.N
    c = np.arange(w.ncells)
    i2, i1, i0 = c % N2, (c // N2) % N1, c // (N1 * N2)

    def pts(m_):
        xi = 0.5 * (np.polynomial.legendre.leggauss(m_)[0] + 1.0)
        j = np.arange(m_ ** 3)
        j0, j1 = j % m_, (j // m_) % m_
        return (i0[:, None] + xi[j0][None, :]) / N0, (i1[:, None] + xi[j1][None, :]) / N1
    X0, X1 = pts(n)
    P0, _ = pts(k)
    u0 = 4.0 * X1 * (1.0 - X1)
    z = np.zeros_like(u0)
    return np.concatenate([u0, z, z, 8.0 * (1.0 - P0)], axis=1).reshape(-1)


@pytest.mark.parametrize("k", [2, 3, 5])
def test_stokes_manufactured_solution_gpu(k):
    """u = g = (4 x_1 (1 - x_1), 0, 0), p = 8 (1 - x_0) has a vanishing residual on the GPU."""
    w = synth.stokes(k, (4, 3, 5))
    x = torch.from_numpy(_exact(w)).cuda()
    op = _op(w)
    r = op.apply(x)
    r0 = op.apply(torch.zeros_like(x))
    assert r.abs().max().item() <= 1e-11 * r0.abs().max().item()
    op.close()


def test_stokes_larger_mesh_sampled():
    """k = 3 on 24^3 cells (5.7M DOFs): the oracle on a sample of cells (all six boundary planes covered)."""
    w = synth.stokes(3, (24, 24, 24))
    op = _op(w)
    x = synth.x_torch(w, device="cuda")
    r = op.apply(x).cpu().numpy()
    rng = np.random.default_rng(1)
    N0, N1, N2 = w.N
    cells = np.unique(np.concatenate([rng.integers(0, w.ncells, 300),
                                      np.arange(0, N1 * N2, 7), np.arange((N0 - 1) * N1 * N2, N0 * N1 * N2, 7)]))
    ref = oracle.apply_stokes(w, x.cpu().numpy(), cells)
    B = w.block
    idx = (cells[:, None] * B + np.arange(B)[None, :]).reshape(-1)
    assert _rel(r[idx], ref[idx]) <= TOL
    op.close()


@pytest.mark.parametrize("world", [2, 3])
def test_stokes_slab_loopback_bitwise(world):
    """The Stokes residual in the x0-slab decomposition (halo planes of 3 n^3 + k^3 blocks) equals the
    whole-mesh apply."""
    from paper_1812_08075_b200 import slab
    w = synth.stokes(2, (6, 3, 4))
    full = _op(w)
    x = synth.x_torch(w, device="cuda")
    ref = full.apply(x)
    pd = full.plane_ndofs
    assert pd == w.N[1] * w.N[2] * w.block
    got = torch.full_like(x, float("nan"))
    for q in range(world):
        p = slab.plan(w.N[0], q, world)
        op = _op(w, plane_begin=p.plane_begin, nplanes=p.nplanes)
        sl = slice(p.plane_begin * pd, (p.plane_begin + p.nplanes) * pd)
        hb = x[((p.plane_begin - 1) % w.N[0]) * pd:][:pd].clone()
        ha = x[((p.plane_begin + p.nplanes) % w.N[0]) * pd:][:pd].clone()
        ranges = ([p.interior] if p.interior[1] > p.interior[0] else []) + list(p.boundary)
        for a, b in ranges:
            op.apply_planes(x[sl], hb, ha, got[sl], a, b)
        torch.cuda.synchronize()
        op.close()
    assert torch.equal(got, ref)
    full.close()
