"""GPU parity of the non-Gauss basis (Lagrange polynomials on the n Gauss-Lobatto nodes, A != I even
with m = n Gauss points; k_quad with M = N), against the oracle evaluated with the same basis and rule, and against
the GPU's own Gauss-Legendre basis through the exact change of basis r^L(x) = T^T r^G(T x) (T_ij = l^L_j(xi^G_i),
built here with numpy; tests/test_oracle_lobatto.py pins the same identity on the oracle)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


def _op(w, **kw):
    from paper_1812_08075_b200 import Operator
    jac = synth.jac_planes_torch(w, -1, w.N[0] + 2, device="cuda").cpu().numpy() if w.geom_kind else None
    return Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale,
                    jac=jac, quad=w.m, basis=w.basis, **kw)


def _lobatto_nodes(n):
    if n == 2:
        return np.array([0.0, 1.0])
    r = np.sort(np.polynomial.legendre.Legendre.basis(n - 1).deriv().roots().real)
    return np.concatenate([[0.0], 0.5 * (1.0 + r), [1.0]])


def _T(n):
    gx, _ = np.polynomial.legendre.leggauss(n)
    pts, nodes = 0.5 * (gx + 1.0), _lobatto_nodes(n)
    T = np.ones((n, n))
    for j in range(n):
        for a in range(n):
            if a != j:
                T[:, j] *= (pts - nodes[a]) / (nodes[j] - nodes[a])
    return T


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("geom,coeff", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("basis", [1, 2])
def test_lobatto_parity(k, geom, coeff, basis):
    """m = n Gauss points with the Gauss-Lobatto / equidistant basis (A != I), ragged meshes, full vectors against the
    oracle."""
    N = (3, 2, 5) if k >= 5 else (3, 3, 5)
    w = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=600 + k, basis=basis)
    op = _op(w)
    assert op.kernel_name == "k_quad"
    x = synth.x_torch(w, device="cuda")
    r = op.apply(x)
    torch.cuda.synchronize()
    jac = synth.jac_cells_np(w, np.arange(w.ncells)) if geom else None
    ref = oracle.apply(w, x.cpu().numpy(), jac)
    op.close()
    err = np.abs(r.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= TOL, err


@pytest.mark.parametrize("k,geom,coeff", [(2, 1, 1), (3, 0, 1), (4, 1, 0)])
def test_lobatto_overintegration_parity(k, geom, coeff):
    """The Gauss-Lobatto basis with k+2 Gauss points."""
    w = synth.small(k, (3, 3, 4), geom_kind=geom, coeff_kind=coeff, seed=620 + k, quad=k + 2, basis=1)
    op = _op(w)
    x = synth.x_torch(w, device="cuda")
    r = op.apply(x)
    torch.cuda.synchronize()
    jac = synth.jac_cells_np(w, np.arange(w.ncells)) if geom else None
    ref = oracle.apply(w, x.cpu().numpy(), jac)
    op.close()
    assert np.abs(r.cpu().numpy() - ref).max() / np.abs(ref).max() <= TOL


@pytest.mark.parametrize("k", [2, 3, 5])
def test_lobatto_change_of_basis_gpu(k):
    """GPU against GPU: the Gauss-Lobatto operator (k_quad, m = n) equals T^T A^G T with the collocated Gauss-Legendre
    operator (k_gen) on an affine c(x) mesh whose tiles k_gen divides."""
    n = k + 1
    N = (4, 4, 8) if n <= 5 else (4, 4, 4)
    wl = synth.small(k, N, geom_kind=1, coeff_kind=1, seed=640 + k, basis=1)
    wg = synth.small(k, N, geom_kind=1, coeff_kind=1, seed=640 + k, basis=0)
    T3 = torch.from_numpy(np.kron(_T(n), np.kron(_T(n), _T(n)))).cuda()
    a, b = _op(wl), _op(wg)
    assert a.kernel_name == "k_quad" and b.kernel_name.startswith("k_gen")
    x = synth.x_torch(wl, device="cuda")
    rl = a.apply(x)
    rg = b.apply((x.view(-1, n ** 3) @ T3.T).reshape(-1).contiguous())
    ref = (rg.view(-1, n ** 3) @ T3).reshape(-1)
    err = ((rl - ref).abs().max() / ref.abs().max()).item()
    a.close()
    b.close()
    assert err <= 1e-11, err


@pytest.mark.parametrize("world", [2, 3])
def test_lobatto_slab_loopback_bitwise(world):
    """The Gauss-Lobatto basis in the slab decomposition (full boundary planes) is bitwise equal to the whole mesh."""
    from paper_1812_08075_b200 import Operator, slab
    w = synth.small(3, (6, 3, 4), geom_kind=0, coeff_kind=1, seed=45, basis=1)
    full = _op(w)
    x = synth.x_torch(w, device="cuda")
    ref = full.apply(x)
    pd = full.plane_ndofs
    got = torch.full_like(x, float("nan"))
    for q in range(world):
        p = slab.plan(w.N[0], q, world)
        op = Operator(w.N, w.k, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale, quad=w.m, basis=1,
                      plane_begin=p.plane_begin, nplanes=p.nplanes)
        xs = x[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        rs = got[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        hb = x[((p.plane_begin - 1) % w.N[0]) * pd:][:pd].clone()
        ha = x[((p.plane_begin + p.nplanes) % w.N[0]) * pd:][:pd].clone()
        op.apply_planes(xs, hb, ha, rs, 0, p.nplanes)
        torch.cuda.synchronize()
        op.close()
    assert torch.equal(got, ref)
    full.close()


def test_lobatto_rejects_other_problems():
    from paper_1812_08075_b200 import dg
    with pytest.raises(dg.DgError):
        dg.dg_setup((2, 2, 2), 3, 5, problem=1, basis=1)
    with pytest.raises(dg.DgError):
        dg.dg_setup((2, 2, 2), 3, 4, basis=3)
