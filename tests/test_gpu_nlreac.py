"""GPU parity of the nonlinear variant of the paper's problem (reading R26): the
residual R(x) and the Jacobian action J(u0) z of k_quad modes 2 and 3 through the C-ABI
against the oracle (oracle.apply_nlreac, pinned in test_oracle_pins.py), the manufactured solution, slab
loopback of both, and Newton-CG driving them."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


def _op(w, **kw):
    from paper_1812_08075_b200 import Operator
    return Operator(w.N, w.k, penalty_scale=w.penalty_scale, quad=w.m, problem=2, **kw)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _interp(w, fn):
    xi, _ = np.polynomial.legendre.leggauss(w.n)
    xi = 0.5 * (xi + 1.0)
    N0, N1, N2 = w.N
    c = np.arange(w.ncells)
    i2, i1, i0 = c % N2, (c // N2) % N1, c // (N1 * N2)
    j = np.arange(w.n ** 3)
    j0, j1, j2 = j % w.n, (j // w.n) % w.n, j // (w.n * w.n)
    X0 = (i0[:, None] + xi[j0][None, :]) / N0
    X1 = (i1[:, None] + xi[j1][None, :]) / N1
    X2 = (i2[:, None] + xi[j2][None, :]) / N2
    return fn(X0, X1, X2).reshape(-1)


@pytest.mark.parametrize("k", range(1, 8))
def test_nlreac_residual_and_jacobian_parity(k):
    """R(x) and J(u0) z on the GPU against the oracle: every degree, boundary cells on all sides, anisotropic
    meshes with ragged CTA tails."""
    N = (3, 4, 5) if k <= 4 else (2, 3, 3)
    w = synth.nlreac(k, N)
    op = _op(w)
    assert op.kernel_name == "k_quad_nlreac"
    x = synth.x_torch(w, device="cuda")
    g = torch.Generator().manual_seed(100 + k)
    u0 = torch.randn(w.ndofs, generator=g, dtype=torch.float64).cuda()
    r = op.apply(x)
    jz = op.apply_jacobian(u0, x)
    torch.cuda.synchronize()
    xn, un = x.cpu().numpy(), u0.cpu().numpy()
    assert _rel(r.cpu().numpy(), oracle.apply_nlreac(w, xn)) <= TOL
    assert _rel(jz.cpu().numpy(), oracle.apply_nlreac(w, xn, u0=un)) <= TOL
    op.close()


@pytest.mark.parametrize("k", [2, 4])
def test_nlreac_manufactured_solution_gpu(k):
    """The interpolant of |x|^2 has a vanishing nonlinear residual on the GPU too (R26)."""
    w = synth.nlreac(k, (4, 3, 5))
    x = torch.from_numpy(_interp(w, lambda a, b, c: a * a + b * b + c * c)).cuda()
    op = _op(w)
    r = op.apply(x)
    r0 = op.apply(torch.zeros_like(x))
    assert r.abs().max().item() <= 1e-11 * r0.abs().max().item()
    op.close()


def test_nlreac_jacobian_rejected_on_linear_problems():
    """dg_apply_jacobian is defined for DG_PROBLEM_NLREAC contexts only (DG_ERR_UNSUPPORTED otherwise)."""
    from paper_1812_08075_b200 import Operator
    from paper_1812_08075_b200.dg import DgError, DG_ERR_UNSUPPORTED
    w = synth.diffreac(2, (3, 3, 3), quad=4)
    op = Operator(w.N, w.k, penalty_scale=w.penalty_scale, quad=w.m, problem=1)
    x = synth.x_torch(w, device="cuda")
    with pytest.raises(DgError) as e:
        op.apply_jacobian(x, x)
    assert e.value.code == DG_ERR_UNSUPPORTED
    op.close()


@pytest.mark.parametrize("world", [2, 3])
def test_nlreac_slab_loopback_bitwise(world):
    """Residual and Jacobian action in the x0-slab decomposition equal the whole-mesh applies bit for bit."""
    from paper_1812_08075_b200 import slab
    w = synth.nlreac(3, (6, 3, 4))
    full = _op(w)
    x = synth.x_torch(w, device="cuda")
    u0 = torch.sin(3.0 * x) + 0.5
    ref_r = full.apply(x)
    ref_j = full.apply_jacobian(u0, x)
    pd = full.plane_ndofs
    got_r = torch.full_like(x, float("nan"))
    got_j = torch.full_like(x, float("nan"))
    for q in range(world):
        p = slab.plan(w.N[0], q, world)
        op = _op(w, plane_begin=p.plane_begin, nplanes=p.nplanes)
        sl = slice(p.plane_begin * pd, (p.plane_begin + p.nplanes) * pd)
        hb = x[((p.plane_begin - 1) % w.N[0]) * pd:][:pd].clone()
        ha = x[((p.plane_begin + p.nplanes) % w.N[0]) * pd:][:pd].clone()
        xs, us = x[sl], u0[sl].contiguous()
        ranges = ([p.interior] if p.interior[1] > p.interior[0] else []) + list(p.boundary)
        for a, b in ranges:
            op.apply_planes(xs, hb, ha, got_r[sl], a, b)
            op.apply_jacobian_planes(us, xs, hb, ha, got_j[sl], a, b)
        torch.cuda.synchronize()
        op.close()
    assert torch.equal(got_r, ref_r)
    assert torch.equal(got_j, ref_j)
    full.close()


@pytest.mark.parametrize("k,graph", [(2, False), (3, False), (3, True)])
def test_newton_solves_the_nonlinear_problem(k, graph):
    """Newton-CG driving dg_apply / dg_apply_jacobian reaches the discrete solution, which for the manufactured
    data is the interpolant of |x|^2; the residual norms fall quadratically in the last steps."""
    from paper_1812_08075_b200 import solve
    w = synth.nlreac(k, (3, 4, 3))
    op = _op(w)
    res = solve.newton(op, w.ndofs, rtol=1e-12, graph=graph)
    assert res.converged, res.residual_norms
    exact = _interp(w, lambda a, b, c: a * a + b * b + c * c)
    err = np.abs(res.x.cpu().numpy() - exact).max()
    assert err <= 1e-9, (err, res.residual_norms)
    h = res.residual_norms
    # quadratic convergence: some step squares the relative residual (within a constant)
    rel = [v / h[0] for v in h]
    assert any(rel[i + 1] <= 10 * rel[i] ** 2 + 1e-13 for i in range(len(rel) - 1) if rel[i] < 1e-2), rel
    op.close()
