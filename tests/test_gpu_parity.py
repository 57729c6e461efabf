"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): max|r_gpu - r_oracle| / max|r_oracle| <= 1e-11 in fp64.
Full vectors where the oracle finishes in seconds (small meshes spanning several CTAs with
ragged tails, cfg0, cfg1); at the full sizes of cfg2/cfg3/cfg4, in the launch configuration
bench.py times, a deterministic sample of cells (slab-boundary planes, wrap planes, random)
computed by the oracle one by one, plus size-independent properties (symmetry, A.1 = 0).
"""
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
                    jac=jac, quad=w.m, **kw)


def _rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def _full_check(w):
    op = _op(w)
    x = synth.x_torch(w, device="cuda")
    r = op.apply(x)
    torch.cuda.synchronize()
    jac = synth.jac_cells_np(w, np.arange(w.ncells)) if w.geom_kind else None
    ref = oracle.apply(w, x.cpu().numpy(), jac)
    err = _rel(r.cpu().numpy(), ref)
    op.close()
    return err


def _sampled_check(w, cells):
    op = _op(w)
    x = synth.x_torch(w, device="cuda")
    r = op.apply(x)
    torch.cuda.synchronize()
    n3 = w.n ** 3
    xv = x.view(w.ncells, n3)
    fetch = lambda ids: xv[torch.from_numpy(ids).cuda()].cpu().numpy()
    jf = (lambda ids: synth.jac_cells_np(w, ids)) if w.geom_kind else None
    ref = oracle.apply_sampled(w, cells, fetch, jf)
    got = r.view(w.ncells, n3)[torch.from_numpy(cells).cuda()].cpu().numpy()
    # the generator is shared: the sampled x blocks equal a fresh host draw
    assert np.array_equal(fetch(cells[:4]), synth.x_cells_np(w, cells[:4]))
    op.close()
    del x, r
    torch.cuda.empty_cache()
    return _rel(got, ref)


@pytest.mark.parametrize("k", range(1, 8))
@pytest.mark.parametrize("geom,coeff", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_small_all_degrees(k, geom, coeff):
    """Every degree, every geometry/coefficient combination; anisotropic N so that the cell count
    is not a multiple of the cells-per-CTA (ragged last CTA)."""
    N = (3, 5, 7) if k <= 3 else (3, 2, 5)
    w = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=100 + k)
    assert _full_check(w) <= TOL


def test_minimum_mesh():
    for k in (1, 4, 7):
        assert _full_check(synth.small(k, (2, 2, 2), geom_kind=1, coeff_kind=1, seed=5)) <= TOL


@pytest.mark.parametrize("cfg", [0, 1])
def test_config_full_vector(cfg):
    assert _full_check(synth.CONFIGS[cfg]) <= TOL


@pytest.mark.parametrize("cfg,nrand,cap", [(2, 3000, 4096), (3, 1500, 1024), (4, 3000, 1024)])
def test_config_sampled(cfg, nrand, cap):
    """Full-size configs in the bench's launch configuration: every cell of each cfg2 slab-boundary plane
    (4096), 1024 random cells of each cfg3 / cfg4 slab-boundary plane (16 planes), 128 cells of each wrap plane,
    and uniform random cells."""
    w = synth.CONFIGS[cfg]
    cells = synth.sample_cells(w, nrandom=nrand, plane_cap=cap, wrap_plane_cells=128)
    assert _sampled_check(w, cells) <= TOL


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_properties_full_size(cfg):
    """Symmetry y.Ax = x.Ay and A.1 = 0 at full size (north_star invariants)."""
    w = synth.CONFIGS[cfg]
    op = _op(w)
    x = synth.x_torch(w, device="cuda")
    import dataclasses
    y = synth.x_torch(dataclasses.replace(w, seed=w.seed + 1000), device="cuda")
    Ax = op.apply(x)
    Ay = op.apply(y)
    lhs = torch.dot(y, Ax).item()
    rhs = torch.dot(x, Ay).item()
    scale = max(torch.linalg.norm(y).item() * torch.linalg.norm(Ax).item(),
                torch.linalg.norm(x).item() * torch.linalg.norm(Ay).item())
    assert abs(lhs - rhs) <= 1e-12 * scale
    one = torch.ones_like(x)
    A1 = op.apply(one)
    assert A1.abs().max().item() <= 1e-12 * Ax.abs().max().item()
    op.close()


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("wi", [0, 1])
def test_slab_loopback_bitwise(world, wi):
    """World-size-P slab decomposition emulated on one GPU: P contexts, halos copied from the
    neighbours' planes, interior/boundary plane split — bitwise equal to the whole-mesh apply."""
    from paper_1812_08075_b200 import Operator, slab
    w = [synth.CONFIGS[1], synth.small(2, (6, 4, 5), geom_kind=1, coeff_kind=1, seed=3)][wi]
    full = _op(w)
    x = synth.x_torch(w, device="cuda")
    ref = full.apply(x)
    pd = full.plane_ndofs
    got = torch.full_like(x, float("nan"))
    for q in range(world):
        p = slab.plan(w.N[0], q, world)
        jac = synth.jac_planes_torch(w, p.plane_begin - 1, p.nplanes + 2).numpy() if w.geom_kind else None
        op = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale,
                      jac=jac, plane_begin=p.plane_begin, nplanes=p.nplanes)
        xs = x[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        rs = got[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        hb = x[((p.plane_begin - 1) % w.N[0]) * pd:][:pd].clone()
        ha = x[((p.plane_begin + p.nplanes) % w.N[0]) * pd:][:pd].clone()
        a, b = p.interior
        if b > a:
            op.apply_planes(xs, hb, ha, rs, a, b)
        for a, b in p.boundary:
            op.apply_planes(xs, hb, ha, rs, a, b)
        torch.cuda.synchronize()
        op.close()
    assert torch.equal(got, ref)
    full.close()


@pytest.mark.parametrize("w,kern", [(synth.CONFIGS[1], "k_line"), (synth.small(7, (16, 8, 8), seed=33), "k_axis8"),
                                    (synth.small(4, (12, 8, 8), geom_kind=1, coeff_kind=1, seed=34), "k_gen")])
def test_host_pipeline_bitwise(w, kern):
    """dg_apply_host (H2D / compute / D2H pipelined over plane chunks; k_axis8: the TMA tensor map re-encoded
    for the staging buffer) == dg_apply, and the oracle."""
    op = _op(w)
    assert op.kernel_name == kern
    x = synth.x_torch(w, device="cuda")
    ref = op.apply(x).cpu()
    xh = x.cpu().pin_memory()
    rh = torch.empty_like(xh).pin_memory()
    op.apply_host(xh, rh)
    assert torch.equal(rh, ref)
    for _ in range(2):  # repeated host applies reuse the staging buffers, streams and events
        rh.zero_()
        op.apply_host(xh, rh)
        assert torch.equal(rh, ref)
    if w.ncells <= 8192:
        jac = synth.jac_cells_np(w, np.arange(w.ncells)) if w.geom_kind else None
        orc = oracle.apply(w, xh.numpy(), jac)
        assert np.abs(rh.numpy() - orc).max() / np.abs(orc).max() <= TOL
    op.close()


def test_apply_rejects_bad_arguments():
    from paper_1812_08075_b200 import DgError, dg
    w = synth.CONFIGS[0]
    op = _op(w)
    x = synth.x_torch(w, device="cuda")
    with pytest.raises(DgError):
        dg.dg_apply(op.ctx, x, x)                        # aliasing
    with pytest.raises(DgError):
        op.apply_planes(x, x[:op.plane_ndofs], x[:op.plane_ndofs], torch.empty_like(x), 0, w.N[0] + 1)
    with pytest.raises(DgError):
        op.apply(x.float())
    op.close()


@pytest.mark.parametrize("N", [(3, 4, 8), (2, 4, 4), (5, 8, 12), (4, 12, 4)])
def test_axis8_fast_path_small(N):
    """k_axis8 (axis-aligned, n = 8, 4x4 tiles marching along x0) on meshes with 1-3 tiles per
    direction (ring cells that wrap onto the tile itself) against the oracle."""
    from paper_1812_08075_b200 import Operator
    w = synth.small(7, N, seed=31)
    op = _op(w)
    assert op.kernel_name == "k_axis8"
    op.close()
    assert _full_check(w) <= TOL


def test_axis8_matches_general_kernel():
    import os
    w = synth.small(7, (4, 8, 8), seed=8)
    x = synth.x_torch(w, device="cuda")
    fast = _op(w)
    os.environ["DG_FORCE_GENERAL"] = "1"
    try:
        gen = _op(w)
    finally:
        del os.environ["DG_FORCE_GENERAL"]
    assert fast.kernel_name == "k_axis8" and gen.kernel_name == "k_cell_general"
    a = fast.apply(x)
    b = gen.apply(x)
    assert (a - b).abs().max().item() <= 1e-13 * b.abs().max().item()
    fast.close()
    gen.close()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_axis8_slab_loopback_bitwise(world):
    from paper_1812_08075_b200 import Operator, slab
    w = synth.small(7, (10, 8, 4), seed=12)
    full = _op(w)
    x = synth.x_torch(w, device="cuda")
    ref = full.apply(x)
    pd = full.plane_ndofs
    got = torch.full_like(x, float("nan"))
    for q in range(world):
        p = slab.plan(w.N[0], q, world)
        op = Operator(w.N, w.k, plane_begin=p.plane_begin, nplanes=p.nplanes)
        xs = x[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        rs = got[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        hb = x[((p.plane_begin - 1) % w.N[0]) * pd:][:pd].clone()
        ha = x[((p.plane_begin + p.nplanes) % w.N[0]) * pd:][:pd].clone()
        a, b = p.interior
        if b > a:
            op.apply_planes(xs, hb, ha, rs, a, b)
        for a, b in p.boundary:
            op.apply_planes(xs, hb, ha, rs, a, b)
        torch.cuda.synchronize()
        op.close()
    assert torch.equal(got, ref)
    full.close()


@pytest.mark.parametrize("k", range(1, 8))
@pytest.mark.parametrize("N", [(3, 5, 7), (2, 2, 2), (5, 2, 3)])
def test_line_all_degrees(k, N):
    """k_line (axis-aligned c = 1, L2-resident meshes: the kernel of cfg0 / cfg1; for k = 7 k_axis8 takes the
    meshes its tiles divide) on ragged meshes incl. the minimum N = 2, against the oracle, and against k_gen's
    line-operator form where k_gen's tiles divide the mesh."""
    w = synth.small(k, N, seed=250 + k)
    op = _op(w)
    if k < 7:
        assert op.kernel_name == "k_line"
    op.close()
    assert _full_check(w) <= TOL


@pytest.mark.parametrize("world", [2, 3])
def test_line_slab_loopback_bitwise(world):
    """k_line in the slab decomposition (block halos; the interior / boundary plane split) == whole mesh."""
    from paper_1812_08075_b200 import Operator, slab
    w = synth.small(3, (7, 5, 6), seed=43)
    full = _op(w)
    assert full.kernel_name == "k_line"
    x = synth.x_torch(w, device="cuda")
    ref = full.apply(x)
    pd = full.plane_ndofs
    got = torch.full_like(x, float("nan"))
    for q in range(world):
        p = slab.plan(w.N[0], q, world)
        op = Operator(w.N, w.k, plane_begin=p.plane_begin, nplanes=p.nplanes)
        xs = x[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        rs = got[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        hb = x[((p.plane_begin - 1) % w.N[0]) * pd:][:pd].clone()
        ha = x[((p.plane_begin + p.nplanes) % w.N[0]) * pd:][:pd].clone()
        a, b = p.interior
        if b > a:
            op.apply_planes(xs, hb, ha, rs, a, b)
        for a, b in p.boundary:
            op.apply_planes(xs, hb, ha, rs, a, b)
        torch.cuda.synchronize()
        op.close()
    assert torch.equal(got, ref)
    full.close()


# k_gen tile shapes (dg_capi.cu GenShape): n -> (T1, T2)
GEN_TILE = {2: (4, 4), 3: (2, 4), 4: (2, 4), 5: (2, 4), 6: (2, 2), 7: (2, 2), 8: (2, 2)}


@pytest.mark.parametrize("k", range(1, 8))
@pytest.mark.parametrize("geom,coeff", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gen_all_degrees(k, geom, coeff, monkeypatch):
    """k_gen (marching tiles with async staging) for every degree and geometry/coefficient
    combination (axis-aligned c = 1: the line-operator form), on meshes of 1 and 2-3 tiles per
    direction (ring cells wrapping onto the tile itself), against the oracle."""
    T1, T2 = GEN_TILE[k + 1]
    N = (3, T1, 3 * T2) if k % 2 else (4, 2 * T1, T2)
    monkeypatch.setenv("DG_AX8_GEN", "1")  # axis-aligned Q7 through k_gen instead of k_axis8
    monkeypatch.setenv("DG_NO_LINE", "1")  # axis-aligned c = 1 through k_gen instead of k_line
    w = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=200 + k)
    op = _op(w)
    assert op.kernel_name == "k_gen"
    op.close()
    assert _full_check(w) <= TOL


@pytest.mark.parametrize("k,geom,coeff", [(4, 1, 1), (5, 1, 1), (3, 0, 0), (2, 1, 0)])
def test_gen_chunks(k, geom, coeff, monkeypatch):
    """Plane chunks (DG_GEN_CHUNK) with a ragged last chunk: each chunk re-evaluates the face
    below its first plane (prologue); the result is identical to one chunk per tile column."""
    T1, T2 = GEN_TILE[k + 1]
    w = synth.small(k, (7, 2 * T1, 2 * T2), geom_kind=geom, coeff_kind=coeff, seed=300 + k)
    x = synth.x_torch(w, device="cuda")
    monkeypatch.setenv("DG_NO_LINE", "1")
    monkeypatch.setenv("DG_GEN_CHUNK", "3")
    a = _op(w)
    monkeypatch.setenv("DG_GEN_CHUNK", "0")
    b = _op(w)
    ra, rb = a.apply(x), b.apply(x)
    assert a.kernel_name == b.kernel_name == "k_gen"
    assert (ra - rb).abs().max().item() <= 1e-14 * rb.abs().max().item()
    a.close()
    b.close()
    assert _full_check(w) <= TOL


@pytest.mark.parametrize("k", [2, 4, 5])
def test_gen_matches_cell_kernel(k, monkeypatch):
    """k_gen against the plain cell-centric kernel (k_cell_general) on an affine c(x) mesh."""
    T1, T2 = GEN_TILE[k + 1]
    w = synth.small(k, (4, 2 * T1, 2 * T2), geom_kind=1, coeff_kind=1, seed=400 + k)
    x = synth.x_torch(w, device="cuda")
    g = _op(w)
    monkeypatch.setenv("DG_FORCE_GENERAL", "1")
    c = _op(w)
    assert g.kernel_name == "k_gen" and c.kernel_name == "k_cell_general"
    a, b = g.apply(x), c.apply(x)
    assert (a - b).abs().max().item() <= 1e-13 * b.abs().max().item()
    g.close()
    c.close()


@pytest.mark.parametrize("world", [2, 3])
def test_gen_slab_loopback_bitwise(world):
    """k_gen in the slab decomposition (halo planes from the neighbours, interior/boundary split)
    is bitwise equal to the whole-mesh apply."""
    from paper_1812_08075_b200 import Operator, slab
    w = synth.small(4, (6, 4, 4), geom_kind=1, coeff_kind=1, seed=41)
    full = _op(w)
    assert full.kernel_name == "k_gen"
    x = synth.x_torch(w, device="cuda")
    ref = full.apply(x)
    pd = full.plane_ndofs
    got = torch.full_like(x, float("nan"))
    for q in range(world):
        p = slab.plan(w.N[0], q, world)
        jac = synth.jac_planes_torch(w, p.plane_begin - 1, p.nplanes + 2).numpy()
        op = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale,
                      jac=jac, plane_begin=p.plane_begin, nplanes=p.nplanes)
        xs = x[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        rs = got[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        hb = x[((p.plane_begin - 1) % w.N[0]) * pd:][:pd].clone()
        ha = x[((p.plane_begin + p.nplanes) % w.N[0]) * pd:][:pd].clone()
        a, b = p.interior
        if b > a:
            op.apply_planes(xs, hb, ha, rs, a, b)
        for a, b in p.boundary:
            op.apply_planes(xs, hb, ha, rs, a, b)
        torch.cuda.synchronize()
        op.close()
    assert torch.equal(got, ref)
    full.close()


@pytest.mark.parametrize("k", range(1, 8))
@pytest.mark.parametrize("geom,coeff", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_quad_overintegration(k, geom, coeff):
    """General quadrature: k+2 Gauss points per direction, A != I (k_quad), every
    degree and geometry/coefficient combination, against the oracle evaluated with the same rule;
    meshes with ragged CTA tails (odd cell counts)."""
    N = (3, 2, 5) if k >= 5 else (3, 3, 5)
    w = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=500 + k, quad=k + 2)
    op = _op(w)
    assert op.kernel_name == "k_quad"
    op.close()
    assert _full_check(w) <= TOL


@pytest.mark.parametrize("k", [2, 4])
def test_quad_equals_collocation_for_polynomial_integrands(k):
    """With c = 1 both rules integrate exactly: the k+2-point operator (k_quad) equals the collocated
    one (k_gen) to rounding on an affine mesh."""
    w1 = synth.small(k, (4, 4, 4), geom_kind=1, coeff_kind=0, seed=77)
    w2 = synth.small(k, (4, 4, 4), geom_kind=1, coeff_kind=0, seed=77, quad=k + 2)
    x = synth.x_torch(w1, device="cuda")
    a, b = _op(w1), _op(w2)
    ra, rb = a.apply(x), b.apply(x)
    assert b.kernel_name.startswith("k_quad")
    assert (ra - rb).abs().max().item() <= 1e-12 * ra.abs().max().item()
    a.close()
    b.close()


def test_quad_rejects_unsupported_rules():
    from paper_1812_08075_b200 import DgError, dg
    for k, q in ((2, 6), (2, 2), (7, 10)):  # k+4, fewer points than k+1, k+3 beyond k = 6
        with pytest.raises(DgError) as ei:
            dg.dg_setup((4, 4, 4), k, q)
        assert ei.value.code == dg.DG_ERR_UNSUPPORTED


@pytest.mark.parametrize("k", range(1, 7))
@pytest.mark.parametrize("geom,coeff", [(0, 0), (1, 1)])
def test_quad_k3_overintegration(k, geom, coeff):
    """k+3 Gauss points per direction (SURVEY §8(f2), P:L604-616 raised quadrature counts): k_quad with
    m = n + 2 against the oracle evaluated with the same rule."""
    N = (3, 2, 5) if k >= 5 else (3, 3, 5)
    w = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=520 + k, quad=k + 3)
    op = _op(w)
    assert op.kernel_name == "k_quad"
    op.close()
    assert _full_check(w) <= TOL


@pytest.mark.parametrize("k", [2, 5])
def test_quad_k3_equals_collocation_for_polynomial_integrands(k):
    """With c = 1 every rule with >= k+1 points integrates exactly: the k+3-point operator equals the collocated one."""
    w1 = synth.small(k, (4, 4, 4), geom_kind=1, coeff_kind=0, seed=78)
    w3 = synth.small(k, (4, 4, 4), geom_kind=1, coeff_kind=0, seed=78, quad=k + 3)
    x = synth.x_torch(w1, device="cuda")
    a, b = _op(w1), _op(w3)
    ra, rb = a.apply(x), b.apply(x)
    assert (ra - rb).abs().max().item() <= 1e-12 * ra.abs().max().item()
    a.close()
    b.close()


@pytest.mark.parametrize("world", [2, 3])
def test_quad_slab_loopback_bitwise(world):
    """k_quad in the slab decomposition (halo planes from the neighbours) equals the whole-mesh apply."""
    from paper_1812_08075_b200 import Operator, slab
    w = synth.small(3, (6, 3, 4), geom_kind=1, coeff_kind=1, seed=43, quad=5)
    full = _op(w)
    x = synth.x_torch(w, device="cuda")
    ref = full.apply(x)
    pd = full.plane_ndofs
    got = torch.full_like(x, float("nan"))
    for q in range(world):
        p = slab.plan(w.N[0], q, world)
        jac = synth.jac_planes_torch(w, p.plane_begin - 1, p.nplanes + 2).numpy()
        op = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale,
                      jac=jac, plane_begin=p.plane_begin, nplanes=p.nplanes, quad=w.m)
        xs = x[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        rs = got[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        hb = x[((p.plane_begin - 1) % w.N[0]) * pd:][:pd].clone()
        ha = x[((p.plane_begin + p.nplanes) % w.N[0]) * pd:][:pd].clone()
        a, b = p.interior
        if b > a:
            op.apply_planes(xs, hb, ha, rs, a, b)
        for a, b in p.boundary:
            op.apply_planes(xs, hb, ha, rs, a, b)
        torch.cuda.synchronize()
        op.close()
    assert torch.equal(got, ref)
    full.close()


def test_quad_config_sampled():
    """k_quad at the full size of cfg2 (Q5 on 64^3 affine cells, c(x)) with 7 Gauss points per direction,
    on the deterministic cell sample (slab-boundary and wrap planes, random cells)."""
    import dataclasses
    w = dataclasses.replace(synth.CONFIGS[2], quad=7)
    cells = synth.sample_cells(w, nrandom=1500, plane_cap=48, wrap_plane_cells=64)
    assert _sampled_check(w, cells) <= TOL


# ------------------------------------------------------------------ the paper's diffusion-reaction problem
def _dr_op(w, **kw):
    from paper_1812_08075_b200 import Operator
    return Operator(w.N, w.k, penalty_scale=w.penalty_scale, quad=w.m, problem=1, **kw)


@pytest.mark.parametrize("k", range(1, 8))
def test_diffreac_parity(k):
    """R(x) of Eq. diffreac_weak (K = xx^T + I, c = 10, f = -6, Dirichlet g = |x|^2 on the
    non-periodic cube, alpha = 3) on the GPU (k_quad, k+2 points) against the oracle, boundary cells on
    every side, anisotropic meshes with ragged CTA tails."""
    N = (3, 4, 5) if k <= 4 else (2, 3, 3)
    w = synth.diffreac(k, N, quad=k + 2)
    op = _dr_op(w)
    assert op.kernel_name == "k_quad_diffreac"
    x = synth.x_torch(w, device="cuda")
    r = op.apply(x)
    torch.cuda.synchronize()
    ref = oracle.apply_diffreac(w, x.cpu().numpy())
    op.close()
    assert _rel(r.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("k", [2, 3, 5])
def test_diffreac_manufactured_solution_gpu(k):
    """The interpolant of g = |x|^2 (in Q_k for k >= 2) has a vanishing residual on the GPU too."""
    w = synth.diffreac(k, (4, 3, 5), quad=k + 2)
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
    x = torch.from_numpy((X0 ** 2 + X1 ** 2 + X2 ** 2).reshape(-1)).cuda()
    op = _dr_op(w)
    r = op.apply(x)
    r0 = op.apply(torch.zeros_like(x))
    assert r.abs().max().item() <= 1e-11 * r0.abs().max().item()
    op.close()


@pytest.mark.parametrize("world", [2, 3])
def test_diffreac_slab_loopback_bitwise(world):
    """The diffusion-reaction residual in the x0-slab decomposition equals the whole-mesh apply (the
    boundary planes of the cube ignore the halos)."""
    from paper_1812_08075_b200 import slab
    w = synth.diffreac(3, (6, 3, 4), quad=5)
    full = _dr_op(w)
    x = synth.x_torch(w, device="cuda")
    ref = full.apply(x)
    pd = full.plane_ndofs
    got = torch.full_like(x, float("nan"))
    for q in range(world):
        p = slab.plan(w.N[0], q, world)
        op = _dr_op(w, plane_begin=p.plane_begin, nplanes=p.nplanes)
        xs = x[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        rs = got[p.plane_begin * pd:(p.plane_begin + p.nplanes) * pd]
        hb = x[((p.plane_begin - 1) % w.N[0]) * pd:][:pd].clone()
        ha = x[((p.plane_begin + p.nplanes) % w.N[0]) * pd:][:pd].clone()
        a, b = p.interior
        if b > a:
            op.apply_planes(xs, hb, ha, rs, a, b)
        for a, b in p.boundary:
            op.apply_planes(xs, hb, ha, rs, a, b)
        torch.cuda.synchronize()
        op.close()
    assert torch.equal(got, ref)
    full.close()


@pytest.mark.parametrize("k", [2, 3])
def test_cg_solves_the_papers_problem(k):
    """CG driving dg_apply solves the paper's diffusion-reaction problem; with the manufactured
    data the discrete solution is the interpolant of g = |x|^2 (consistency + uniqueness), which CG must reach."""
    from paper_1812_08075_b200 import solve
    w = synth.diffreac(k, (3, 4, 3), quad=k + 2)
    op = _dr_op(w)
    res = solve.solve_residual(op, w.ndofs, rtol=1e-13, maxiter=3000)
    assert res.converged, res.residual_norms[-5:]
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
    exact = (X0 ** 2 + X1 ** 2 + X2 ** 2).reshape(-1)
    err = np.abs(res.x.cpu().numpy() - exact).max()
    assert err <= 1e-9, (err, res.iterations)
    op.close()


def test_cg_graph_matches_cg():
    """The CUDA-graph CG (one captured iteration replayed, no host syncs inside) reaches the same discrete solution
    as the plain CG loop, in the same number of iterations up to the check granularity, and is faster per
    iteration (printed)."""
    import time
    from paper_1812_08075_b200 import solve
    w = synth.diffreac(3, (8, 8, 8), quad=5)
    op = _dr_op(w)
    t0 = time.perf_counter()
    a = solve.solve_residual(op, w.ndofs, rtol=1e-12, maxiter=3000)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    b = solve.solve_residual(op, w.ndofs, rtol=1e-12, maxiter=3000, graph=True, check_every=16)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    assert a.converged and b.converged
    assert abs(b.iterations - a.iterations) <= 17
    assert (a.x - b.x).abs().max().item() <= 1e-9 * a.x.abs().max().item()
    print(f"CG {a.iterations} it {1e6 * (t1 - t0) / a.iterations:.1f} us/it; graph CG {b.iterations} it "
          f"{1e6 * (t2 - t1) / b.iterations:.1f} us/it incl. capture, {1e6 * b.seconds_per_iteration:.1f} us/it replayed")
    # the stream was restored after capture: a later apply runs on the original stream
    x = synth.x_torch(w, device="cuda")
    assert torch.isfinite(op.apply(x)).all()
    op.close()


