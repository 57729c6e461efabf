"""Traces-only halo exchange (include/dg.h dg_pack_halo / dg_apply_planes_tr) on one GPU.

A slab needs from each x0-neighbour only u and d_0 u at the n^2 face points of every boundary cell
(P:L143-146 1-point face tables; P:L883-886 the normal direction contracted first). Splitting the mesh into
P slabs, packing each slab's boundary traces and handing them to its neighbours must reproduce the whole-mesh
apply bit for bit (same kernels, same line algebra for the traces), for the general kernel (axis-aligned and
affine + c(x)) and for the Q7 kernel; and the slab decomposition must match the oracle.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ops(w, P):
    from paper_1812_08075_b200 import Operator, slab
    whole = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale,
                     jac=synth.jac_planes_torch(w, -1, w.N[0] + 2).numpy() if w.geom_kind else None)
    parts = []
    for q in range(P):
        pl = slab.plan(w.N[0], q, P)
        jac = synth.jac_planes_torch(w, pl.plane_begin - 1, pl.nplanes + 2).numpy() if w.geom_kind else None
        parts.append(Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale,
                              jac=jac, plane_begin=pl.plane_begin, nplanes=pl.nplanes))
    return whole, parts


CASES = [
    # (k, N, geom, coeff, kernel)
    (2, (6, 4, 8), 1, 1, "k_gen"),
    (4, (6, 4, 8), 1, 1, "k_gen"),
    (5, (7, 2, 4), 1, 1, "k_gen"),
    (3, (6, 4, 8), 0, 0, "k_line"),
    (1, (5, 3, 4), 0, 0, "k_line"),
    (3, (6, 4, 8), 0, 1, "k_gen"),
    (7, (6, 2, 4), 0, 0, "k_axis8"),
]


@pytest.mark.parametrize("k,N,geom,coeff,kern", CASES)
@pytest.mark.parametrize("P", [2, 3])
def test_trace_halo_slabs_bitwise(k, N, geom, coeff, kern, P):
    w = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=60 + k)
    whole, parts = _ops(w, P)
    assert whole.kernel_name == kern and all(o.kernel_name == kern for o in parts)
    x = synth.x_torch(w, device="cuda")
    r_ref = whole.apply(x)
    n2 = w.n ** 2
    assert parts[0].halo_ndofs == w.N[1] * w.N[2] * 2 * n2
    xs, los, his = [], [], []
    for o in parts:
        xo = x[o.offset:o.offset + o.ndofs].clone()
        lo = torch.empty(o.halo_ndofs, dtype=torch.float64, device="cuda")
        hi = torch.empty_like(lo)
        o.pack_halo(xo, lo, hi)
        xs.append(xo)
        los.append(lo)
        his.append(hi)
    out = []
    for q, o in enumerate(parts):
        r = torch.full_like(xs[q], float("nan"))
        o.apply_planes_tr(xs[q], his[(q - 1) % P], los[(q + 1) % P], r, 0, o.nplanes)
        out.append(r)
    torch.cuda.synchronize()
    got = torch.cat(out).cpu().numpy()
    ref = r_ref.cpu().numpy()
    assert np.array_equal(got, ref), np.abs(got - ref).max() / np.abs(ref).max()
    jac = synth.jac_cells_np(w, np.arange(w.ncells)) if geom else None
    orc = oracle.apply(w, x.cpu().numpy(), jac)
    assert np.abs(got - orc).max() / np.abs(orc).max() <= 1e-11
    for o in parts + [whole]:
        o.close()


def test_trace_halo_unsupported_kernel():
    from paper_1812_08075_b200 import Operator
    from paper_1812_08075_b200.dg import DG_ERR_UNSUPPORTED, DgError
    w = synth.diffreac(2, (3, 3, 3), quad=4)
    op = Operator(w.N, w.k, quad=w.m, problem=1, penalty_scale=w.penalty_scale)
    x = torch.zeros(op.ndofs, dtype=torch.float64, device="cuda")
    lo = torch.zeros(op.halo_ndofs, dtype=torch.float64, device="cuda")
    with pytest.raises(DgError) as e:
        op.pack_halo(x, lo, lo.clone())
    assert e.value.code == DG_ERR_UNSUPPORTED
    op.close()
