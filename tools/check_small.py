"""One small application of each kernel family (quick per-kernel check against the oracle on a GPU box):
k_gen (affine, c(x)), k_gen line-operator, k_axis8, k_quad (periodic, diffusion-reaction, nonlinear residual
and Jacobian), k_stokes. Checks the results against the oracle as well."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import synth
from paper_1812_08075_b200 import Operator


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def run(w, kind):
    x = synth.x_torch(w, device="cuda")
    if kind == "periodic":
        jac = synth.jac_planes_torch(w, -1, w.N[0] + 2, device="cuda").cpu().numpy() if w.geom_kind else None
        op = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale,
                      jac=jac, quad=w.m)
        r = op.apply(x).cpu().numpy()
        jg = synth.jac_cells_np(w, np.arange(w.ncells)) if w.geom_kind else None
        ref = oracle.apply(w, x.cpu().numpy(), jg)
    elif kind == "dr":
        op = Operator(w.N, w.k, penalty_scale=w.penalty_scale, quad=w.m, problem=1)
        r = op.apply(x).cpu().numpy()
        ref = oracle.apply_diffreac(w, x.cpu().numpy())
    elif kind == "jac":
        op = Operator(w.N, w.k, penalty_scale=w.penalty_scale, quad=w.m, problem=2)
        u0 = torch.sin(x)
        r = op.apply_jacobian(u0, x).cpu().numpy()
        ref = oracle.apply_nlreac(w, x.cpu().numpy(), u0=u0.cpu().numpy())
    else:
        op = Operator(w.N, w.k, penalty_scale=w.penalty_scale, problem=3)
        r = op.apply(x).cpu().numpy()
        ref = oracle.apply_stokes(w, x.cpu().numpy())
    torch.cuda.synchronize()
    e = rel(r, ref)
    print(f"{op.kernel_name:18s} {w.name:40s} rel {e:.2e}")
    op.close()
    return e


errs = [
    run(synth.small(4, (4, 4, 4), geom_kind=1, coeff_kind=1, seed=3), "periodic"),  # k_gen n=5
    run(synth.small(2, (4, 4, 4), seed=4), "periodic"),                              # k_gen line operator
    run(synth.small(7, (3, 2, 4), seed=5), "periodic"),                              # k_axis8
    run(synth.small(3, (3, 3, 5), geom_kind=1, coeff_kind=1, seed=6, quad=5), "periodic"),  # k_quad
    run(synth.diffreac(3, (3, 4, 5), quad=5), "dr"),
    run(synth.nlreac(3, (3, 4, 5)), "jac"),
    run(synth.stokes(3, (3, 4, 5)), "stokes"),
]
assert max(errs) <= 1e-11, errs
print("ok")
