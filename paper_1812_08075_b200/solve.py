"""Conjugate gradients driving dg_apply ("a CG solve driving dg_apply" — the next use of the
same kernels). Every operator application is one libdg launch; the vector updates and dot products are
torch device ops (plumbing).

For the paper's diffusion-reaction problem (DG_PROBLEM_DIFFREAC) dg_apply returns the affine residual
R(x) = A x - b of Eq. diffreac_weak; A is symmetric positive definite (SIPG with theta = -1 and
the reaction mass, Dirichlet boundary faces), so CG on A x = b with b = -R(0), A y = R(y) - R(0) converges
to the discrete solution — for the manufactured data of the paper (g = |x|^2) and k >= 2 that
is exactly the interpolant of |x|^2.

For the nonlinear variant (DG_PROBLEM_NLREAC, reading R26) `newton` drives dg_apply (the residual) and
dg_apply_jacobian (the action J(u) z) in a Newton-CG iteration: J(u) is symmetric
(SIPG theta = -1 plus the mass weighted by 2 c u) and positive definite while u > -1/(2c)-ish, which holds
along the iteration from u = 0 for the manufactured data.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class CGResult:
    x: object
    iterations: int
    residual_norms: list
    converged: bool


def cg(apply_A, b, x0=None, rtol: float = 1e-12, maxiter: int = 2000) -> CGResult:
    """Solve A x = b for SPD A given as a function y = apply_A(x) (torch tensors on the device)."""
    import torch
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    r = b - apply_A(x) if x0 is not None else b.clone()
    p = r.clone()
    rr = torch.dot(r, r)
    bn = torch.linalg.norm(b).item()
    hist = [rr.sqrt().item()]
    it = 0
    while it < maxiter and hist[-1] > rtol * bn:
        Ap = apply_A(p)
        alpha = rr / torch.dot(p, Ap)
        x.add_(alpha * p)
        r.sub_(alpha * Ap)
        rr_new = torch.dot(r, r)
        p.mul_(rr_new / rr).add_(r)
        rr = rr_new
        it += 1
        hist.append(rr.sqrt().item())
    return CGResult(x, it, hist, hist[-1] <= rtol * bn)


def solve_residual(op, ndofs: int, device="cuda", rtol: float = 1e-12, maxiter: int = 2000) -> CGResult:
    """Solve R(x) = 0 for an affine residual operator (op.apply(x) = A x - b): CG on A x = -R(0)."""
    import torch
    z = torch.zeros(ndofs, dtype=torch.float64, device=device)
    r0 = op.apply(z).clone()
    tmp = torch.empty_like(z)

    def apply_A(v):
        op.apply(v, tmp)
        return tmp - r0

    return cg(apply_A, -r0, rtol=rtol, maxiter=maxiter)


@dataclass
class NewtonResult:
    x: object
    iterations: int
    residual_norms: list
    cg_iterations: list
    converged: bool


def newton(op, ndofs: int, device="cuda", x0=None, rtol: float = 1e-12, maxiter: int = 20,
           cg_rtol: float = 1e-13, cg_maxiter: int = 4000) -> NewtonResult:
    """Solve R(x) = 0 for a DG_PROBLEM_NLREAC operator: x <- x - J(x)^{-1} R(x), the linear systems by CG on
    the matrix-free Jacobian action op.apply_jacobian(x, .) (one libdg launch each)."""
    import torch
    x = torch.zeros(ndofs, dtype=torch.float64, device=device) if x0 is None else x0.clone()
    r = op.apply(x).clone()
    r_init = torch.linalg.norm(op.apply(torch.zeros_like(x))).item()
    hist = [torch.linalg.norm(r).item()]
    cgits = []
    it = 0
    jz = torch.empty_like(x)

    def apply_J(v):
        op.apply_jacobian(x, v, jz)
        return jz

    while it < maxiter and hist[-1] > rtol * r_init:
        res = cg(apply_J, -r, rtol=cg_rtol, maxiter=cg_maxiter)
        cgits.append(res.iterations)
        x.add_(res.x)
        op.apply(x, r)
        it += 1
        hist.append(torch.linalg.norm(r).item())
    return NewtonResult(x, it, hist, cgits, hist[-1] <= rtol * r_init)
