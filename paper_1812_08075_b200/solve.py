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
    seconds_per_iteration: float | None = None  # cg_graph: wall time of the replayed iterations


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


def cg_graph(apply_into, b, rtol: float = 1e-12, maxiter: int = 2000, check_every: int = 16,
             on_capture=None, timed_iterations: int | None = None) -> CGResult:
    """CG with one iteration (operator application, two dot products, three vector updates) captured in a CUDA
    graph and replayed `check_every` times between host-side convergence checks: no host synchronisation
    inside the iteration, one graph launch per iteration instead of ~10 kernel launches.

    apply_into(v, out) writes A v into `out` on the current stream (libdg: dg_apply on the context stream;
    `on_capture(stream)` is called inside the capture so the caller can point the context at the capture
    stream, and with None afterwards to restore it). Iterates equal those of `cg` up to rounding; the
    iteration count is rounded up to a multiple of check_every (extra iterations after convergence are
    harmless: alpha = beta = 0 once r = 0)."""
    import torch
    x = torch.zeros_like(b)
    r = b.clone()
    p = r.clone()
    Ap = torch.empty_like(b)
    rr = torch.dot(r, r)
    zero = torch.zeros((), dtype=b.dtype, device=b.device)
    bn = torch.linalg.norm(b).item()

    def step():
        apply_into(p, Ap)
        pAp = torch.dot(p, Ap)
        alpha = torch.where(pAp != 0, rr / pAp, zero)
        x.add_(p * alpha)
        r.sub_(Ap * alpha)
        rr_new = torch.dot(r, r)
        beta = torch.where(rr != 0, rr_new / rr, zero)
        p.mul_(beta).add_(r)
        rr.copy_(rr_new)

    hist = [rr.sqrt().item()]
    it = 0
    # warm-up iterations on a side stream (library handles, caching allocator), then capture one iteration
    side = torch.cuda.Stream(device=b.device)
    side.wait_stream(torch.cuda.current_stream(b.device))
    with torch.cuda.stream(side):
        if on_capture:
            on_capture(side)
        for _ in range(2):
            if hist[-1] <= rtol * bn:
                break
            step()
            it += 1
        if on_capture:
            on_capture(None)
    torch.cuda.current_stream(b.device).wait_stream(side)
    hist.append(rr.sqrt().item())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        if on_capture:
            on_capture(torch.cuda.current_stream(b.device))
        step()
    if on_capture:
        on_capture(None)
    if timed_iterations:
        # measurement mode (bench.py --solve): exactly timed_iterations replays timed with CUDA events on the
        # launching stream after 3 warm-up replays; no convergence loop
        st = torch.cuda.current_stream(b.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(timed_iterations):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        it += 3 + timed_iterations
        hist.append(rr.sqrt().item())
        return CGResult(x, it, hist, hist[-1] <= rtol * bn, e0.elapsed_time(e1) * 1e-3 / timed_iterations)
    import time
    t0, it0 = time.perf_counter(), it
    while it < maxiter and hist[-1] > rtol * bn:
        for _ in range(check_every):
            g.replay()
        it += check_every
        hist.append(rr.sqrt().item())
    spi = (time.perf_counter() - t0) / max(it - it0, 1)
    return CGResult(x, it, hist, hist[-1] <= rtol * bn, spi)


def solve_residual(op, ndofs: int, device="cuda", rtol: float = 1e-12, maxiter: int = 2000,
                   graph: bool = False, check_every: int = 16, timed_iterations: int | None = None) -> CGResult:
    """Solve R(x) = 0 for an affine residual operator (op.apply(x) = A x - b): CG on A x = -R(0).
    graph=True: the CUDA-graph CG (cg_graph); op must be a libdg Operator (its stream is pointed at the
    capture stream during capture)."""
    import torch
    z = torch.zeros(ndofs, dtype=torch.float64, device=device)
    r0 = op.apply(z).clone()
    tmp = torch.empty_like(z)
    if graph:
        orig = op._stream

        def apply_into(v, out):
            op.apply(v, out)
            out.sub_(r0)

        def on_capture(stream):
            op.set_stream(stream if stream is not None else orig)

        return cg_graph(apply_into, -r0, rtol=rtol, maxiter=maxiter, check_every=check_every,
                        on_capture=on_capture, timed_iterations=timed_iterations)

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
           cg_rtol: float = 1e-13, cg_maxiter: int = 4000, graph: bool = False) -> NewtonResult:
    """Solve R(x) = 0 for a DG_PROBLEM_NLREAC operator: x <- x - J(x)^{-1} R(x), the linear systems by CG on
    the matrix-free Jacobian action op.apply_jacobian(x, .) (one libdg launch each; graph=True: the inner CG
    as cg_graph, the linearization point x being a fixed buffer updated in place)."""
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

    orig = op._stream

    def on_capture(stream):
        op.set_stream(stream if stream is not None else orig)

    while it < maxiter and hist[-1] > rtol * r_init:
        if graph:
            res = cg_graph(lambda v, out: op.apply_jacobian(x, v, out), -r, rtol=cg_rtol, maxiter=cg_maxiter,
                           on_capture=on_capture)
        else:
            res = cg(apply_J, -r, rtol=cg_rtol, maxiter=cg_maxiter)
        cgits.append(res.iterations)
        x.add_(res.x)
        op.apply(x, r)
        it += 1
        hist.append(torch.linalg.norm(r).item())
    return NewtonResult(x, it, hist, cgits, hist[-1] <= rtol * r_init)
