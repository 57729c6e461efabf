"""x0-slab domain decomposition with a nearest-neighbour halo exchange.

Rank q of P owns the x0-planes [q N0 / P, (q+1) N0 / P). Because cells are ordered with i0
slowest, a slab is a contiguous range of the canonical vector and so are its first and last
planes: the halo messages are plain contiguous slices of x, sent without any packing kernel.
Per application (the only exchange step of the method):

    comm stream (high priority)           compute stream
    ---------------------------           --------------
    wait x ready                          planes [1, L-1)   (interior: x0-neighbours local)
    send plane 0     -> rank q-1
    send plane L-1   -> rank q+1
    recv halo_above  <- rank q+1
    recv halo_below  <- rank q-1
    record done  ───────────────────────> wait done; planes 0 and L-1 (use the halos)

The periodic wrap makes the ranks a ring (neighbours q +- 1 mod P). With P = 2 both
neighbours are the same rank: the two messages are distinguished by tag (gloo) and by posting
order (NCCL matches point-to-point operations between a pair in order: the sender posts
[plane 0, plane L-1], the receiver posts [halo_above, halo_below], which pair up).
P = 1 needs no exchange: the halos are x's own wrap planes.

The exchange uses torch.distributed point-to-point ops (NCCL over NVLink on GPUs, gloo on
CPU for the tests; gloo with CUDA tensors stages through pinned host buffers); the compute is libdg
(dg_apply_planes). On GPUs with k_gen / k_axis8 the payload is the boundary planes' face traces
(dg_pack_halo: u and d_0 u at the n^2 face points of each cell, SURVEY §8(e) "traces only"), consumed by
dg_apply_planes_tr: cfg3 9.4 MB instead of 37.7 MB per message, cfg4 26.2 MB instead of 65.5 MB.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class SlabPlan:
    rank: int
    world: int
    N0: int
    plane_begin: int
    nplanes: int

    @property
    def below(self) -> int:
        return (self.rank - 1) % self.world

    @property
    def above(self) -> int:
        return (self.rank + 1) % self.world

    @property
    def interior(self):
        """Local planes whose x0-neighbours are both local."""
        return (1, max(1, self.nplanes - 1))

    @property
    def boundary(self):
        """Local plane ranges that read a halo (computed after the exchange)."""
        L = self.nplanes
        if L == 1:
            return [(0, 1)]
        return [(0, 1), (L - 1, L)]


def plan(N0: int, rank: int, world: int) -> SlabPlan:
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if N0 < world:
        raise ValueError(f"N0={N0} planes cannot be split over {world} ranks")
    b = (rank * N0) // world
    e = ((rank + 1) * N0) // world
    return SlabPlan(rank, world, N0, b, e - b)


def exchange(send_lo, send_hi, recv_below, recv_above, p: SlabPlan, group=None, staged=None):
    """One halo exchange: send_lo (my lowest plane's payload) -> rank below, send_hi (my highest plane's) ->
    rank above; receive recv_above from the rank above and recv_below from the rank below. NCCL (or gloo on CPU
    tensors) point-to-point; `staged` = (host send_lo, host send_hi, host recv_below, host recv_above) pinned
    buffers for a CPU backend with CUDA tensors (gloo cannot send device memory): device -> host, exchange,
    host -> device on the current stream."""
    import torch.distributed as dist
    if staged is not None:
        import torch
        h_lo, h_hi, h_rb, h_ra = staged
        h_lo.copy_(send_lo)
        h_hi.copy_(send_hi)
        exchange(h_lo, h_hi, h_rb, h_ra, p, group)
        recv_below.copy_(h_rb, non_blocking=True)
        recv_above.copy_(h_ra, non_blocking=True)
        return
    ops = [
        dist.P2POp(dist.isend, send_lo, p.below, group, tag=0),   # -> their recv_above
        dist.P2POp(dist.isend, send_hi, p.above, group, tag=1),   # -> their recv_below
        dist.P2POp(dist.irecv, recv_above, p.above, group, tag=0),
        dist.P2POp(dist.irecv, recv_below, p.below, group, tag=1),
    ]
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def exchange_halos(x, halo_below, halo_above, plane_ndofs: int, p: SlabPlan, group=None):
    """Post the two sends and two receives of one full-plane halo exchange and wait for them.
    x: this rank's slab (1D, contiguous); halo_*: plane_ndofs-sized receive buffers."""
    if p.world == 1:
        halo_below.copy_(x[-plane_ndofs:])
        halo_above.copy_(x[:plane_ndofs])
        return
    exchange(x[:plane_ndofs], x[-plane_ndofs:], halo_below, halo_above, p, group)


class SlabApply:
    """One rank's share of r = A x with the halo exchange overlapped with interior planes.

    planes_fn(x, x_below, x_above, r, p_begin, p_end) computes the rows of local planes
    [p_begin, p_end) — libdg's dg_apply_planes on GPUs (see SlabOperator).
    Traces mode (pack_fn and planes_tr_fn given, GPU): the payload is the boundary planes' face traces
    (dg_pack_halo, 2 n^2 doubles per cell instead of n^3) and the boundary planes run dg_apply_planes_tr.
    NVTX ranges mark the pack, interior, halo and boundary parts of an application."""

    def __init__(self, p: SlabPlan, plane_ndofs: int, planes_fn, group=None, device=None, pack_fn=None,
                 planes_tr_fn=None, halo_ndofs: int = 0, staged: bool = False):
        import torch
        self.p = p
        self.plane_ndofs = plane_ndofs
        self.fn = planes_fn
        self.group = group
        self.device = device
        self.cuda = device is not None and torch.device(device).type == "cuda"
        self.traces = self.cuda and pack_fn is not None and planes_tr_fn is not None
        self.pack_fn, self.fn_tr = pack_fn, planes_tr_fn
        n = halo_ndofs if self.traces else plane_ndofs
        self.halo_below = torch.empty(n, dtype=torch.float64, device=device)
        self.halo_above = torch.empty(n, dtype=torch.float64, device=device)
        if self.traces:
            self.tr_lo = torch.empty(n, dtype=torch.float64, device=device)
            self.tr_hi = torch.empty(n, dtype=torch.float64, device=device)
        self.staged = None
        if staged and self.cuda:
            self.staged = tuple(torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4))
        self.payload_doubles = n  # per message (two messages each way per application)
        if self.cuda:
            self.comm_stream = torch.cuda.Stream(device=device, priority=-1)
            self.ev_x = torch.cuda.Event()
            self.ev_halo = torch.cuda.Event()
        # kernel launches per application: whole mesh 1; slab with L <= 2 planes 1 (after the
        # exchange); otherwise interior + 2 boundary planes; + the pack kernel in traces mode
        self.launches_per_apply = (1 if (p.world == 1 or p.nplanes <= 2) else 3) + (1 if self.traces and p.world > 1 else 0)

    def __call__(self, x, r, fn=None):
        """r = the rows of this slab; fn overrides the planes function for this call (same signature;
        e.g. the Jacobian action with its linearization point bound)."""
        import torch
        p = self.p
        if fn is not None and self.traces:
            raise ValueError("a planes-function override needs full-plane halos (SlabApply without traces)")
        traces = self.traces
        fn = self.fn if fn is None else fn
        if p.world == 1:
            # whole mesh on one rank: halos are the wrap planes of x itself, one launch
            L = p.nplanes
            fn(x, x[(L - 1) * self.plane_ndofs:], x[:self.plane_ndofs], r, 0, L)
            return r
        if not self.cuda:
            exchange_halos(x, self.halo_below, self.halo_above, self.plane_ndofs, p, self.group)
            a, b = p.interior
            if b > a:
                fn(x, self.halo_below, self.halo_above, r, a, b)
            for a, b in p.boundary:
                fn(x, self.halo_below, self.halo_above, r, a, b)
            return r
        nvtx = torch.cuda.nvtx
        cur = torch.cuda.current_stream(self.device)
        if traces:
            nvtx.range_push("slab:pack")
            self.pack_fn(x, self.tr_lo, self.tr_hi)
            nvtx.range_pop()
            send_lo, send_hi, bfn = self.tr_lo, self.tr_hi, self.fn_tr
        else:
            send_lo, send_hi, bfn = x[:self.plane_ndofs], x[-self.plane_ndofs:], fn
        self.ev_x.record(cur)
        # interior planes first (their x0-neighbours are local): the launch is queued before the exchange so a
        # host-blocking (staged) exchange still overlaps it on the GPU
        a, b = p.interior
        nvtx.range_push("slab:interior")
        if b > a and p.nplanes > 2:
            bfn(x, self.halo_below, self.halo_above, r, a, b)  # never reads the halos
        nvtx.range_pop()
        nvtx.range_push("slab:halo")
        with torch.cuda.stream(self.comm_stream):
            self.comm_stream.wait_event(self.ev_x)
            exchange(send_lo, send_hi, self.halo_below, self.halo_above, p, self.group, self.staged)
            self.ev_halo.record(self.comm_stream)
        nvtx.range_pop()
        cur.wait_event(self.ev_halo)
        nvtx.range_push("slab:boundary")
        if p.nplanes <= 2:
            bfn(x, self.halo_below, self.halo_above, r, 0, p.nplanes)
        else:
            for a, b in p.boundary:
                bfn(x, self.halo_below, self.halo_above, r, a, b)
        nvtx.range_pop()
        # keep the halo buffers alive until the compute stream is done with them
        self.halo_below.record_stream(cur)
        self.halo_above.record_stream(cur)
        return r


class SlabOperator:
    """libdg context for one rank's slab + the overlapped halo exchange (GPU, NCCL)."""

    def __init__(self, N, k: int, rank: int, world: int, *, geom_kind=0, coeff_kind=0, penalty_scale=10.0,
                 jac_fn=None, group=None, device=0, quad=None, problem=0, traces: bool = True, staged: bool = False,
                 basis: int = 0):
        """jac_fn(plane_begin, nplanes) -> host float64 [(nplanes) N1 N2, 9] (affine only); called for the
        L+2 planes plane_begin-1 .. plane_begin+L."""
        from .dg import Operator
        self.plan = plan(int(N[0]), rank, world)
        jac = None
        if geom_kind == 1:
            jac = jac_fn(self.plan.plane_begin - 1, self.plan.nplanes + 2)
        self.op = Operator(N, k, geom_kind=geom_kind, coeff_kind=coeff_kind, penalty_scale=penalty_scale, jac=jac,
                           plane_begin=self.plan.plane_begin, nplanes=self.plan.nplanes, device=device, quad=quad,
                           problem=problem, basis=basis)
        self.ndofs = self.op.ndofs
        self.offset = self.op.offset
        self.plane_ndofs = self.op.plane_ndofs
        # traces-only halos where the kernel supports them (k_gen, k_axis8, k_line), full boundary planes otherwise
        use_tr = traces and self.op.kernel_name in ("k_gen", "k_axis8", "k_line")
        self._apply = SlabApply(self.plan, self.plane_ndofs, self.op.apply_planes, group=group,
                                device=f"cuda:{device}", pack_fn=self.op.pack_halo if use_tr else None,
                                planes_tr_fn=self.op.apply_planes_tr if use_tr else None,
                                halo_ndofs=self.op.halo_ndofs, staged=staged)

    @property
    def launches_per_apply(self) -> int:
        return self._apply.launches_per_apply

    def _follow_current_stream(self):
        """SlabApply orders the halo events on torch's current stream; the libdg launches must go to the same
        stream (else a boundary-plane launch would not wait for the halo)."""
        import torch
        cur = torch.cuda.current_stream(self.op._stream.device)
        if cur != self.op._stream:
            self.op.set_stream(cur)

    def apply(self, x, r=None):
        import torch
        if r is None:
            r = torch.empty_like(x)
        self._follow_current_stream()
        return self._apply(x, r)

    def apply_jacobian(self, u0, z, r=None):
        """r = J(u0) z on this rank's slab (DG_PROBLEM_NLREAC): the halo exchange of z as for apply; u0 is
        needed on the owned planes only."""
        import torch
        if r is None:
            r = torch.empty_like(z)
        self._follow_current_stream()
        return self._apply(z, r, fn=lambda zz, zb, za, rr, a, b: self.op.apply_jacobian_planes(u0, zz, zb, za, rr, a, b))

    def close(self):
        self.op.close()
