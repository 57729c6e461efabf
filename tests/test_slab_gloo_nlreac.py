"""Multi-rank x0-slab path of the Jacobian action on CPU over gloo: SlabApply with a
per-call planes function (the one SlabOperator.apply_jacobian binds the linearization point into) exchanges
halos of z only; the per-plane compute is the oracle restricted to the planes it may read (NaN everywhere
else: z outside [a-1, b], u0 outside the rank's own planes), so any read outside the slab + halos shows up."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1812_08075_b200 import slab


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.nlreac(*spec)
        p = slab.plan(w.N[0], rank, world)
        pc, n3 = w.plane_cells, w.n ** 3
        pd = pc * n3
        z = torch.from_numpy(synth.x_np(w, p.plane_begin * pd, p.nplanes * pd))
        u0_local = np.sin(3.0 * synth.x_np(w, p.plane_begin * pd, p.nplanes * pd)) + 0.25

        def jac_planes(zl, zb, za, r, a, b):
            zg = np.full(w.ndofs, np.nan)
            ug = np.full(w.ndofs, np.nan)
            g0 = p.plane_begin
            zg[(g0 + a) * pd:(g0 + b) * pd] = zl.numpy()[a * pd:b * pd]
            ug[(g0 + a) * pd:(g0 + b) * pd] = u0_local[a * pd:b * pd]
            # the x0-neighbour planes: local or halo (the cube is not periodic: no wrap)
            for gp, lp in ((g0 + a - 1, a - 1), (g0 + b, b)):
                if 0 <= gp < w.N[0]:
                    src = zl.numpy()[lp * pd:(lp + 1) * pd] if 0 <= lp < p.nplanes else (zb if lp < 0 else za).numpy()
                    zg[gp * pd:(gp + 1) * pd] = src
            cells = np.arange((g0 + a) * pc, (g0 + b) * pc)
            # NaN rows of z the oracle never reads stay NaN; it reads only the cells' own blocks and neighbours
            rows = oracle.apply_nlreac(w, zg, u0=ug, cells=cells)
            r.numpy()[a * pd:b * pd] = rows[(g0 + a) * pd:(g0 + b) * pd]

        ap = slab.SlabApply(p, pd, None, device=None)
        r = torch.full_like(z, float("nan"))
        ap(z, r, fn=jac_planes)
        out_q.put((rank, p.plane_begin, p.nplanes, r.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,spec", [(2, (1, (4, 2, 3))), (3, (2, (6, 2, 2)))])
def test_slab_jacobian_matches_oracle(world, spec):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spec, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    w = synth.nlreac(*spec)
    x = synth.x_np(w)
    u0 = np.sin(3.0 * x) + 0.25
    ref = oracle.apply_nlreac(w, x, u0=u0)
    pd = w.plane_cells * w.n ** 3
    got = np.full(w.ndofs, np.nan)
    for rank, b, L, r in res:
        got[b * pd:(b + L) * pd] = r
    assert not np.isnan(got).any()
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
