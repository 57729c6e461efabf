"""Multi-rank x0-slab path on CPU: world sizes 2-4 over gloo (no GPU).

The orchestration of paper_1812_08075_b200.slab (plane ranges, halo sends/receives on the
ring, interior/boundary split, P = 2 where both neighbours are the same rank) runs unchanged;
only the per-plane compute is replaced by the oracle's cell-local residual (test
infrastructure), so the assembled global r must equal the oracle's whole-mesh apply.
"""
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


def _oracle_planes_fn(w, p, jac_global):
    """planes_fn backed by the oracle: rows of local planes [a, b) from x, halo_below, halo_above."""
    n3 = w.n ** 3
    pc = w.plane_cells
    N0, N1, N2 = w.N

    def fn(x, xb, xa, r, a, b):
        xl = x.numpy().reshape(p.nplanes, pc, n3)
        hb = xb.numpy().reshape(pc, n3)
        ha = xa.numpy().reshape(pc, n3)
        cells, x7, j7 = [], [], []
        for lp in range(a, b):
            for rem in range(pc):
                i1, i2 = divmod(rem, N2)
                g0 = (p.plane_begin + lp) % N0
                cells.append(synth.cell_id(w, g0, i1, i2))
                blk = [xl[lp, rem]]
                blk.append(xl[lp - 1, rem] if lp - 1 >= 0 else hb[rem])
                blk.append(xl[lp + 1, rem] if lp + 1 < p.nplanes else ha[rem])
                for d, (ii, NN) in ((1, (i1, N1)), (2, (i2, N2))):
                    for delta in (-1, 1):
                        j1, j2 = i1, i2
                        if d == 1:
                            j1 = (i1 + delta) % N1
                        else:
                            j2 = (i2 + delta) % N2
                        blk.append(xl[lp, j1 * N2 + j2])
                x7.append(np.stack(blk))
        cells = np.array(cells)
        nb = oracle.neighbours(w, cells)
        j7 = jac_global[nb] if jac_global is not None else None
        rows = oracle.apply_cells_local(w, cells, np.stack(x7), j7)
        r.numpy().reshape(p.nplanes, pc, n3)[a:b] = rows.reshape(b - a, pc, n3)

    return fn


def _worker(rank, world, port, wspec, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.small(*wspec[:2], geom_kind=wspec[2], coeff_kind=wspec[3], seed=9)
        p = slab.plan(w.N[0], rank, world)
        n3 = w.n ** 3
        pd = w.plane_cells * n3
        x = torch.from_numpy(synth.x_np(w, p.plane_begin * pd, p.nplanes * pd))
        jac = synth.jac_cells_np(w, np.arange(w.ncells)) if w.geom_kind else None
        ap = slab.SlabApply(p, pd, _oracle_planes_fn(w, p, jac), device=None)
        # halo exchange alone
        hb = torch.empty(pd, dtype=torch.float64)
        ha = torch.empty(pd, dtype=torch.float64)
        slab.exchange_halos(x, hb, ha, pd, p)
        gb = ((p.plane_begin - 1) % w.N[0]) * pd
        ga = ((p.plane_begin + p.nplanes) % w.N[0]) * pd
        ok_halo = np.array_equal(hb.numpy(), synth.x_np(w, gb, pd)) and np.array_equal(ha.numpy(), synth.x_np(w, ga, pd))
        r = torch.full_like(x, float("nan"))
        ap(x, r)
        out_q.put((rank, p.plane_begin, p.nplanes, ok_halo, r.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,wspec", [(2, (1, (4, 3, 3), 0, 0)), (3, (2, (6, 3, 2), 1, 1)),
                                         (4, (1, (5, 2, 3), 1, 0)), (2, (2, (2, 3, 3), 0, 1))])
def test_slab_ring_matches_oracle(world, wspec):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, wspec, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    w = synth.small(*wspec[:2], geom_kind=wspec[2], coeff_kind=wspec[3], seed=9)
    jac = synth.jac_cells_np(w, np.arange(w.ncells)) if w.geom_kind else None
    ref = oracle.apply(w, synth.x_np(w), jac)
    pd = w.plane_cells * w.n ** 3
    got = np.full(w.ndofs, np.nan)
    for rank, b, L, ok_halo, r in res:
        assert ok_halo, f"rank {rank}: halo planes differ from the neighbours' planes"
        got[b * pd:(b + L) * pd] = r
    assert not np.isnan(got).any()
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


def test_plan_partitions_cover_mesh():
    for N0 in (2, 5, 8, 96, 256):
        for world in (1, 2, 3, 4, 8):
            if world > N0:
                continue
            ps = [slab.plan(N0, r, world) for r in range(world)]
            assert ps[0].plane_begin == 0
            for a, b in zip(ps, ps[1:]):
                assert a.plane_begin + a.nplanes == b.plane_begin
            assert ps[-1].plane_begin + ps[-1].nplanes == N0
            for p in ps:
                covered = set()
                a, b = p.interior
                covered |= set(range(a, b))
                for a, b in p.boundary:
                    covered |= set(range(a, b))
                assert covered == set(range(p.nplanes))
    with pytest.raises(ValueError):
        slab.plan(3, 0, 4)
