"""Two processes on ONE GPU run the real libdg kernels through SlabOperator (x0-slabs, traces-only halo,
comm stream, events, NVTX ranges) with a host-staged gloo exchange standing in for NCCL (the CUDA
overlap branch of slab.py had never executed). The assembled slabs must equal the whole-mesh apply bit for bit.
The ranks do not wait on each other's kernels (each exchange completes on the host), so sharing one GPU is safe.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, N, geom, coeff, traces, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import synth
    from paper_1812_08075_b200 import slab
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=70 + k)
    jf = (lambda pb, npl: synth.jac_planes_torch(w, pb, npl).numpy()) if geom else None
    sop = slab.SlabOperator(w.N, w.k, rank, world, geom_kind=geom, coeff_kind=coeff, penalty_scale=w.penalty_scale,
                            jac_fn=jf, device=0, traces=traces, staged=True)
    x = synth.x_torch(w, start=sop.offset, count=sop.ndofs, device="cuda")
    r = torch.full_like(x, float("nan"))
    for _ in range(3):  # repeated applies reuse the buffers, events and streams
        sop.apply(x, r)
    torch.cuda.synchronize()
    parts = [torch.zeros(0, dtype=torch.float64) for _ in range(world)]
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([sop.ndofs]))
    buf = [torch.zeros(int(s.item()), dtype=torch.float64) for s in sizes]
    dist.all_gather(buf, r.cpu())
    if rank == 0:
        q.put((torch.cat(buf).numpy(), sop._apply.traces, sop._apply.payload_doubles, sop.launches_per_apply))
    sop.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("k,N,geom,coeff,traces", [(4, (6, 4, 8), 1, 1, True), (4, (6, 4, 8), 1, 1, False),
                                                   (7, (6, 2, 4), 0, 0, True)])
def test_two_ranks_one_gpu(k, N, geom, coeff, traces):
    import multiprocessing as mp

    import synth
    from paper_1812_08075_b200 import Operator
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, 2, port, k, N, geom, coeff, traces, q)) for rk in range(2)]
    for p in procs:
        p.start()
    got, used_tr, payload, launches = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = synth.small(k, N, geom_kind=geom, coeff_kind=coeff, seed=70 + k)
    op = Operator(w.N, w.k, geom_kind=geom, coeff_kind=coeff, penalty_scale=w.penalty_scale,
                  jac=synth.jac_planes_torch(w, -1, w.N[0] + 2).numpy() if geom else None)
    ref = op.apply(synth.x_torch(w, device="cuda")).cpu().numpy()
    op.close()
    assert used_tr == traces
    n = k + 1
    assert payload == (N[1] * N[2] * 2 * n * n if traces else N[1] * N[2] * n ** 3)
    assert launches == 3 + (1 if traces else 0)
    assert np.array_equal(got, ref), np.abs(got - ref).max() / np.abs(ref).max()
