"""The collective C-ABI (include/dg.h dg_setup_dist / dg_apply_dist): a library-owned NCCL
communicator, one point-to-point halo step per application overlapped with the interior planes. With one rank the
step is an NCCL send / receive to itself (the wrap planes), so the full collective code path — NCCL communicator,
comm stream, events, trace packing, the three plane launches — runs on a single GPU and must reproduce dg_apply bit
for bit. (Two ranks on one GPU are not possible with NCCL; tests/test_gpu_slab_2proc.py covers two processes with
the torch.distributed form.)
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = [
    # (w, kernel, trace payload)
    (synth.small(4, (6, 4, 8), geom_kind=1, coeff_kind=1, seed=81), "k_gen", True),
    (synth.small(7, (6, 2, 4), seed=82), "k_axis8", True),
    (synth.small(3, (6, 5, 7), seed=83), "k_line", True),
    (synth.small(2, (5, 3, 4), geom_kind=1, coeff_kind=1, seed=84, quad=4), "k_quad", False),
    (synth.small(2, (2, 4, 8), geom_kind=1, coeff_kind=1, seed=85), "k_gen", True),  # L = 2: one launch after the exchange
]


@pytest.mark.parametrize("w,kern,tr", CASES, ids=lambda v: getattr(v, "name", str(v)))
def test_dist_single_rank_loopback(w, kern, tr):
    from paper_1812_08075_b200 import Operator, dg
    jac = synth.jac_planes_torch(w, -1, w.N[0] + 2).numpy() if w.geom_kind else None
    ref_op = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale, jac=jac,
                      quad=w.m)
    uid = dg.dg_get_unique_id()
    op = dg.DistOperator(w.N, w.k, 0, 1, uid, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind,
                         penalty_scale=w.penalty_scale, jac=jac, quad=w.m)
    assert op.kernel_name == kern == ref_op.kernel_name
    L = w.N[0]
    assert op.launches_per_apply == (3 if L > 2 else 1) + (1 if tr else 0)
    x = synth.x_torch(w, device="cuda")
    ref = ref_op.apply(x)
    for _ in range(3):  # repeated collective applies reuse the communicator, buffers and events
        r = torch.full_like(x, float("nan"))
        op.apply(x, r)
        torch.cuda.synchronize()
        assert torch.equal(r, ref)
    jac_all = synth.jac_cells_np(w, np.arange(w.ncells)) if w.geom_kind else None
    orc = oracle.apply(w, x.cpu().numpy(), jac_all)
    assert np.abs(r.cpu().numpy() - orc).max() / np.abs(orc).max() <= 1e-11
    op.close()
    ref_op.close()


def test_dist_rejects_mismatched_slab():
    from paper_1812_08075_b200 import dg
    from paper_1812_08075_b200.dg import DgError
    uid = dg.dg_get_unique_id()
    assert len(uid) == 128
    with pytest.raises(DgError):
        dg.dg_setup_dist((4, 4, 4), 2, 3, 1, 1, uid)  # rank out of range
