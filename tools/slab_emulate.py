#!/usr/bin/env python
"""Per-rank time of the x0-slab decomposition, emulated on ONE GPU (no multi-GPU node in this run): for each rank q
of P, its slab context runs exactly what dg_apply_dist runs on that rank — dg_pack_halo, the interior planes, the two
boundary planes with trace halos (here produced by the neighbours' dg_pack_halo on the same GPU, i.e. without the
NCCL transfer) — timed with CUDA events, ranks one after another. Reports the max over ranks against the whole-mesh
apply / P (the ideal), and the payload per message. Checks the assembled slabs against the whole-mesh apply.

    python tools/slab_emulate.py --config 4 --P 8
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--P", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--R", type=int, default=5)
    a = ap.parse_args()
    import torch

    import synth
    from paper_1812_08075_b200 import Operator, slab
    w = synth.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    x = synth.x_torch(w, device=dev)
    jf = (lambda pb, npl: synth.jac_planes_torch(w, pb, npl, device=dev).cpu().numpy()) if w.geom_kind else None
    whole = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale,
                     jac=jf(-1, w.N[0] + 2) if jf else None)
    r_ref = whole.apply(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timeit(fn):
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.R):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.R

    t_whole = timeit(lambda: whole.apply(x, r_ref))
    whole.close()
    out = {"workload": w.name, "kernel": None, "whole_ms": t_whole, "P": {}}
    for P in a.P:
        ops, lo, hi, xs = [], [], [], []
        for q in range(P):
            pl = slab.plan(w.N[0], q, P)
            op = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale,
                          jac=jf(pl.plane_begin - 1, pl.nplanes + 2) if jf else None, plane_begin=pl.plane_begin,
                          nplanes=pl.nplanes)
            ops.append(op)
            xs.append(x[op.offset:op.offset + op.ndofs])
            lo.append(torch.empty(op.halo_ndofs, dtype=torch.float64, device=dev))
            hi.append(torch.empty(op.halo_ndofs, dtype=torch.float64, device=dev))
            op.pack_halo(xs[q], lo[q], hi[q])
        out["kernel"] = ops[0].kernel_name
        rs = [torch.empty_like(v) for v in xs]
        per = []
        for q, op in enumerate(ops):
            L = op.nplanes
            below, above = hi[(q - 1) % P], lo[(q + 1) % P]

            def rank_step(q=q, op=op, L=L, below=below, above=above):
                op.pack_halo(xs[q], lo[q], hi[q])
                if L > 2:
                    op.apply_planes_tr(xs[q], below, above, rs[q], 1, L - 1)
                    op.apply_planes_tr(xs[q], below, above, rs[q], 0, 1)
                    op.apply_planes_tr(xs[q], below, above, rs[q], L - 1, L)
                else:
                    op.apply_planes_tr(xs[q], below, above, rs[q], 0, L)
            per.append(timeit(rank_step))
        ok = bool(torch.equal(torch.cat(rs), r_ref))
        pmax = max(per)
        out["P"][P] = {"rank_ms_max": pmax, "rank_ms": per, "ideal_ms": t_whole / P,
                       "compute_efficiency": t_whole / (P * pmax), "bitwise_equal_whole": ok,
                       "message_MB": 8 * ops[0].halo_ndofs / 1e6}
        for op in ops:
            op.close()
        del rs, lo, hi
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
