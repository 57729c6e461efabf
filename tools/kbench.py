#!/usr/bin/env python
"""Quick kernel timing for development (not the bench contract): r = A x on a synthetic mesh,
CUDA events over R back-to-back applies after warm-up.

    python tools/kbench.py --k 4 --N 128 --geom 1 --coeff 1 [--R 20] [--parity]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--N", type=int, nargs="+", default=[128])
    ap.add_argument("--geom", type=int, default=1)
    ap.add_argument("--coeff", type=int, default=1)
    ap.add_argument("--R", type=int, default=20)
    ap.add_argument("--parity", action="store_true", help="also check a small mesh against the oracle")
    ap.add_argument("--graph", action="store_true", help="replay the R applies from one CUDA graph")
    a = ap.parse_args()
    import numpy as np
    import torch

    import synth
    from paper_1812_08075_b200 import Operator
    N = tuple(a.N) if len(a.N) == 3 else (a.N[0],) * 3
    w = synth.small(a.k, N, geom_kind=a.geom, coeff_kind=a.coeff, seed=9)
    jac = synth.jac_planes_torch(w, -1, w.N[0] + 2, device="cuda").cpu().numpy() if a.geom else None
    op = Operator(w.N, w.k, geom_kind=a.geom, coeff_kind=a.coeff, jac=jac)
    x = synth.x_torch(w, device="cuda")
    r = torch.empty_like(x)
    for _ in range(3):
        op.apply(x, r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.graph:
        gs = torch.cuda.Stream()
        with torch.cuda.stream(gs):
            op.set_stream(gs)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=gs):
                for _ in range(a.R):
                    op.apply(x, r)
        op.set_stream(torch.cuda.current_stream())
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
    else:
        e0.record()
        for _ in range(a.R):
            op.apply(x, r)
        e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.R
    F = op.alg_flops
    frac = F / (ms * 1e-3) / 37.22496e12
    print(f"{op.kernel_name} k={a.k} N={N} geom={a.geom} coeff={a.coeff}: {ms:.4f} ms  {w.ndofs / ms / 1e6:.1f} GDOF/s"
          f"  frac(F_alg) {frac:.3f}")
    if a.parity:
        import oracle
        for Nn in ((4, 4, 8), (3, 4, 8), (6, 8, 8)):
            ws = synth.small(a.k, Nn, geom_kind=a.geom, coeff_kind=a.coeff, seed=11)
            jacs = synth.jac_planes_torch(ws, -1, ws.N[0] + 2).numpy() if a.geom else None
            ops = Operator(ws.N, ws.k, geom_kind=a.geom, coeff_kind=a.coeff, jac=jacs)
            xs = synth.x_torch(ws, device="cuda")
            rs = ops.apply(xs).cpu().numpy()
            ja = synth.jac_cells_np(ws, np.arange(ws.ncells)) if a.geom else None
            ref = oracle.apply(ws, xs.cpu().numpy(), ja)
            print(f"  parity {Nn} ({ops.kernel_name}): {np.abs(rs - ref).max() / np.abs(ref).max():.2e}")
            ops.close()


if __name__ == "__main__":
    main()
