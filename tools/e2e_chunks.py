#!/usr/bin/env python
"""dg_apply_host timing against the host-pipeline chunk count (development): python tools/e2e_chunks.py CFG"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import synth
    from paper_1812_08075_b200 import Operator
    w = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
    jac = synth.jac_planes_torch(w, -1, w.N[0] + 2).numpy() if w.geom_kind == 1 else None
    op = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale, jac=jac)
    xh = synth.x_torch(w, device="cpu").pin_memory()
    rh = torch.empty_like(xh).pin_memory()
    for _ in range(2):
        op.apply_host(xh, rh)
    R = 5
    t0 = time.perf_counter()
    for _ in range(R):
        op.apply_host(xh, rh)
    dt = (time.perf_counter() - t0) / R
    print(f"{w.name} chunks={os.environ.get('DG_HOST_CHUNKS', 'default')}: {dt * 1e3:.2f} ms per apply_host, "
          f"{w.ndofs / dt / 1e9:.2f} GDOF/s, {2 * 8 * w.ndofs / dt / 1e9:.1f} GB/s over PCIe (both directions)")


if __name__ == "__main__":
    main()
