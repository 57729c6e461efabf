"""Phase timing of k_gen from clock64 stamps (build with DG_BUILD_FLAGS=-DDG_GEN_TRACE, run with DG_TRACE=path):
per step, cycles in: wait(top barrier) | P1 stage1+traces | lineA(+pointwise) | lineB | lineC | stage3 d0/d1 | d2+store."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1812_08075_b200 import Operator

path = "/tmp/dg_gen_trace.bin"
os.environ["DG_TRACE"] = path
w = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
jac = synth.jac_planes_torch(w, -1, w.N[0] + 2, device="cuda").cpu().numpy() if w.geom_kind else None
op = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, penalty_scale=w.penalty_scale, jac=jac)
x = synth.x_torch(w, device="cuda")
r = torch.empty_like(x)
for _ in range(3):
    op.apply(x, r)
torch.cuda.synchronize()
op.close()
d = np.fromfile(path, dtype=np.int64).reshape(1024, 16, 8)[:296].astype(np.float64)
names = ["top_wait", "P1", "A", "B", "C", "P5a", "P5b"]
for s in range(1, 8):
    seg = [d[:, s, i + 1] - d[:, s, i] for i in range(7)]
    tot = d[:, s, 7] - d[:, s, 0]
    print(f"step {s:2d} total {np.median(tot):8.0f} | " + " ".join(f"{n}={np.median(v):6.0f}" for n, v in zip(names, seg)))
