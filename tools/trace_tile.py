"""Phase timing of k_tile from clock64 stamps (DG_TRACE): cycles between consecutive barriers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1812_08075_b200 import Operator

path = "/tmp/dg_trace_tile.bin"
os.environ["DG_TRACE"] = path
w = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
jac = synth.jac_planes_torch(w, -1, w.N[0] + 2, device="cuda").cpu().numpy() if w.geom_kind else None
op = Operator(w.N, w.k, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind, jac=jac)
x = synth.x_torch(w, device="cuda")
r = torch.empty_like(x)
op.apply(x, r)
torch.cuda.synchronize()
op.close()
d = np.fromfile(path, dtype=np.int64).reshape(1024, 8, 32)[:148].astype(np.float64)
nph = int((d[0, 2] > 0).sum())
for s in range(2, 6):
    dd = np.diff(d[:, s, :nph], axis=1)
    print(f"step {s}: total {np.median(d[:, s + 1, 0] - d[:, s, 0]):8.0f} | " + " ".join(f"{np.median(dd[:, i]):6.0f}" for i in range(nph - 1)))
