"""Phase timing of k_axis8 from clock64 stamps (DG_TRACE): per step, the cycles spent in
TMA wait, pass d=1 (+barrier), pass d=2 (+barrier), pass d=0 (+barrier)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1812_08075_b200 import Operator

path = "/tmp/dg_trace.bin"
os.environ["DG_TRACE"] = path
w = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
op = Operator(w.N, w.k)
x = synth.x_torch(w, device="cuda")
r = torch.empty_like(x)
for _ in range(3):
    op.apply(x, r)
torch.cuda.synchronize()
op.close()
d = np.fromfile(path, dtype=np.int64).reshape(1024, 16, 8)
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 148
d = d[:nb].astype(np.float64)
names = ["tma_wait", "pass1", "bar1", "pass2", "bar2", "pass0", "bar0", "next"]
for s in range(1, 12):
    seg = [d[:, s, i + 1] - d[:, s, i] for i in range(7)]
    seg.append(d[:, s + 1, 0] - d[:, s, 7] if s < 15 else d[:, s, 7] * 0)
    tot = d[:, s + 1, 0] - d[:, s, 0]
    print(f"step {s:2d} total {np.median(tot):8.0f} | " + " ".join(f"{n}={np.median(v):6.0f}" for n, v in zip(names, seg)))
