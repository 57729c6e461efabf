"""Summary of a DG_GEN_TRACE dump (tools/trace_gen.py): median cycles per phase of thread 0 (warp 0)."""
import numpy as np
d = np.fromfile("/tmp/dg_gen_trace.bin", dtype=np.int64).reshape(1024, 16, 8)[:296].astype(np.float64)
for s in range(2, 7):
    t = lambda i: d[:, s, i]
    m = lambda a, b: np.median(t(b) - t(a))
    print(f"step {s} total {m(0, 7):7.0f} | top {m(0, 1):6.0f} P1 {m(1, 2):6.0f} stage2 {m(2, 4):6.0f} faces(warp0) {m(4, 5):6.0f} "
          f"barrier {m(5, 3):6.0f} P5a {m(3, 6):6.0f} P5b {m(6, 7):6.0f}")
