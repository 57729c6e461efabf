"""Host<->device copy ceiling for the e2e leg (dg_apply_host): pinned H2D alone, D2H alone, and both at once on two
streams, in chunks like dg_apply_host's. Prints one JSON line (GB/s)."""
import json
import sys

import torch


def main(gb: float = 3.62, nch: int = 32):
    n = int(gb * 1e9) // 8
    h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h_in.fill_(1.0)
    d_a = torch.empty(n, dtype=torch.float64, device="cuda")
    d_b = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    b = [n * i // nch for i in range(nch + 1)]

    def run(h2d: bool, d2h: bool) -> float:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        for i in range(nch):
            if h2d:
                with torch.cuda.stream(s1):
                    d_a[b[i]:b[i + 1]].copy_(h_in[b[i]:b[i + 1]], non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_out[b[i]:b[i + 1]].copy_(d_b[b[i]:b[i + 1]], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    out = {}
    for name, a, c in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
        run(a, c)
        ms = min(run(a, c) for _ in range(3))
        out[name + "_ms"] = ms
        out[name + "_GBps_per_dir"] = n * 8 / ms / 1e6
    out["bytes_per_dir"] = n * 8
    out["chunks"] = nch
    print(json.dumps(out))


if __name__ == "__main__":
    main(*(float(a) for a in sys.argv[1:2]))
