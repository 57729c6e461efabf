#!/usr/bin/env python
"""Shared-memory wavefronts (actual, excess over ideal) and executed instructions of one ncu report,
aggregated over CUDA source line ranges given as name:file:first-last (development tool).

    python tools/ncu_smem_regions.py rep.ncu-rep "stage1:kernel_gen.cuh:909-945" ...
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    regs = []
    for spec in sys.argv[2:]:
        name, f, rng = spec.split(":")
        a, b = rng.split("-")
        regs.append((name, f, int(a), int(b)))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    hdr, fname = None, ""
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0].isdigit():
            continue
        try:
            wf = float(r[hdr.index("L1 Wavefronts Shared")])
            wi = float(r[hdr.index("L1 Wavefronts Shared Ideal")])
            ie = float(r[hdr.index("Instructions Executed")])
            ns = float(r[hdr.index("# Samples")])
        except (ValueError, IndexError):
            continue
        line = int(r[0])
        key = f"{fname}:other"
        for name, f, a, b in regs:
            if f == fname and a <= line <= b:
                key = name
                break
        v = agg[key]
        v[0] += wf
        v[1] += wi
        v[2] += ie
        v[3] += ns
    T = sum(v[0] for v in agg.values()) or 1
    I = sum(v[2] for v in agg.values()) or 1
    S = sum(v[3] for v in agg.values()) or 1
    print(f"total shared wavefronts {T:.3e}, instructions {I:.3e}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:34s} wf {100 * v[0] / T:5.1f}%  excess {100 * (v[0] - v[1]) / T:5.1f}%  inst {100 * v[2] / I:5.1f}%  "
              f"samples {100 * v[3] / S:5.1f}%")


if __name__ == "__main__":
    main()
