#!/usr/bin/env python
"""Aggregate warp-stall samples and the executed-opcode mix of one kernel in an ncu report
(`--page source --print-source sass`), optionally per CUDA source line range.

    python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [--lines]
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = Counter()
    S = 0
    ops, ops_s = Counter(), Counter()
    thr = Counter()  # predicated-on thread instructions per opcode (exact lane counts)
    ti = idx.get("Predicated-On Thread Instructions Executed")
    for r in data:
        for s in stalls:
            try:
                tot[s] += int(r[idx[s]])
            except ValueError:
                pass
        try:
            ns = int(r[idx["# Samples"]])
        except ValueError:
            ns = 0
        S += ns
        src = r[idx["Source"]].split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") else src[0]
        op = op.split(".")[0]
        try:
            ops[op] += int(r[idx["Instructions Executed"]])
        except ValueError:
            pass
        if ti is not None:
            try:
                thr[op] += int(r[ti])
            except ValueError:
                pass
        ops_s[op] += ns
    print(f"samples {S}")
    for s, v in tot.most_common(12):
        print(f"  {s:28s} {v:9d} {100 * v / max(S, 1):5.1f}%")
    T = sum(ops.values())
    print(f"warp instructions executed {T}")
    if thr:
        f64 = 2 * thr["DFMA"] + thr["DADD"] + thr["DMUL"]
        print(f"issued FP64 flops (2 DFMA + DADD + DMUL, predicated-on lanes) {f64:.4e}  "
              f"[DFMA {thr['DFMA']:.3e}, DADD {thr['DADD']:.3e}, DMUL {thr['DMUL']:.3e} thread-instructions]")
    for k, v in ops.most_common(22):
        print(f"  {k:10s} {v:12d} {100 * v / T:5.1f}%  samples {ops_s[k]}")


if __name__ == "__main__" and len(sys.argv) == 2:
    main()


def by_line(rep, top=30):
    """Per CUDA source line: samples and the top stall reasons (cuda,sass correlated view)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = []
    fname = ""
    hdr = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 7:
            continue
        try:
            ns = int(r[6])
        except ValueError:
            continue
        st = {}
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    st[h[6:]] = int(r[i])
                except ValueError:
                    pass
        tops = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
        res.append((ns, f"{fname}:{r[0]}", r[1][:70], tops))
    S = sum(x[0] for x in res)
    for ns, loc, src, tops in sorted(res, reverse=True)[:top]:
        print(f"{100 * ns / S:5.1f}% {loc:24s} {src:70s} | {tops}")


if __name__ == "__main__" and "--lines" in sys.argv:
    by_line(sys.argv[1])


def smem_by_line(rep, top=30):
    """Per CUDA source line: shared-memory wavefronts (actual / ideal) and executed instructions."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = []
    fname = ""
    hdr = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        try:
            wf = float(r[hdr.index("L1 Wavefronts Shared")])
            wi = float(r[hdr.index("L1 Wavefronts Shared Ideal")])
            ie = float(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        res.append((wf, wi, ie, f"{fname}:{r[0]}", r[1][:70]))
    T = sum(x[0] for x in res) or 1
    print(f"shared wavefronts total {T:.3e}")
    for wf, wi, ie, loc, src in sorted(res, reverse=True)[:top]:
        print(f"{100 * wf / T:5.1f}% wf {wf:.2e} ideal {wi:.2e} inst {ie:.2e} {loc:24s} {src}")


if __name__ == "__main__" and "--smem" in sys.argv:
    smem_by_line(sys.argv[1])
