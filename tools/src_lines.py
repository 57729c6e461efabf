#!/usr/bin/env python
"""Per-source-line shared-memory wavefronts of an ncu source export (tools/prof_gen.sh), development tool.

    python tools/src_lines.py gpurun_out/prof_g1/source.csv.gz DOFS [file] [first-last ...]
"""
import csv
import gzip
import io
import sys


def load(path):
    rows, hdr, fname = [], None, ""
    for r in csv.reader(io.TextIOWrapper(gzip.open(path))):
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        d["file"] = fname
        rows.append(d)
    return rows


def f(d, k):
    try:
        return float(d.get(k, "0") or 0)
    except ValueError:
        return 0.0


if __name__ == "__main__":
    rows = load(sys.argv[1])
    dof = float(sys.argv[2])
    fn = sys.argv[3] if len(sys.argv) > 3 else "kernel_gen.cuh"
    rngs = [tuple(map(int, a.split("-"))) for a in sys.argv[4:]]
    T = sum(f(d, "L1 Wavefronts Shared") for d in rows)
    I = sum(f(d, "L1 Wavefronts Shared Ideal") for d in rows)
    S = sum(f(d, "# Samples") for d in rows)
    print(f"total wf/DOF {T / dof:.3f} (ideal {I / dof:.3f}), inst/DOF {sum(f(d, 'Instructions Executed') for d in rows) / dof:.2f}")
    for d in rows:
        if d["file"] != fn:
            continue
        ln = int(d["Line No"])
        if rngs and not any(a <= ln <= b for a, b in rngs):
            continue
        wf = f(d, "L1 Wavefronts Shared")
        if wf == 0 and not rngs:
            continue
        print(f"{ln:5d} wf/DOF {wf / dof:.3f} ideal {f(d, 'L1 Wavefronts Shared Ideal') / dof:.3f} "
              f"inst/DOF {f(d, 'Instructions Executed') / dof:.3f} samples {100 * f(d, '# Samples') / S:4.1f}%")
