#!/usr/bin/env python
"""Per-(workload, kernel) ncu counters for bench.py's roofline keys: one `ncu --set full` report per entry
-> profiles/<round>/ncu_counters.json (merged).

    python tools/ncu_counters.py OUT.json workload:kernel:report.ncu-rep [...]

Stored per entry (per launch): dram_bytes (dram__bytes_read.sum + dram__bytes_write.sum), fp64_flops_issued
(2 x DFMA + DADD + DMUL predicated-on thread instructions), duration_ms, fp64_pipe_pct, l1tex_pct, dram_pct,
warps_active_pct, registers."""
import csv
import io
import json
import os
import subprocess
import sys


def sass_fp64(rep):
    """Predicated-on thread instructions of DFMA, DADD, DMUL summed over the SASS of the source page (the raw page
    of `--set full` carries no per-opcode FP64 counters)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1] if len(rows) > 1 else []
    idx = {h: i for i, h in enumerate(hdr)}
    ti = idx.get("Predicated-On Thread Instructions Executed")
    tot = {"DFMA": 0.0, "DADD": 0.0, "DMUL": 0.0}
    if ti is None or "Source" not in idx:
        return 0.0, 0.0, 0.0
    for r in rows[2:]:
        src = r[idx["Source"]].split() if len(r) > idx["Source"] else []
        if not src:
            continue
        op = (src[1] if src[0].startswith("@") and len(src) > 1 else src[0]).split(".")[0]
        if op in tot:
            try:
                tot[op] += float(r[ti])
            except ValueError:
                pass
    return tot["DFMA"], tot["DADD"], tot["DMUL"]


def metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]

    def get(k, scale=None):
        if k not in h:
            return None
        s = v[h.index(k)].replace(",", "")
        try:
            x = float(s)
        except ValueError:
            return None
        unit = u[h.index(k)]
        if scale == "bytes":
            x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
        if scale == "ms":
            x *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                  "second": 1e3, "s": 1e3}.get(unit, 1)
        return x

    dfma, dadd, dmul = sass_fp64(rep)
    rd, wr = get("dram__bytes_read.sum", "bytes"), get("dram__bytes_write.sum", "bytes")
    return {"dram_bytes": (rd or 0) + (wr or 0), "dram_read_bytes": rd, "dram_write_bytes": wr,
            "fp64_flops_issued": 2 * dfma + dadd + dmul,
            "duration_ms": get("gpu__time_duration.sum", "ms"),
            "fp64_pipe_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "l1tex_pct": get("l1tex__throughput.avg.pct_of_peak_sustained_active"),
            "dram_pct": get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers": get("launch__registers_per_thread"),
            "smem_wavefronts": get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "smem_bank_conflicts": get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")}


def main():
    out = sys.argv[1]
    d = json.load(open(out)) if os.path.exists(out) else {}
    for spec in sys.argv[2:]:
        wl, kern, rep = spec.split(":", 2)
        if not os.path.exists(rep):
            print("missing", rep)
            continue
        d.setdefault(wl, {})[kern] = metrics(rep)
        print(wl, kern, d[wl][kern])
    json.dump(d, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
