#!/usr/bin/env python
"""Summarise ncu evidence for profiles/: a launch list CSV (gpu__time_duration per launch) and/or a
`--set full` report (.ncu-rep) -> markdown table + JSON.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/prof.ncu-rep \
        --out profiles/r01_cfg3 [--alg-bytes B --alg-flops F]
"""
import argparse
import csv
import io
import json
import subprocess
from collections import OrderedDict, defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-inst"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread-inst"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread-inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_static", "static smem/block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1tex throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall barrier"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ui = h.index("Metric Unit")
    agg = defaultdict(list)
    unit = {}
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[vi]:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
            unit[r[ki]] = r[ui]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
    out = []
    tot = 0.0
    for k, v in agg.items():
        us = sum(v) * scale.get(unit[k], 1.0)
        tot += us
        out.append({"kernel": k[:120], "launches": len(v), "total_us": us, "mean_us": us / len(v)})
    for o in out:
        o["share"] = o["total_us"] / tot
    return sorted(out, key=lambda o: -o["total_us"])


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = OrderedDict()
        d["kernel"] = r[h.index("Kernel Name")][:120]
        for k, name in KEYS:
            if k in h:
                d[name] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="")
    args = ap.parse_args()
    js = {"title": args.title}
    md = [f"# {args.title}\n"]
    if args.launches:
        L = launches(args.launches)
        js["launches"] = L
        md.append("## Launch list (ncu gpu__time_duration, --clock-control none; cold, serialised)\n")
        md.append("| kernel | launches | mean us | share |\n|---|---|---|---|")
        for o in L:
            md.append(f"| `{o['kernel'][:90]}` | {o['launches']} | {o['mean_us']:.1f} | {100 * o['share']:.1f}% |")
        md.append("")
    if args.rep:
        F = full(args.rep)
        js["full"] = F
        for d in F:
            md.append(f"## ncu --set full: `{d['kernel'][:90]}`\n")
            md.append("| metric | value |\n|---|---|")
            for k, v in d.items():
                if k != "kernel":
                    md.append(f"| {k} | {v} |")
            md.append("")
    open(args.out + ".md", "w").write("\n".join(md) + "\n")
    json.dump(js, open(args.out + ".json", "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
