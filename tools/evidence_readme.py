#!/usr/bin/env python
"""Regenerate profiles/<round>/README.md from the collected bench lines and ncu traffic table."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RND = sys.argv[1] if len(sys.argv) > 1 else "r01"
R = os.path.join(ROOT, "profiles", RND)
T = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
files = [f"bench_cfg{c}_n1.json" for c in range(5)] + ["bench_cfg2_quad7.json", "bench_diffreac_k3_64.json",
                                                        "bench_diffreac_k5_48.json", "bench_nlreac_k3_64.json",
                                                        "bench_nljac_k3_64.json", "bench_stokes_k3_48.json", "bench_stokes_k5_32.json"]
L = ["# Round 1 evidence (B200, 1 GPU)\n",
     "Produced by `tools/round_evidence.sh` on one gpurun box, copied by `tools/collect_evidence.py`, this file by",
     "`tools/evidence_readme.py`. Bench lines: `python bench.py --config C` (timed region = K applies, CUDA events on",
     "the launch stream; L2 flushed between steps when the vectors fit in L2). Roofline per SURVEY §8(d):",
     "T_roof = max(F_alg/P_fp64, B_alg/BW_HBM), P_fp64 = 148 x 64 DFMA/clk x 2 x 1965 MHz = 37.2 TFLOP/s (nominal),",
     "BW_HBM = measured copy bandwidth (MEASURED_PEAKS.json). DRAM traffic = ncu dram read+write of one launch",
     "(`--set full`, caches flushed before the launch); for the affine configs it includes the per-cell setup tables",
     "(geometry records 288 B, c(x) factor tables 96(n+1) B, face c values 8(3n^2 rounded to even) B per cell) that",
     "`B_alg` (x, r and J only) does not count. Rows below the line: SURVEY §8(f2) general quadrature and §8(f1) the",
     "paper's diffusion-reaction problem, §8(f3) its nonlinear variant (residual and Jacobian action, reading R26),",
     "§8(f4) the paper's Stokes problem (correctness-first kernels; F_alg = their contractions as executed; ncu",
     "captures: `ncu_quad_dr3`, `ncu_quad_nljac3`, `ncu_stokes_k3`, stalls in `stalls_*.txt`).\n",
     "| line | workload | ms / apply | GDOF/s | kernel | bound | frac of roofline | frac HBM (alg bytes) | frac of measured DFMA peak | DRAM traffic / alg bytes |",
     "|---|---|---|---|---|---|---|---|---|---|"]
for f in files:
    p = os.path.join(R, f)
    if not os.path.exists(p):
        continue
    d = json.load(open(p))
    rf = d["roofline"]
    wl = d["config"]["workload"]
    tr = rf.get("traffic") or T.get(wl, {}).get(rf["kernel"])
    trs = f"{tr / 1e9:.3f} GB / {rf['alg_bytes_per_launch'] / 1e9:.3f} GB" if tr else "—"
    if f == "bench_cfg2_quad7.json":
        L.append("| | | | | | | | | | |")
    L.append(f"| `{f}` | {wl} | {d['ms_per_step']:.4f} | {d['value'] / 1e9:.1f} | `{rf['kernel']}` | {rf['bound']} | "
             f"{rf['frac']:.3f} | {rf['frac_hbm']:.3f} | {rf['frac_fp64_measured_dfma']:.3f} | {trs} |")
b3 = json.load(open(os.path.join(R, "bench_cfg3_n1.json")))
ref = json.load(open(os.path.join(R, "bench_reference_cfg3.json")))
L.append("")
L.append(f"Default bench line (cfg3): e2e through `dg_apply_host` (pinned host buffers, PCIe in the timed region) = "
         f"{b3['e2e']['value'] / 1e9:.2f} GDOF/s; clocks {b3['clocks']}; CPU oracle on {b3['cpu_baseline']['cores']} host cores = "
         f"{b3['cpu_baseline']['value'] / 1e6:.2f} MDOF/s ({b3['cpu_baseline']['sample']}). Reference arm (`--impl reference`, "
         f"the oracle): {ref['value'] / 1e6:.2f} MDOF/s. cfg3 measured 3.13-3.26 ms across boxes this round.\n")
L.append("Files: `bench_*.json` (bench lines), `bench_reference_cfg3.json`, `launches_cfg{2,3,4}.csv` (ncu launch lists")
L.append("of the timed region, `--profile-from-start off`: one kernel launch per apply, 100% of the step), `ncu_*.md/json`")
L.append("(`--set full` summaries), `stalls_*.txt` (warp-stall samples, opcode mix, per-source-line stalls),")
L.append("`pytest_gpu.txt`, `smoke.txt`, `clocks_bench.csv` (nvidia-smi during the default bench). `history/` holds the")
L.append("first measured version (v1 cell kernel, 16.9 ms on cfg3).")
pdr = os.path.join(R, "bench_diffreac_k3_64.json")
if os.path.exists(pdr):
    sv = json.load(open(pdr)).get("solve")
    if sv:
        L.append("")
        L.append("`bench_diffreac_k3_64.json` also carries `solve`: one CUDA-graph CG iteration driving `dg_apply`")
        L.append(f"(`bench.py --problem diffreac --solve`, SURVEY §8(f3)): {sv['ms_per_iteration']:.2f} ms per iteration "
                 f"at 64^3, k = 3, the apply {100 * sv['apply_share']:.0f} % of it.")
open(os.path.join(R, "README.md"), "w").write("\n".join(L) + "\n")
print("\n".join(L))
