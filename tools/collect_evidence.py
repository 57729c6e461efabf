#!/usr/bin/env python
"""Copy a round_evidence.sh run (gpurun_out/ev) into profiles/<round>/ and refresh
profiles/ncu_traffic.json (DRAM bytes per launch of each hot kernel, from the --set full captures)."""
import glob
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "ev")
RND = sys.argv[1] if len(sys.argv) > 1 else "r01"
DST = os.path.join(ROOT, "profiles", RND)
os.makedirs(DST, exist_ok=True)

cp = {"bench.json": "bench_cfg3_n1.json", "bench_ref.json": "bench_reference_cfg3.json",
      "pytest_gpu.log": "pytest_gpu.txt", "smoke.log": "smoke.txt", "clocks.csv": "clocks_bench.csv"}
for c in (0, 1, 2, 4):
    cp[f"bench_cfg{c}.json"] = f"bench_cfg{c}_n1.json"
for f in ("bench_cfg2_quad7.json", "bench_diffreac_k3_64.json", "bench_diffreac_k5_48.json", "bench_nlreac_k3_64.json",
          "bench_nljac_k3_64.json", "bench_stokes_k3_48.json", "bench_stokes_k5_32.json"):
    cp[f] = f
for f in glob.glob(os.path.join(SRC, "ncu_*.md")) + glob.glob(os.path.join(SRC, "ncu_*.json")) + \
        glob.glob(os.path.join(SRC, "stalls_*.txt")) + glob.glob(os.path.join(SRC, "launches_*.csv")):
    cp[os.path.basename(f)] = os.path.basename(f)
n = 0
for a, b in cp.items():
    if os.path.exists(os.path.join(SRC, a)):
        shutil.copy(os.path.join(SRC, a), os.path.join(DST, b))
        n += 1

WORK = {"axis8_cfg3": "cfg3_poisson_q7_96", "gen_cfg1": "cfg1_poisson_q3_32", "gen_cfg2": "cfg2_diffusion_q5_64_affine",
        "gen_cfg4": "cfg4_diffusion_q4_256_affine",
        # (workload, the kernel name dg_kernel_name reports)
        "quad_dr3": ("diffreac_k3_N64x64x64_m5", "k_quad_diffreac"), "stokes_k3": ("stokes_k3_N48x48x48", "k_stokes")}
tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
traffic = json.load(open(tp)) if os.path.exists(tp) else {}
unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(s):
    v, u = s.split()
    return float(v.replace(",", "")) * unit[u]


for key, wl in WORK.items():
    path = os.path.join(SRC, f"ncu_{key}.json")
    if not os.path.exists(path):
        continue
    kname = None
    if isinstance(wl, tuple):
        wl, kname = wl
    for d in json.load(open(path)).get("full", []):
        m = re.match(r"void (k_\w+)", d["kernel"])
        if m:
            traffic.setdefault(wl, {})[kname or m.group(1)] = val(d["DRAM read"]) + val(d["DRAM write"])
json.dump(traffic, open(tp, "w"), indent=1)
print("copied", n, "files ->", DST)
print(json.dumps(traffic, indent=1))
