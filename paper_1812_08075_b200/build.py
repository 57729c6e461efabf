"""Build libdg.so in-tree with nvcc for sm_100a (B200). No JIT, no torch extension cache:
the .so lives at paper_1812_08075_b200/lib/libdg.so and travels with the repo snapshot."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.environ.get("DG_LIB_OUT") or os.path.join(LIBDIR, "libdg.so")  # DG_LIB_OUT: experiment variants only
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["dg_capi.cu", "tables.cpp", "fp64_peak.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-ldl"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "dg.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    extra = os.environ.get("DG_BUILD_FLAGS", "").split()  # experiments only (e.g. -DDG_AX8_TRACE)
    cmd = [NVCC] + ARCH + FLAGS + extra + ["-o", LIB] + [os.path.join(CSRC, s) for s in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = LIB + ".build.log" if os.environ.get("DG_LIB_OUT") else os.path.join(LIBDIR, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-20000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(res.stderr)
    return LIB


if __name__ == "__main__":
    if "--bounds" in sys.argv:
        # bounds-checked debug library (-DDG_BOUNDS) next to the release one; select it with DG_LIB
        os.environ["DG_BUILD_FLAGS"] = (os.environ.get("DG_BUILD_FLAGS", "") + " -DDG_BOUNDS").strip()
        os.environ.setdefault("DG_LIB_OUT", os.path.join(LIBDIR, "libdg_bounds.so"))
        LIB = os.environ["DG_LIB_OUT"]
    print(build(force="--force" in sys.argv or "--bounds" in sys.argv, verbose="-v" in sys.argv))
