#!/usr/bin/env python
"""Benchmark: DOF/s per SIPG-DG residual evaluation (fp64) on B200, 1-8 GPUs, with roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N ...

One "step" = one application r = A x of the whole hot path (volume + all faces + halo
exchange for N > 1) over the workload of BASELINE.json config C (default 3: Poisson Q7 on 96^3
periodic cells, 453M DOFs, the configuration BASELINE.json defines for 1/2/4/8 GPUs; N > 1
splits the same mesh into x0-slabs: strong scaling). Prints ONE JSON line on rank 0.

`--impl reference` times the CPU oracle (the slow plain definition) on the host cores instead,
on a bounded sample of the same workload per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DOF/s per DG residual evaluation (fp64)"
UNIT = "DOF/s"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)), "src": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "src": "fallback"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and clock-event reasons through NVML in a thread during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.01):
        self.samples = []
        self.reasons = 0
        self.ok = False
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _reasons(self):
        nv = self.nv
        for fn in ("nvmlDeviceGetCurrentClocksEventReasons", "nvmlDeviceGetCurrentClocksThrottleReasons"):
            if hasattr(nv, fn):
                try:
                    return getattr(nv, fn)(self.h)
                except Exception:
                    pass
        return 0

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self._reasons())
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"], "samples": 0}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU oracle timing
def oracle_sample_rate(w, budget_s: float, seed: int = 2024, jacobian: bool = False):
    """Time the oracle (as it stands) on a deterministic random sample of cells of workload w,
    sized to roughly budget_s seconds of host CPU work. Returns (DOF/s, cells, seconds, threads)."""
    import numpy as np

    import oracle
    import synth
    rng = np.random.default_rng(seed)
    n3 = w.block

    def run(ncell):
        cells = np.sort(rng.choice(w.ncells, ncell, replace=False)).astype(np.int64)
        if w.problem in (1, 2, 3):  # the paper's problems: the oracle on the whole host vector, sampled rows
            x = synth.x_np(w)
            t0 = time.perf_counter()
            if w.problem == 3:
                oracle.apply_stokes(w, x, cells)
            elif w.problem == 1:
                oracle.apply_diffreac(w, x, cells)
            elif jacobian:
                oracle.apply_nlreac(w, x, u0=np.sin(x), cells=cells)
            else:
                oracle.apply_nlreac(w, x, cells=cells)
            return time.perf_counter() - t0
        nb = oracle.neighbours(w, cells)
        x7 = synth.x_cells_np(w, nb.reshape(-1)).reshape(len(cells), 7, n3)
        j7 = synth.jac_cells_np(w, nb.reshape(-1)).reshape(len(cells), 7, 9) if w.geom_kind else None
        t0 = time.perf_counter()
        oracle.apply_cells_local(w, cells, x7, j7)
        return time.perf_counter() - t0

    th = oracle.num_threads()
    ncell = max(th, 8)
    t = run(ncell)
    while t < 0.2 * budget_s and ncell < w.ncells:      # grow the probe until it costs ~20% of the budget
        ncell = min(w.ncells, ncell * 4)
        t = run(ncell)
    target = int(min(w.ncells, max(ncell, ncell * budget_s / max(t, 1e-9))))
    if target > ncell * 1.2:
        ncell = target
        t = run(ncell)
    return ncell * n3 / t, ncell, t, th


def run_reference(args, w, rank):
    """--impl reference: the oracle on the host cores, rank 0 only."""
    if rank != 0:
        return 0
    budget = max(0.5, min(5.0, 150.0 / (args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample_rate(w, budget, jacobian=args.jacobian)
    rates, cells, secs = [], 0, 0.0
    th = 1
    for _ in range(args.steps):
        v, c, t, th = oracle_sample_rate(w, budget, jacobian=args.jacobian)
        rates.append(v)
        cells, secs = c, t
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": w.ndofs / value * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(w, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": th, "kind": "oracle",
                         "sample": f"{cells} random cells ({cells * w.block} DOFs) of {w.name} per step, "
                                   f"~{secs:.1f} s each; ms_per_step extrapolated to the whole mesh"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(w, ngpu):
    return {"workload": w.name, "mesh": list(w.N), "k": w.k, "quad_points": w.m, "dofs": w.ndofs,
            "geometry": "axis-aligned" if w.geom_kind == 0 else "per-cell affine",
            "coefficient": "1" if w.coeff_kind == 0 else "1+0.5sin(2pi x0)cos(2pi x1)",
            "penalty": (f"{w.penalty_scale:g}*k(k+1)/h" if w.problem == 0 else f"alpha={w.penalty_scale:g}: alpha*k(k+2)|F|/|T|"),
            "problem": ("periodic SIPG (configs)", "diffusion-reaction, Dirichlet g=|x|^2 (P:L945-1003)",
                        "nonlinear diffusion-reaction c u^2 (R26), Dirichlet g=|x|^2",
                        "Stokes Q_k/Q_{k-1}, mu=1, Dirichlet g=(4x_1(1-x_1),0,0) / Neumann x_0=1 (P:L1077-1118)")[w.problem],
            "parallelism": f"x0-slab{ngpu}",
            "l2": f"inputs larger than L2 ({8 * w.ndofs / 1e9:.2f} GB per vector vs 126 MB L2)"
            if 8 * w.ndofs > 2 * 126e6 else "L2 flushed between steps"}


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--problem", default="config", choices=["config", "diffreac", "nlreac", "stokes"],
                    help="diffreac: the paper's diffusion-reaction problem (SURVEY §8(f1)) with --k / --N, k+2 points; "
                         "nlreac: its nonlinear variant (SURVEY §8(f3), R26); stokes: the paper's Stokes problem "
                         "(SURVEY §8(f4), R27)")
    ap.add_argument("--solve", action="store_true",
                    help="diffreac, N=1: also time the CUDA-graph CG iteration driving dg_apply (SURVEY §8(f3)); "
                         "reported under 'solve' next to the operator line")
    ap.add_argument("--jacobian", action="store_true",
                    help="nlreac: time the Jacobian action J(u0) z (dg_apply_jacobian) instead of the residual")
    ap.add_argument("--k", type=int, default=3)
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--quad", type=int, default=-1,
                    help="Gauss points per direction (default k+1; k+2 = overintegration, SURVEY §8(f2))")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps

    import synth
    w = synth.CONFIGS[args.config]
    if args.problem == "diffreac":
        w = synth.diffreac(args.k, args.N, quad=args.k + 2)
    if args.problem == "nlreac":
        w = synth.nlreac(args.k, args.N)
    if args.problem == "stokes":
        w = synth.stokes(args.k, args.N)
    if args.jacobian and w.problem != 2:
        raise SystemExit("--jacobian needs --problem nlreac")
    if args.quad > 0 and args.quad != w.k + 1:
        import dataclasses
        w = dataclasses.replace(w, quad=args.quad, name=f"{w.name}_quad{args.quad}")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, w, rank)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1812_08075_b200 import dg, slab
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    stream = torch.cuda.current_stream(dev)

    def jac_fn(pb, npl):
        return synth.jac_planes_torch(w, pb, npl, device=dev).cpu().numpy()

    sop = slab.SlabOperator(w.N, w.k, rank, world, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind,
                            penalty_scale=w.penalty_scale, jac_fn=jac_fn, device=local_rank, quad=w.m,
                            problem=w.problem)
    op = sop.op
    x = synth.x_torch(w, start=sop.offset, count=sop.ndofs, device=dev)
    r = torch.empty_like(x)
    u0 = torch.sin(x) if args.jacobian else None  # linearization point (same distribution scale as x)

    def step(xin, rout):
        if args.jacobian:
            sop.apply_jacobian(u0, xin, rout)
        else:
            sop.apply(xin, rout)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up
    for _ in range(args.warmup):
        step(x, r)
    barrier()

    # ---- timed region: K steps, events on the launching stream; per-step event pairs give the
    #      kernel's average duration (N = 1: one launch per step, so step == kernel)
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local_rank)
    barrier()
    flush = None
    if 8 * sop.ndofs * 2 < 4 * 126e6:
        # vectors fit in L2: flush it between timed steps (write 512 MB), time the steps alone
        flush = torch.empty(64 << 20, dtype=torch.float64, device=dev)
    with clk:
        # the timed region is the profiled range: `ncu --profile-from-start off` lists exactly its launches
        torch.cuda.profiler.start()
        t_start.record(stream)
        for i in range(K):
            if flush is not None:
                flush.fill_(float(i))
            ev[i][0].record(stream)
            step(x, r)
            ev[i][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    warm_ms = None
    if flush is not None:
        # L2-resident vectors: also the warm number (no flush between applies; SURVEY §8(d) timing protocol)
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        w0.record(stream)
        for _ in range(K):
            step(x, r)
        w1.record(stream)
        torch.cuda.synchronize()
        warm_ms = w0.elapsed_time(w1) / K
    total_ms = t_start.elapsed_time(t_end) if flush is None else sum(step_ms)
    t_local = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms = t_local.item()
    ms_per_step = total_ms / K
    value = w.ndofs / (ms_per_step * 1e-3)

    # ---- roofline of the dominant kernel (per launch, this rank)
    pk = _peaks()
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    fp64_nominal = sms * 64 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12  # TFLOP/s: SMs x 64 DFMA/clk x 2 flop x clock
    fp64_meas, _ = dg.dg_bench_fp64(local_rank, 4000)
    kern_ms = statistics.mean(step_ms)
    F = op.alg_flops
    if args.jacobian:
        # J(u0) z: + u0 at the m^3 points (2 (n^3 m + n^2 m^2 + n m^3) per cell), reaction 2 c u0 z without f
        # (6 flops per point fewer than the residual's c u^2 - f(x)); DESIGN.md §5
        nn, mm = w.n, w.m
        F += (2.0 * (nn ** 3 * mm + nn ** 2 * mm ** 2 + nn * mm ** 3) - 6.0 * mm ** 3) * (sop.ndofs / nn ** 3)
    B = op.alg_bytes
    t_flop = F / (fp64_nominal * 1e12)
    t_byte = B / (pk["hbm_gbs"] * 1e9)
    ach_tf = F / (kern_ms * 1e-3) / 1e12
    ach_gbs = B / (kern_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(w.name, {}).get(op.kernel_name)
        except Exception:
            traffic = None
    if t_flop >= t_byte:
        roof = {"bound": "alu", "achieved": ach_tf, "peak": fp64_nominal, "unit": "TFLOP/s",
                "frac": ach_tf / fp64_nominal, "traffic": traffic,
                "peak_src": f"derived: {sms} SMs x 64 DFMA/clk x 2 x {pk['sm_max_mhz']:.0f} MHz (DESIGN.md §5)"}
    else:
        roof = {"bound": "hbm", "achieved": ach_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": ach_gbs / pk["hbm_gbs"], "traffic": traffic, "peak_src": f"{pk['src']} copy bandwidth"}
    roof.update({"kernel": op.kernel_name, "kernel_ms": kern_ms, "alg_flops_per_launch": F,
                 "alg_bytes_per_launch": B, "frac_fp64": ach_tf / fp64_nominal,
                 "frac_fp64_measured_dfma": ach_tf / fp64_meas, "fp64_dfma_measured_tflops": fp64_meas,
                 "frac_hbm": ach_gbs / pk["hbm_gbs"], "t_roof_ms": max(t_flop, t_byte) * 1e3,
                 "frac_roof": max(t_flop, t_byte) * 1e3 / kern_ms})

    # ---- e2e: same metric through the public API with host buffers (pinned), copies timed
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        rh = torch.empty_like(xh).pin_memory()
        KE = max(1, args.e2e_steps)
        uh = u0.cpu().pin_memory() if args.jacobian else None
        if world == 1 and not args.jacobian:
            op.apply_host(xh, rh)  # warm-up (allocates staging buffers)
            barrier()
            t0 = time.perf_counter()
            for _ in range(KE):
                op.apply_host(xh, rh)
            te = time.perf_counter() - t0
        else:
            xd = torch.empty_like(x)
            rd = torch.empty_like(x)

            ud = torch.empty_like(x) if args.jacobian else None

            def host_step():
                xd.copy_(xh, non_blocking=True)
                if args.jacobian:
                    ud.copy_(uh, non_blocking=True)
                    sop.apply_jacobian(ud, xd, rd)
                else:
                    sop.apply(xd, rd)
                rh.copy_(rd, non_blocking=True)
                torch.cuda.synchronize()
            host_step()
            barrier()
            t0 = time.perf_counter()
            for _ in range(KE):
                host_step()
            te = time.perf_counter() - t0
            if world > 1:
                tt = torch.tensor([te], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                te = tt.item()
        e2e = {"value": w.ndofs / (te / KE), "unit": UNIT,
               "h2d_bytes_per_step": (16 if args.jacobian else 8) * w.ndofs,
               "d2h_bytes_per_step": 8 * w.ndofs, "steps": KE,
               "how": "pinned H2D of u0 and z, dg_apply_jacobian, D2H of r" if args.jacobian else
               ("dg_apply_host (pinned host x -> H2D -> kernels -> D2H r, plane-chunk pipelined)"
                if world == 1 else "per rank: pinned H2D of the slab, halo exchange + kernels, D2H of r")}
        del xh, rh, uh

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        v, cells, secs, th = oracle_sample_rate(w, args.cpu_seconds, jacobian=args.jacobian)
        cpu = {"value": v, "unit": UNIT, "cores": th, "kind": "oracle",
               "sample": f"{cells} random cells ({cells * w.block} DOFs) of {w.name}, {secs:.1f} s"}

    # ---- sanity of the timed result (not a parity claim: tests/ do that): finite, nonzero
    ok = bool(torch.isfinite(r).all().item()) and r.abs().max().item() > 0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": _config(w, world), "roofline": roof,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": K * sop.launches_per_apply,
        "clocks": clk.summary(), "result_finite": ok,
        "step_ms": {"median": statistics.median(step_ms), "min": min(step_ms), "max": max(step_ms)},
        "warm_ms_per_step": warm_ms,
    }
    if args.solve and world == 1 and w.problem == 1:
        from paper_1812_08075_b200 import solve as _solve
        res = _solve.solve_residual(op, sop.ndofs, device=dev, graph=True, timed_iterations=K)
        line["solve"] = {"what": "CG iteration on A x = -R(0): libdg apply + 2 dots + 3 updates, one CUDA graph "
                                 "replay (solve.cg_graph), CUDA events over K replays",
                         "ms_per_iteration": res.seconds_per_iteration * 1e3,
                         "apply_share": (statistics.mean(step_ms) if flush is None else warm_ms or kern_ms) /
                         (res.seconds_per_iteration * 1e3),
                         "dof_iterations_per_s": w.ndofs / res.seconds_per_iteration}
    if args.jacobian:
        line["config"]["operator"] = "Jacobian action J(u0) z (dg_apply_jacobian), u0 = sin(x)"
        line["roofline"]["kernel"] = op.kernel_name + " (mode 3: Jacobian)"
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(line), flush=True)
    sop.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
