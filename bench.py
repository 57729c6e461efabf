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
def _host_info():
    """lscpu model, host cores and the oracle's OpenMP thread count (SURVEY §8(d) oracle timing)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}


class OracleSample:
    """The oracle (as it stands) on a fixed, deterministic random sample of cells of workload w, sized once
    (calibrate) to about `budget_s` seconds of host CPU work; run() times one evaluation of that sample."""

    def __init__(self, w, seed: int = 2024, jacobian: bool = False):
        import numpy as np

        import synth
        self.w, self.jacobian = w, jacobian
        self.rng = np.random.default_rng(seed)
        self.x = synth.x_np(w) if w.problem in (1, 2, 3) else None
        self.cells = None

    def _prepare(self, ncell):
        import numpy as np

        import oracle
        import synth
        w = self.w
        self.cells = np.sort(self.rng.choice(w.ncells, ncell, replace=False)).astype(np.int64)
        if w.problem not in (1, 2, 3):
            nb = oracle.neighbours(w, self.cells)
            self.x7 = synth.x_cells_np(w, nb.reshape(-1)).reshape(len(self.cells), 7, w.block)
            self.j7 = synth.jac_cells_np(w, nb.reshape(-1)).reshape(len(self.cells), 7, 9) if w.geom_kind else None

    def run(self):
        import numpy as np

        import oracle
        w, cells = self.w, self.cells
        t0 = time.perf_counter()
        if w.problem == 3:
            oracle.apply_stokes(w, self.x, cells)
        elif w.problem == 1:
            oracle.apply_diffreac(w, self.x, cells)
        elif w.problem == 2:
            oracle.apply_nlreac(w, self.x, u0=np.sin(self.x) if self.jacobian else None, cells=cells)
        else:
            oracle.apply_cells_local(w, cells, self.x7, self.j7)
        return time.perf_counter() - t0

    def calibrate(self, budget_s: float):
        import oracle
        th = oracle.num_threads()
        ncell = min(self.w.ncells, max(th, 8))
        self._prepare(ncell)
        t = self.run()
        while t < 0.1 * budget_s and ncell < self.w.ncells:  # grow the probe until it costs ~10% of the budget
            ncell = min(self.w.ncells, ncell * 4)
            self._prepare(ncell)
            t = self.run()
        target = int(min(self.w.ncells, max(ncell, ncell * budget_s / max(t, 1e-9))))
        if target != ncell:
            self._prepare(target)
        return self

    @property
    def dofs(self):
        return len(self.cells) * self.w.block


def oracle_sample_rate(w, budget_s: float, seed: int = 2024, jacobian: bool = False, threads: int | None = None):
    """Time the oracle on a random cell sample of about budget_s seconds. Returns (DOF/s, cells, seconds, threads)."""
    import oracle
    th0 = oracle.num_threads()
    if threads:
        oracle.set_threads(threads)
    try:
        s = OracleSample(w, seed, jacobian).calibrate(budget_s)
        t = s.run()
        return s.dofs / t, len(s.cells), t, oracle.num_threads()
    finally:
        oracle.set_threads(th0)


def run_reference(args, w, rank):
    """--impl reference: the oracle on the host cores, rank 0 only; one calibrated sample per step so that the
    whole --steps K --warmup W run stays within a few minutes."""
    if rank != 0:
        return 0
    import oracle
    budget = max(0.3, min(4.0, 100.0 / (args.steps + args.warmup)))
    s = OracleSample(w, jacobian=args.jacobian).calibrate(budget)
    for _ in range(args.warmup):
        s.run()
    times = [s.run() for _ in range(args.steps)]
    t_step = statistics.median(times)
    value = s.dofs / t_step
    th = oracle.num_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": w.ndofs / value * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(w, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": th, "kind": "oracle",
                         "sample": f"{len(s.cells)} random cells ({s.dofs} DOFs) of {w.name} per step, "
                                   f"median {t_step:.2f} s per step; ms_per_step extrapolated to the whole mesh",
                         **_host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    _emit(line)
    return 0


class _DistSlab:
    """bench.py's view of a DistOperator (the same attributes it uses of slab.SlabOperator)."""

    def __init__(self, op):
        self.op = op
        self.ndofs, self.offset, self.plane_ndofs = op.ndofs, op.offset, op.plane_ndofs
        self.launches_per_apply = op.launches_per_apply
        self.traces = op.kernel_name in ("k_gen", "k_axis8", "k_line")
        self.payload_doubles = op.halo_ndofs if self.traces else op.plane_ndofs

    def apply(self, x, r=None):
        return self.op.apply(x, r)

    def close(self):
        self.op.close()


def _profile_record(workload, kernel):
    """ncu numbers of this kernel on this workload from the newest profiles/<round>/ncu_counters.json
    (written by tools/ncu_summary.py from an `ncu --set full` capture of the same command)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_counters.json")), reverse=True):
        try:
            rec = json.load(open(path)).get(workload, {}).get(kernel)
        except Exception:
            rec = None
        if rec:
            rec = dict(rec)
            rec["src"] = os.path.relpath(path, ROOT)
            return rec
    return None


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
            if 8 * w.ndofs > 2 * 126e6 else "L2 flushed between steps (512 MB written, then 512 MB read so the "
                                                "flush's write-backs land before the timed apply)"}


# ----------------------------------------------------------------------------- main
_OUT = None  # the original stdout: exactly one JSON line goes there


def _emit(line):
    out = _OUT if _OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _stdout_for_json_only():
    """Point fd 1 at stderr for the rest of the run (NCCL writes its version / INFO lines to stdout from native
    code), keeping the original stdout for the one JSON line."""
    global _OUT
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def main():
    _stdout_for_json_only()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--comm", default="libdg", choices=["libdg", "torch"],
                    help="N > 1: the halo exchange of libdg's collective C-ABI (dg_apply_dist, its own NCCL "
                         "communicator; default) or of slab.py over torch.distributed")
    ap.add_argument("--dist-loopback", action="store_true",
                    help="N = 1: run the collective multi-GPU step (dg_setup_dist / dg_apply_dist with one rank: trace "
                         "packing, interior planes, NCCL send/recv of the wrap halos to itself, boundary planes) instead "
                         "of the single dg_apply launch; measures the cost of the slab-step structure on one GPU")
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
    ap.add_argument("--basis", default="gauss", choices=["gauss", "lobatto", "equidistant"],
                    help="Lagrange basis nodes: gauss (the configs, reading R8) or lobatto (the non-Gauss basis of SURVEY "
                         "§8(f2): A != I at every rule, k_quad)")
    ap.add_argument("--quad", type=int, default=-1,
                    help="Gauss points per direction (default k+1; k+2 = overintegration, SURVEY §8(f2))")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.dist_loopback:
        args.no_e2e = True  # the loopback mode measures the device-side slab step only

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
    if args.basis != "gauss":
        import dataclasses
        w = dataclasses.replace(w, basis=1 if args.basis == "lobatto" else 2,
                                name=f"{w.name}_{'gll' if args.basis == 'lobatto' else 'equi'}")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and args.impl != "reference":
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch N ranks with torchrun "
                         f"(python -m torch.distributed.run --nproc-per-node {args.gpus} ... bench.py --gpus {args.gpus})")
    if args.impl == "reference":
        return run_reference(args, w, rank)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1812_08075_b200 import dg, slab
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        # NCCL's own init lines (transport, rings / channels over NVLink) in the run log (stderr: fd 1 points there,
        # see _stdout_for_json_only): the communicator the halo exchange uses is visible
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,P2P")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    stream = torch.cuda.current_stream(dev)

    def jac_fn(pb, npl):
        return synth.jac_planes_torch(w, pb, npl, device=dev).cpu().numpy()

    if (world > 1 or args.dist_loopback) and args.comm == "libdg" and not args.jacobian:
        # the collective C-ABI (dg_setup_dist / dg_apply_dist): libdg's own NCCL communicator and halo step
        uid = [dg.dg_get_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        pb, npl = dg.dg_slab_range(w.N[0], rank, world)
        jac = jac_fn(pb - 1, npl + 2) if w.geom_kind else None
        sop = _DistSlab(dg.DistOperator(w.N, w.k, rank, world, uid[0], geom_kind=w.geom_kind, coeff_kind=w.coeff_kind,
                                        penalty_scale=w.penalty_scale, jac=jac, device=local_rank, quad=w.m,
                                        problem=w.problem, basis=w.basis))
    else:
        sop = slab.SlabOperator(w.N, w.k, rank, world, geom_kind=w.geom_kind, coeff_kind=w.coeff_kind,
                                penalty_scale=w.penalty_scale, jac_fn=jac_fn, device=local_rank, quad=w.m,
                                problem=w.problem, basis=w.basis)
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

    # ---- timed region: exactly K steps, events on the launching stream, barrier + synchronize on both sides;
    #      per-step event pairs give the kernel's average duration (N = 1: one launch per step, so step == kernel)
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local_rank)
    barrier()
    flush = None
    if 8 * sop.ndofs * 2 < 4 * 126e6:
        # vectors fit in L2: flush it between timed steps (write 512 MB), time the steps alone; then read another
        # 512 MB so that the write-backs of the flush's dirty lines happen before the timed apply, not inside it
        # (otherwise the apply's first loads evict 126 MB of dirty flush data and pay its DRAM write-back)
        flush = torch.empty(64 << 20, dtype=torch.float64, device=dev)
        flush_rd = torch.ones(64 << 20, dtype=torch.float64, device=dev)
        flush_sink = torch.empty((), dtype=torch.float64, device=dev)
    with clk:
        # the timed region is the profiled range: `ncu --profile-from-start off` lists exactly its launches
        torch.cuda.profiler.start()
        t_start.record(stream)
        for i in range(K):
            if flush is not None:
                flush.fill_(float(i))
                torch.sum(flush_rd, dim=0, out=flush_sink)
            ev[i][0].record(stream)
            step(x, r)
            ev[i][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        barrier()
        step_ms = [a.elapsed_time(b) for a, b in ev]
        # ---- sustained: >= 200 ms of back-to-back applies (SURVEY §8(d) timing protocol: >= 100 ms per line),
        #      replayed from one CUDA graph when an apply is short (cfg0 / cfg1: launch latency), under the same
        #      clock sampler; the roofline below uses this per-apply time (warm L2 for L2-resident vectors)
        est = max(statistics.median(step_ms), 1e-3)
        R = int(min(400000, max(K, 200.0 / est)))
        graph = None
        if est < 1.0 and world == 1:
            gs = torch.cuda.Stream(dev)
            gs.wait_stream(stream)
            with torch.cuda.stream(gs):
                op.set_stream(gs)
                step(x, r)  # warm the capture stream
                graph = torch.cuda.CUDAGraph()
                reps = min(R, 500)
                with torch.cuda.graph(graph, stream=gs):
                    for _ in range(reps):
                        step(x, r)
            stream.wait_stream(gs)
            op.set_stream(stream)
            nrep = max(1, R // reps)
            R = reps * nrep
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        s0.record(stream)
        if graph is not None:
            for _ in range(nrep):
                graph.replay()
        else:
            for _ in range(R):
                step(x, r)
        s1.record(stream)
        torch.cuda.synchronize()
        sustained_ms = s0.elapsed_time(s1) / R
    barrier()
    warm_ms = sustained_ms if flush is not None else None
    total_ms = t_start.elapsed_time(t_end) if flush is None else sum(step_ms)
    t_local = torch.tensor([total_ms, sustained_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms = t_local[0].item()
    ms_per_step = total_ms / K
    value = w.ndofs / (ms_per_step * 1e-3)

    # ---- roofline of the dominant kernel (per launch, this rank; per-apply time of the sustained region)
    pk = _peaks()
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    fp64_nominal = sms * 64 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12  # TFLOP/s: SMs x 64 DFMA/clk x 2 flop x clock
    fp64_meas, _ = dg.dg_bench_fp64(local_rank, 4000)
    kern_ms = sustained_ms if world == 1 else statistics.mean(step_ms)
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
    prof = _profile_record(w.name, op.kernel_name)
    traffic = prof.get("dram_bytes") if prof else None
    if t_flop >= t_byte:
        roof = {"bound": "alu", "achieved": ach_tf, "peak": fp64_nominal, "unit": "TFLOP/s",
                "frac": ach_tf / fp64_nominal, "traffic": traffic,
                "peak_src": f"derived: {sms} SMs x 64 DFMA/clk x 2 x {pk['sm_max_mhz']:.0f} MHz (DESIGN.md §4); "
                            f"'achieved' = F_alg (SURVEY §8(d) algorithmic flops) / kernel time"}
    else:
        roof = {"bound": "hbm", "achieved": ach_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": ach_gbs / pk["hbm_gbs"], "traffic": traffic, "peak_src": f"{pk['src']} copy bandwidth"}
    roof.update({"kernel": op.kernel_name, "kernel_ms": kern_ms,
                 "kernel_ms_src": "sustained region (>= 200 ms back-to-back, graph-replayed if short)" if world == 1
                 else "mean of the K timed steps",
                 "alg_flops_per_launch": F, "alg_bytes_per_launch": B, "frac_fp64": ach_tf / fp64_nominal,
                 "frac_fp64_measured_dfma": ach_tf / fp64_meas, "fp64_dfma_measured_tflops": fp64_meas,
                 "frac_hbm": ach_gbs / pk["hbm_gbs"], "t_roof_ms": max(t_flop, t_byte) * 1e3,
                 "frac_roof": max(t_flop, t_byte) * 1e3 / kern_ms,
                 "traffic_src": (f"ncu --set full of this kernel on this config ({prof.get('src')}): "
                                 "dram__bytes_read.sum + dram__bytes_write.sum per launch") if prof else None})
    if w.problem == 0 and w.geom_kind == 0 and w.coeff_kind == 0 and op.kernel_name in ("k_axis8", "k_gen"):
        # the axis-aligned kernels run the Kronecker-sum line operator (S_d = D^T W D along each line): SURVEY §8(d)
        # asks for the fraction against that smaller count too (volume 6 n^4 instead of 12 n^4 + 3 n^3 per cell)
        nn = w.n
        F_kron = (6.0 * nn + 48.0 + 30.0 / nn) * sop.ndofs
        roof["frac_kron"] = F_kron / (kern_ms * 1e-3) / 1e12 / fp64_nominal
        roof["alg_flops_kron_per_launch"] = F_kron
    if prof and prof.get("fp64_flops_issued"):
        # what the FP64 pipe actually executed (ncu: 2 dfma + dadd + dmul thread instructions), at this run's time
        roof["fp64_flops_issued_per_launch"] = prof["fp64_flops_issued"]
        roof["frac_exec"] = prof["fp64_flops_issued"] / (kern_ms * 1e-3) / 1e12 / fp64_nominal

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
        if world == 1 and not args.jacobian and 8 * w.ndofs >= (256 << 20):
            # the e2e leg's own ceiling on this box: the same bytes as plain pinned copies, H2D and D2H concurrently
            # on two streams in dg_apply_host's 32 chunks, no kernels (tools/mb_pcie.py standalone); only for vectors
            # >= 256 MB: below that the 64 Python-issued copies are launch-bound and say nothing about the link
            cd_in, cd_out = torch.empty_like(x), torch.empty_like(x)
            s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
            nb = [x.numel() * i // 32 for i in range(33)]

            def copies():
                s_in.wait_stream(torch.cuda.current_stream())
                s_out.wait_stream(torch.cuda.current_stream())
                for i in range(32):
                    with torch.cuda.stream(s_in):
                        cd_in[nb[i]:nb[i + 1]].copy_(xh[nb[i]:nb[i + 1]], non_blocking=True)
                    with torch.cuda.stream(s_out):
                        rh[nb[i]:nb[i + 1]].copy_(cd_out[nb[i]:nb[i + 1]], non_blocking=True)
                torch.cuda.current_stream().wait_stream(s_in)
                torch.cuda.current_stream().wait_stream(s_out)
                torch.cuda.synchronize()
            copies()
            t0 = time.perf_counter()
            for _ in range(KE):
                copies()
            tc = (time.perf_counter() - t0) / KE
            e2e["copy_ceiling"] = {"ms": tc * 1e3, "value": w.ndofs / tc,
                                   "frac": (tc * KE) / te,
                                   "how": "pinned H2D of x and D2H of r concurrently (2 streams, 32 chunks), no kernels"}
            del cd_in, cd_out
        del xh, rh, uh

    # ---- CPU baseline (rank 0, N = 1 only): the oracle as it stands on all host cores; for the small configs
    #      (cfg0 / cfg1) also on one thread (SURVEY §8(d) oracle timing)
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        v, cells, secs, th = oracle_sample_rate(w, args.cpu_seconds, jacobian=args.jacobian)
        cpu = {"value": v, "unit": UNIT, "cores": th, "kind": "oracle",
               "sample": f"{cells} random cells ({cells * w.block} DOFs) of {w.name}, {secs:.1f} s", **_host_info()}
        if w.ndofs <= 4_000_000:
            v1, c1, s1, _ = oracle_sample_rate(w, min(4.0, args.cpu_seconds / 3), jacobian=args.jacobian, threads=1)
            cpu["one_thread"] = {"value": v1, "unit": UNIT, "cores": 1,
                                 "sample": f"{c1} random cells ({c1 * w.block} DOFs), {s1:.1f} s"}

    # ---- sanity of the timed result (not a parity claim: tests/ do that): finite, nonzero
    ok = bool(torch.isfinite(r).all().item()) and r.abs().max().item() > 0
    halo = None
    if world > 1 or (args.dist_loopback and isinstance(sop, _DistSlab)):
        ap = sop if isinstance(sop, _DistSlab) else sop._apply
        halo = {"payload": "face traces (u, d_0 u at the n^2 face points, dg_pack_halo)" if ap.traces else "boundary planes",
                "bytes_per_message": 8 * ap.payload_doubles, "messages_per_rank": 4,
                "exchange": ("libdg dg_apply_dist (own NCCL communicator)" if isinstance(sop, _DistSlab)
                             else "slab.py over torch.distributed (NCCL)")
                            + (": one rank, the wrap halos sent / received to itself (--dist-loopback)" if world == 1 else ""),
                "overlap": "interior planes on the compute stream while the exchange runs on a high-priority stream; "
                           "NVTX ranges slab:pack / slab:interior / slab:halo / slab:boundary"}
        if isinstance(sop, _DistSlab) and ap.traces and op.nplanes >= 3:
            # SURVEY §8(d) interior / halo / boundary breakdown (no nsys on this pool): the step's pieces through the
            # same context, each launched alone and timed with events on the launching stream; what the overlapped
            # step costs beyond their sum is the exchange time the interior planes did not hide
            tlo, thi = (torch.empty(op.halo_ndofs, dtype=torch.float64, device=dev) for _ in range(2))
            op.pack_halo(x, tlo, thi)
            L = op.nplanes

            def _phase(fn, reps=20):
                fn()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record(stream)
                for _ in range(reps):
                    fn()
                b.record(stream)
                torch.cuda.synchronize()
                return a.elapsed_time(b) / reps
            t_pack = _phase(lambda: op.pack_halo(x, tlo, thi))
            t_int = _phase(lambda: op.apply_planes_tr(x, thi, tlo, r, 1, L - 1))
            t_bnd = _phase(lambda: (op.apply_planes_tr(x, thi, tlo, r, 0, 1), op.apply_planes_tr(x, thi, tlo, r, L - 1, L)))
            med = statistics.median(step_ms)
            halo["phases_ms"] = {"pack": t_pack, "interior": t_int, "boundary": t_bnd, "sum": t_pack + t_int + t_bnd,
                                 "step_median": med, "exposed_exchange": med - (t_pack + t_int + t_bnd),
                                 "how": "each piece alone on the compute stream (events, 20 launches); exposed_exchange = "
                                        "step median - sum (the exchange and stream hand-offs the interior did not hide)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": dict(_config(w, world), **({"mode": "dist-loopback: the collective slab step on one rank"}
                                             if args.dist_loopback and world == 1 else {})), "roofline": roof,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": K * sop.launches_per_apply,
        "clocks": clk.summary(), "result_finite": ok,
        "step_ms": {"median": statistics.median(step_ms), "min": min(step_ms), "max": max(step_ms)},
        "sustained": {"ms_per_apply": sustained_ms, "applies": R, "graph": graph is not None,
                      "value": w.ndofs / (sustained_ms * 1e-3), "l2": "warm" if flush is not None else "cold (vectors > L2)"},
        "warm_ms_per_step": warm_ms,
    }
    if halo:
        line["halo"] = halo
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
        _emit(line)
    sop.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
