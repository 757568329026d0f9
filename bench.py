#!/usr/bin/env python
"""Benchmark: range-space Schur solves/sec (two complex FETI-DP(H) solves on K -/+ i beta M)
on BASELINE.json configs[1] (2D heat control, 1024x1024 Q1 grid, 32x32 subdomains of
32x32 elements, FP64 complex, relative dual residual 1e-10).

One step = one range-space Schur solve (rhs = K ybar, FETI on K + cV, V a, FETI on K - cV,
primal recovery) for a fresh seeded sine-mode target ybar (seed = step index), factors
reused across steps (the reference's per_solve_seconds regime, experiments.cpp:265).

  value : solves/s through fetigpu_schur_solve_device (ybar resident in HBM), CUDA events
          on the library stream, max over ranks
  e2e   : solves/s through fetigpu_schur_solve (host buffers; H2D of ybar and D2H of y, u,
          lambda inside the timed region)
  --impl reference : the REFERENCE's own CPU implementation (oracle/_ref: the unmodified
          pdeopt sources built against the Eigen-API shim; its ComplexFactorSolver(FetiDp)
          pair set up once, rate = 1 / per_solve_seconds, experiments.cpp:265) on this host's
          cores, same workload string and metric (rank 0 only under torchrun); the C++
          restatement oracle/ where oracle/_ref is absent (kind "port").

Multi-GPU (N > 1, torchrun, one rank per GPU): weak scaling on the subdomain-sharded NCCL
path.  The mesh grows with N at a fixed 1024 subdomains of 32x32 elements
per GPU: N=2 1024x2048 (32x64 subdomains), N=4 2048x2048 (64x64, the BASELINE config-3
mesh), N=8 2048x4096 (64x128); subdomain rows are sharded block-wise, cut-line multipliers
are exchanged with NCCL send/recv, Krylov dots allreduced, the coarse problem solved
redundantly.  value = Schur solves/s x N (config-2-equivalent solves/s: each solve of the
N-GPU mesh is N config-2 blocks of work), so ideal weak scaling is value_N = N value_1.
--config 3 --gpus N: BASELINE config 3 exactly (2048^2, 64x64 subdomains, phi = 1e-6) on
every N, value = config-3 solves/s (strong scaling; N = 1 equals the --config 3 line).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Schur solves/sec (2 complex FETI-DPH solves), 2D Poisson 1M dofs"
UNIT = "solves/s"
N_GRID, S_SUB, PHI, TOL, MAX_ITER = 1024, 32, 1e-4, 1e-10, 2000
PHI_SWEEP = (1e-2, 1e-4, 1e-6, 1e-8)
# weak-scaling meshes: N -> (blocks along x, blocks along y) of 1024^2 elements / 32x32 subdomains
WEAK_BLOCKS = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}


def weak_problem_args(world):
    """(n_x, n_y, s_x, s_y, len_x, len_y) of the N-GPU weak-scaling mesh (square elements)."""
    if world not in WEAK_BLOCKS:
        raise SystemExit(f"bench.py: --gpus must be one of {sorted(WEAK_BLOCKS)}")
    a, b = WEAK_BLOCKS[world]
    m = max(a, b)
    return N_GRID * a, N_GRID * b, S_SUB * a, S_SUB * b, a / m, b / m


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device=0, period=0.005):
        self.samples, self.reasons, self.period = [], set(), period
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


WORKLOAD2D = {  # one string per BASELINE config, used by BOTH arms (same_config)
    2: "config2: 1024x1024 Q1 heat, 32x32 subdomains of 32x32, phi=1e-4, tol 1e-10, FP64 complex",
    3: "config3: 2048x2048 Q1 heat, 64x64 subdomains of 32x32, phi=1e-6, tol 1e-10, FP64 complex",
}
CONFIG2D = {2: (N_GRID, S_SUB, PHI), 3: (2 * N_GRID, 2 * S_SUB, 1e-6)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample_reference(config, threads, steps, warmup, budget_s=150.0):
    """The REFERENCE on the host cores: its unmodified sources (oracle/_ref, built against the
    Eigen-API shim) through its own classes -- solve_range_space's two
    ComplexFactorSolver(FetiDp) set up once (control.cpp:302-304), then per step the dual part
    of solve_range_space (control.cpp:306-320) on a fresh seeded target.  The rate is
    1 / per_solve_seconds, the reference's own per-solve time (the wall time of the two
    factor solves, experiments.cpp:265).  Falls back to the C++ restatement (oracle/) where
    oracle/_ref was not built.  Returns a dict."""
    n, s, phi = CONFIG2D[config]
    import paper_1312_5653_b200 as F

    def target(k):
        return F.make_seeded_problem(n, phi, seed=k).target_state

    try:
        from oracle import refbind as R

        R.lib()
        kind = "reference"
    except Exception:
        kind = "port"
    if kind == "reference":
        pair = R.FactorPair(n, s, s, phi, tol=TOL, max_iter=MAX_ITER, threads=threads)
        run = lambda yb: pair.solve(yb)[1]  # noqa: E731
        what = (f"pdeopt ComplexFactorSolver(FetiDp) x2 (unmodified reference sources, Eigen-API shim), "
                f"FetiConfig::threads={threads}")
    else:
        from oracle import oracle as O

        op = O.Problem(n)
        pair = O.SchurPair(op, s, s, phi, tol=TOL, max_iter=MAX_ITER, threads=threads)

        def run(yb):
            t0 = time.perf_counter()
            r = pair.run(yb)
            return {"per_solve_seconds": time.perf_counter() - t0,
                    "iterations": (r["plus_stats"]["iterations"], r["minus_stats"]["iterations"])}
        what = f"oracle/ (C++ restatement), std::thread x{threads}"
    for w in range(warmup):
        run(target(1000 + w))
    times, its = [], None
    t_start = time.perf_counter()
    for k in range(steps):
        st = run(target(k))
        times.append(st["per_solve_seconds"])
        its = st["iterations"]
        if time.perf_counter() - t_start > budget_s:
            break
    rate = len(times) / sum(times)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": kind, "cpu_model": cpu_model(),
            "sample": f"{len(times)} {WORKLOAD2D[config].split(':')[0]} Schur solves with the factors reused, "
                      f"{what}; setup {pair.setup_seconds:.1f} s; iterations {list(its)}",
            "setup_seconds": pair.setup_seconds, "iterations": list(its), "steps_run": len(times)}


def solve_roofline(solver, prof, steps, ms_per_step, hbm_peak):
    """Schur-solve roofline: the operator bytes streamed per solve (both GEMV
    classes and the interior solves, algorithmic bytes x launches) over the HBM peak, as a
    fraction of the measured time per solve."""
    b = 0.0
    for c in ("precond_gemv", "dual_gemv", "band"):
        b += solver.class_bytes(c) * prof[c]["launches"] / steps
    t_roof = b / (hbm_peak * 1e9) * 1e3
    return {"bytes_per_solve": b, "t_roof_ms": t_roof, "ms_per_solve": ms_per_step, "frac": t_roof / ms_per_step,
            "classes": ["precond_gemv", "dual_gemv", "band"]}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path (oracle/_ref) on
    this host's cores, rank 0 only, on the same workload / metric as our arm.  The 3D configs
    (4, 5) have no reference counterpart (the reference is 2D only): the oracle's 3D
    restatement on a bounded sample stands in."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    if args.config in CONFIG3D:
        cfg = CONFIG3D[args.config]
        rate, ts, its_s, su, m = cpu_sample_oracle3d(cfg, threads, None)
        cb = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
              "sample": f"oracle/ 3D restatement ({threads} threads) on the {m}^3 mesh with 2x2x2 subdomains of the "
                        f"config's size, one Schur solve {ts:.2f} s, scaled by {cfg['s'] ** 3}/8 subdomains"}
        workload = cfg["workload"]
        metric = METRIC.replace("2D Poisson 1M dofs", "3D config %d" % args.config)
    else:
        config = 3 if args.config == 3 else 2
        # each step is one config-2 Schur solve (~5-15 s on 16 cores); warm-up capped at one
        # solve and the timed steps at a 150 s budget so the arm ends within minutes
        cb = cpu_sample_reference(config, threads, args.steps, min(args.warmup, 1))
        rate = cb["value"]
        workload = WORKLOAD2D[config]
        metric = METRIC
    line = {
        "impl": "reference", "metric": metric, "value": rate, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 / rate, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded sine-mode ybar, seed = step)",
        "config": {"workload": workload},
        "cpu_baseline": cb,
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    rank, world, local = dist_env()
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1312_5653_b200 as F

    steps, warmup = args.steps, max(args.warmup, 3)
    n_x, n_y, s_x, s_y, len_x, len_y = weak_problem_args(world)
    phi = PHI
    if args.config == 3:  # BASELINE config 3: 2048^2, 64x64 subdomains, phi 1e-6 -- the same mesh on
        # every N (subdomain rows sharded over the ranks: strong scaling of the config)
        n_x = n_y = 2 * N_GRID
        s_x = s_y = 2 * S_SUB
        len_x = len_y = 1.0
        phi = 1e-6

    def problem(seed):
        return F.make_problem(n_x, n_y, phi, len_x=len_x, len_y=len_y, target="sine", seed=seed)

    p = problem(0)
    # one-time process costs (CUDA module load of the library, stream / event pools) are not
    # part of the solver's setup: create and drop a small context first
    if world == 1:
        F.SchurSolver(F.make_seeded_problem(64, phi, seed=0), 4, 4, tol=TOL, max_iter=50, device=local).close()
    t0 = time.perf_counter()
    if world > 1:  # subdomain-sharded over NCCL; rank 0 makes the NCCL id
        import torch.distributed as dist

        obj = [F.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        solver = F.SchurSolver(p, s_x, s_y, tol=TOL, max_iter=MAX_ITER, device=local, rank=rank, world=world,
                               nccl_id=obj[0])
    else:
        solver = F.SchurSolver(p, s_x, s_y, tol=TOL, max_iter=MAX_ITER, device=local, augment=args.augment)
    setup_s = time.perf_counter() - t0
    n = p.n
    # seeded targets for every step (the same on every rank), resident in HBM before the timed region
    seeds = list(range(warmup + steps))
    targets = [problem(s).target_state for s in seeds]
    d_ybar = [torch.from_numpy(t).cuda() for t in targets]
    d_y = torch.empty(n, dtype=torch.float64, device="cuda")
    d_u = torch.empty_like(d_y)
    d_l = torch.empty_like(d_y)
    stream = torch.cuda.ExternalStream(solver.stream)

    def device_step(k):
        return solver.solve_device(d_ybar[k].data_ptr(), 0, d_y.data_ptr(), d_u.data_ptr(), d_l.data_ptr())

    for k in range(warmup):
        st = device_step(k)
    torch.cuda.synchronize()
    its = []
    # ---------------- timed region: value (inputs resident in HBM) ----------------
    barrier(world)
    torch.cuda.synchronize()
    launches0 = solver.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for k in range(warmup, warmup + steps):
            st = device_step(k)
            its.append((st["plus_stats"]["iterations"], st["minus_stats"]["iterations"]))
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = solver.launch_count() - launches0
    t_dev = ev0.elapsed_time(ev1) / 1000.0
    t_max = max_over_ranks(t_dev, world)
    # weak ladder: config-2-equivalent solves/s (module docstring); --config 3: config-3 solves/s
    mult = 1 if args.config == 3 else world
    value = steps * mult / t_max
    # ---------------- e2e: host buffers through the public API ----------------
    # host buffers in pinned memory (the path a serving caller would use)
    host_t = [torch.from_numpy(t).pin_memory().numpy() for t in targets]
    outs = tuple(torch.empty(n, dtype=torch.float64).pin_memory().numpy() for _ in range(3))
    solver.solve(host_t[0], None, out=outs)
    barrier(world)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for k in range(warmup, warmup + steps):
        r = solver.solve(host_t[k], None, out=outs)
    w1 = time.perf_counter()
    barrier(world)
    e2e_t = max_over_ranks(w1 - w0, world)
    e2e = steps * mult / e2e_t
    # ---------------- per-kernel roofline pass (same K steps, events per launch) ----------------
    solver.profile(True)
    solver.profile_read(reset=True)
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    for k in range(warmup, warmup + steps):
        device_step(k)
    ev3.record(stream)
    torch.cuda.synchronize()
    prof = solver.profile_read(reset=True)
    solver.profile(False)
    t_prof = ev2.elapsed_time(ev3) / steps
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    kclass = max(("dual_gemv", "precond_gemv"), key=lambda c: prof[c]["ms"])
    kb = solver.class_bytes(kclass)
    eager_ms = prof[kclass]["ms"] / max(prof[kclass]["launches"], 1)
    # average launch duration under the Arnoldi graph's launch conditions: CUDA events around
    # a captured graph of 20 consecutive launches of each GEMV on the solver stream (the eager
    # per-launch events above also time the launch latency of every ~25 us kernel)
    graph_ms = None
    if world == 1:
        try:
            graph_ms = solver.gemv_timing(20)[kclass]
        except Exception:
            graph_ms = None
    avg_ms = graph_ms if graph_ms else eager_ms
    achieved = kb / (avg_ms / 1000.0) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(kclass)
    except Exception:
        pass
    if traffic and not (0.5 * kb <= traffic <= 4 * kb):
        traffic = None  # the committed ncu capture is of another config's launch size
    kernel_breakdown = {c: {"ms_per_step": v["ms"] / steps, "launches_per_step": v["launches"] / steps}
                        for c, v in prof.items() if v["launches"]}
    # in-graph kernel spans (first CTA start .. last CTA end, %globaltimer) of the last
    # FETI solve of the timed device run above: the GEMVs' streaming rate without the
    # per-launch event brackets of the profiling pass
    device_step(warmup)
    torch.cuda.synchronize()
    spans = solver.step_spans()
    in_graph = None
    if spans:
        # a span whose %globaltimer stamps were not both written reads as garbage: null it
        in_graph = {"spans_us": {k: (round(v, 3) if 0.0 <= v < 1e6 else None)
                                 for k, v in spans.items() if k != "steps"}, "steps": spans["steps"]}
        for cls, key in (("precond_gemv", "precond"), ("dual_gemv", "dual")):
            if in_graph["spans_us"].get(key) and in_graph["spans_us"][key] > 0.0:
                gbs = solver.class_bytes(cls) / (spans[key] * 1e-6) / 1e9
                in_graph[cls] = {"achieved_gbs": gbs, "frac": gbs / hbm_peak}
            else:
                in_graph[cls] = None
    # per-solve HBM bytes of the local operators (both GEMV classes) -> effective GB/s
    iters = np.mean([a + b for a, b in its])
    ms_solve = t_max / steps * 1000.0 / (1 if args.config == 3 else world)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": t_max / steps * 1000.0, "higher_is_better": True,
        "scaling": "strong" if (args.config == 3 and world > 1) else "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (seeded sine-mode ybar, seed = step; factors random-free FEM)",
        "config": {
            "workload": (WORKLOAD2D[args.config] if (world == 1 or args.config == 3) else
                         f"weak scaling: {n_x}x{n_y} Q1 heat, {s_x}x{s_y} subdomains of 32x32 ({s_x * s_y // world} "
                         f"per GPU), phi=1e-4, tol 1e-10, FP64 complex; value = solves/s x {world}"),
            "phi": phi, "n_free": n, "n_lambda": solver.n_lambda, "coarse_dim": solver.coarse_dim,
            "augment": bool(args.augment),
            "iterations_plus_minus_mean": [float(np.mean([a for a, _ in its])), float(np.mean([b for _, b in its]))],
            "setup_seconds": setup_s,
            # SURVEY §8d / experiments.cpp:264-265: solves/s including the setup (factorization)
            "solves_per_s_including_setup": 1.0 / (setup_s + ms_solve / 1000.0),
            "l2": "inputs larger than L2 (local operators 0.3 GB streamed per iteration)",
            "parallelism": f"subdomain rows sharded over {world} GPUs (NCCL)" if world > 1 else "1 GPU",
            "weak_or_strong": ("strong: BASELINE config 3 on every N" if args.config == 3 else
                               "weak: 1024 subdomains of 32x32 per GPU"),
            "kernel_ms_per_step": kernel_breakdown, "profiled_ms_per_step": t_prof,
        },
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 3 * 8 * n},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": kclass, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_launch": kb, "avg_launch_ms": avg_ms,
                     "timing": ("CUDA events on the solver stream around a captured graph of 20 consecutive "
                                "launches of the kernel (average launch duration incl. the PDL gaps)" if graph_ms else
                                "CUDA events around each eager launch of the profiling pass"),
                     "eager_avg_launch_ms": eager_ms, "eager_frac": kb / (eager_ms / 1000.0) / 1e9 / hbm_peak,
                     "in_graph": in_graph,
                     "note": ("bytes_per_launch = the GEMV's operands only; at config 2 the dual GEMV's launch "
                              "(k_sym_gemv_aside) also holds the coarse CTAs of the step's coarse solve, whose "
                              "14.8 MB read of C^-1 (L2-resident in the solve, cold under ncu) is part of `traffic` "
                              "but not of bytes_per_launch (DESIGN.md section 4)") if kclass == "dual_gemv" else None},
        "clocks": clk.summary(),
    }
    line["solve_roofline"] = solve_roofline(solver, prof, steps, t_max / steps * 1000.0, hbm_peak)
    # BASELINE config 2 is a phi sweep: rates and iteration counts per phi (own factors each)
    if rank == 0 and world == 1 and args.config == 2 and not args.no_sweep:
        sweep = {}
        for phi in PHI_SWEEP:
            q = F.make_seeded_problem(N_GRID, phi, seed=0)
            t1 = time.perf_counter()
            sv = F.SchurSolver(q, S_SUB, S_SUB, tol=TOL, max_iter=MAX_ITER, device=local)
            su = time.perf_counter() - t1
            sv.solve_device(d_ybar[0].data_ptr(), 0, d_y.data_ptr(), d_u.data_ptr(), d_l.data_ptr())
            sstream = torch.cuda.ExternalStream(sv.stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(sstream)
            for k in range(3):
                st = sv.solve_device(d_ybar[k].data_ptr(), 0, d_y.data_ptr(), d_u.data_ptr(), d_l.data_ptr())
            e1.record(sstream)
            torch.cuda.synchronize()
            sweep[f"{phi:g}"] = {"solves_per_s": 3000.0 / e0.elapsed_time(e1), "setup_s": su,
                                 "iterations_plus_minus": [st["plus_stats"]["iterations"],
                                                           st["minus_stats"]["iterations"]]}
            sv.close()
        line["config"]["phi_sweep"] = sweep
    if rank == 0 and world == 1 and args.config == 2 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_sample_reference(2, os.cpu_count() or 1, 1, 0)
    if rank == 0:
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


CONFIG3D = {  # BASELINE.json configs 4-5 (the 3D extension; one GPU)
    4: dict(n=128, s=8, phi=1e-6, physics=0, mmax=6,
            workload="config4: 128^3 Q1 hexahedra heat, 8x8x8 subdomains of 16^3, phi=1e-6, tol 1e-10, FP64 complex"),
    5: dict(n=64, s=4, phi=1e-4, physics=1, mmax=6,
            workload="config5: 64^3 Q1 hexahedra linear elasticity (E=1, nu=0.3, clamped x=0), 4x4x4 subdomains of "
                     "16^3, phi=1e-4, tol 1e-10, FP64 complex"),
}


def cpu_sample_oracle3d(cfg, threads, its_gpu):
    """Oracle (3D restatement) on a bounded sample with the config's subdomain size: the
    2x2x2-subdomain cube of 16^3-element subdomains (32^3 mesh), setup once, one Schur solve.
    Scaled to the config by subdomain count and iteration count (work per Krylov step is
    per-subdomain), i.e. rate = 1 / (t_sample * (S_config / 8) * (its_gpu / its_sample))."""
    from oracle import oracle as O

    e = cfg["n"] // cfg["s"]
    p = O.Problem(2 * e, 2 * e, n_z=2 * e, physics=cfg["physics"], young=1.0, poisson=0.3)
    pair = O.SchurPair(p, 2, 2, cfg["phi"], tol=TOL, max_iter=MAX_ITER, threads=threads, s_z=2, setup_threads=threads)
    t0 = time.perf_counter()
    r = pair.run(p.target_sine(0, mmax=cfg["mmax"]))
    t = time.perf_counter() - t0
    its = r["plus_stats"]["iterations"] + r["minus_stats"]["iterations"]
    scale = (cfg["s"] ** 3 / 8.0) * (its_gpu / max(its, 1))
    return 1.0 / (t * scale), t, its, pair.setup_seconds, 2 * e


def run_gpu3d(args):
    """BASELINE configs 4-5.  N > 1 (torchrun): strong scaling of the same mesh, contiguous
    subdomain ranges (z-layers, or y-row blocks of a layer: config 5 on 8 GPUs) per rank (NCCL allreduce of the jump partials per operator
    application, coarse problem assembled by allreduce and solved redundantly)."""
    rank, world, local = dist_env()
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1312_5653_b200 import box

    cfg = CONFIG3D[args.config]
    steps, warmup = args.steps, max(args.warmup, 3)

    def problem(seed):
        return box.make_box_problem(cfg["n"], phi=cfg["phi"], physics=cfg["physics"], young=1.0, poisson=0.3,
                                    seed=seed, mmax=cfg["mmax"])

    p = problem(0)
    t0 = time.perf_counter()
    if world > 1:
        import paper_1312_5653_b200 as F
        import torch.distributed as dist

        obj = [F.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        solver = box.BoxSchurSolver(p, cfg["s"], tol=TOL, max_iter=MAX_ITER, device=local, rank=rank, world=world,
                                    nccl_id=obj[0])
    else:
        solver = box.BoxSchurSolver(p, cfg["s"], tol=TOL, max_iter=MAX_ITER, device=local)
    setup_s = time.perf_counter() - t0
    n = p.n
    seeds = list(range(warmup + steps))
    targets = [problem(sd).target_state for sd in seeds]
    d_ybar = [torch.from_numpy(t).cuda() for t in targets]
    d_y = torch.empty(n, dtype=torch.float64, device="cuda")
    d_u, d_l = torch.empty_like(d_y), torch.empty_like(d_y)
    stream = torch.cuda.ExternalStream(solver.stream)

    def device_step(k):
        return solver.solve_device(d_ybar[k].data_ptr(), 0, d_y.data_ptr(), d_u.data_ptr(), d_l.data_ptr())

    for k in range(warmup):
        device_step(k)
    torch.cuda.synchronize()
    its = []
    barrier(world)
    torch.cuda.synchronize()
    launches0 = solver.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for k in range(warmup, warmup + steps):
            st = device_step(k)
            its.append((st["plus_stats"]["iterations"], st["minus_stats"]["iterations"]))
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = solver.launch_count() - launches0
    t_dev = max_over_ranks(ev0.elapsed_time(ev1) / 1000.0, world)
    value = steps / t_dev  # strong scaling: the same config solved by all ranks together
    host_t = [torch.from_numpy(t).pin_memory().numpy() for t in targets]
    outs = tuple(torch.empty(n, dtype=torch.float64).pin_memory().numpy() for _ in range(3))
    solver.solve(host_t[0], None, out=outs)
    barrier(world)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for k in range(warmup, warmup + steps):
        solver.solve(host_t[k], None, out=outs)
    w1 = time.perf_counter()
    barrier(world)
    e2e = steps / max_over_ranks(w1 - w0, world)
    solver.profile(True)
    solver.profile_read(reset=True)
    for k in range(warmup, warmup + steps):
        device_step(k)
    torch.cuda.synchronize()
    prof = solver.profile_read(reset=True)
    solver.profile(False)
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    kclass = max(("dual_gemv", "precond_gemv"), key=lambda c: prof[c]["ms"])
    kb = solver.class_bytes(kclass)
    avg_ms = prof[kclass]["ms"] / max(prof[kclass]["launches"], 1)
    achieved = kb / (avg_ms / 1000.0) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"config{args.config}_{kclass}")
    except Exception:
        pass
    iters = [float(np.mean([a for a, _ in its])), float(np.mean([b for _, b in its]))]
    line = {
        "metric": METRIC.replace("2D Poisson 1M dofs", "3D config %d" % args.config), "value": value, "unit": UNIT,
        "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": t_dev / steps * 1000.0,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded sine-mode ybar on the cube, seed = step)",
        "config": {"workload": cfg["workload"], "phi": cfg["phi"], "n_free": n, "n_lambda": solver.n_lambda,
                   "coarse_dim": solver.coarse_dim, "iterations_plus_minus_mean": iters, "setup_seconds": setup_s,
                   "setup_phases_s": solver.setup_times(),
                   "l2": "inputs larger than L2 (packed S_bb, S_bb^-1: %.1f GB each)" % (kb / 1e9),
                   "parallelism": (f"contiguous subdomain ranges (z-layers / y-row blocks) over {world} GPUs (NCCL allreduce of jump partials)"
                                   if world > 1 else "1 GPU"),
                   "kernel_ms_per_step": {c: {"ms_per_step": v["ms"] / steps, "launches_per_step": v["launches"] / steps}
                                          for c, v in prof.items() if v["launches"]}},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 3 * 8 * n},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": kclass, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "peak_source": "measured" if "hbm_gbs" in peaks else "fallback",
                     "bytes_per_launch": kb, "avg_launch_ms": avg_ms},
        "clocks": clk.summary(),
    }
    line["solve_roofline"] = solve_roofline(solver, prof, steps, t_dev / steps * 1000.0, hbm_peak)
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, ts, its_s, su, m = cpu_sample_oracle3d(cfg, threads, sum(iters))
        line["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"oracle/ ({threads} threads) on the {m}^3 mesh with 2x2x2 subdomains of the config's size: "
                      f"setup {su:.1f} s, one Schur solve {ts:.2f} s with {its_s} iterations, scaled by "
                      f"{cfg['s'] ** 3}/8 subdomains and {sum(iters):.0f}/{its_s} iterations"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                    help="2: the headline config (default); 3: BASELINE config 3 on one GPU; 4/5: the 3D configs")
    ap.add_argument("--augment", action="store_true",
                    help="edge-RBM augmented coarse space (reference default; BASELINE configs use augment=false)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.config in CONFIG3D:
        return run_gpu3d(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
