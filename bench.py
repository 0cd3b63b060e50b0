#!/usr/bin/env python
"""Benchmark: DoF-updates/s of the ADER-DG hot path on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg3]

One "step" is one ADER-DG time step (admissible-dt reduction, space-time
predictor, fused Riemann + corrector) of the configuration over its whole
mesh, state resident in HBM.  The headline workload is the largest
single-GPU configuration, BASELINE.json configs[2] (config 3: 3-D Euler, 64^3
cells, p = 4, 1.64e8 DoF); its state plus predictor buffers (~5.7 GB) exceed
the 126 MB L2 many times, so no flush is needed between steps.  W warm-up
steps run first; the state is then reset to the initial condition and the
timed steps are steps 1..K of the stated trajectory (20 steps for config 3).
Under torchrun (N > 1) every rank runs an independent replica (the path does
not shard in this tier: "replicas only"); the value is the
aggregate over ranks, timed as the max over ranks.

--impl reference times the reference package's own per-cell CPU kernels
(oracle/refarm.py: the reference vendored into oracle/_ref by build(), else
the numpy port) on all host cores, each timed step on a bounded sample of
that same step's cells whose Picard counts follow the step's histogram
(tests/golden/refarm_cfg3.npz).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1806_07984_b200 import configs as cf  # noqa: E402
from paper_1806_07984_b200 import costs  # noqa: E402

METRIC = "DoF-updates/s per time step on 1 B200; % of FP64/HBM roofline per kernel"
EAGER_GATE_US = 3000     # GPU spin ahead of each eager (kernel-event) step, see run_ours
UNIT = "DoF-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(cf.CONFIGS))
    ap.add_argument("--no-secondary", action="store_true", help="skip the cfg2 (configs[1]) secondary line item")
    ap.add_argument("--lib", default=None, help="load this build of libenclavedg_b200.so (A/B of build_lib --variant)")
    ap.add_argument("--cfl", type=float, default=None, help="override the config's CFL safety")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-slabs", type=int, default=None, help="slabs of the streamed host step (default: step_host's)")
    ap.add_argument("--e2e-only", action="store_true", help="A/B helper: print only the e2e object")
    ap.add_argument("--no-variant", action="store_true", help="skip the parity-safe CFL 0.2 variant line item")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


# ------------------------------------------------------------------ ranks --

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def dist_init(ws, backend):
    if ws > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group(backend)
        return dist
    return None


def max_over_ranks(dist, x, device):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------- workloads --

def workload_name(cfg):
    if cfg.kind == "fv":
        return f"{cfg.name}: 3D Euler patch FV {cfg.cells}^3 cells in {cfg.patch}^3 patches, CFL {cfg.cfl}"
    what = "advection" if cfg.pde == "advection" else "Euler"
    mesh = f"{cfg.cells}^{cfg.dim}" + (" + refined disc (2-level 3:1)" if cfg.kind == "dg-amr" else "")
    return f"{cfg.name}: {cfg.dim}D {what} ADER-DG p={cfg.order} on {mesh}, CFL {cfg.cfl}/(2p+1)"


def build_solver(cfg):
    from paper_1806_07984_b200 import mesh as M, pde as P, solver as S
    if cfg.kind == "fv":
        s = S.FVSolver(P.euler(3), cfg.cells, cfg.patch, cfg.cfl, check_finite=False)
        return s, cf.initial_fv(cfg), cfg.cells ** 3
    pde = P.advection(cfg.velocity) if cfg.pde == "advection" else P.euler(cfg.dim)
    if cfg.kind == "dg-amr":
        mesh = M.AdaptiveMesh(cf.amr_cells(cfg), cfg.dim, cfg.periodic)
        Q0 = cf.initial_dg_amr(cfg, mesh.cells)
    else:
        mesh = M.CartesianMesh(cfg.cells, cfg.dim, cfg.periodic)
        Q0 = cf.initial_dg_uniform(cfg)
    return S.DGSolver(pde, cfg.order, mesh, cfg.cfl, check_finite=False), Q0, mesh.ncells


# ---------------------------------------------------------------- clocks --

class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------ FP64 peak --

def fp64_peak_tflops():
    """Measured DFMA throughput (MEASURED_PEAKS.json carries no FP64 figure)."""
    import ctypes
    import torch
    from paper_1806_07984_b200 import _lib
    lib = _lib.load()
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = nsm * 8, 4096
    best = 0.0
    for _ in range(6):   # clocks ramp up from idle: untimed launches first
        _lib.check(lib.edg_probe_fp64(_lib.ptr(sink), blocks, iters, st), "probe")
    for _ in range(8):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(lib.edg_probe_fp64(_lib.ptr(sink), blocks, iters, st), "probe")
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = max(best, blocks * 256 * 8 * iters * 2 / (ms * 1e-3) / 1e12)
    return best


def measured_peaks():
    try:
        return json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


# ----------------------------------------------------------- CPU (port) --

_CPU = {}


def _cpu_init(cfg_name, cfl):
    cfg = cf.CONFIGS[cfg_name]
    if cfl is not None:
        cfg = cfg.with_(cfl=cfl)
    from oracle import ops
    _CPU["cfg"] = cfg
    _CPU["Q"] = cf.initial_dg_uniform(cfg)
    _CPU["pde"] = ops.euler(cfg.dim) if cfg.pde == "euler" else ops.advection(cfg.velocity)
    _CPU["basis"] = ops.basis_for(cfg.order)


def _cpu_chunk(args):
    """Per-cell reference structure on a contiguous chunk of cells:
    admissible-dt loop, stp_picard per cell, Rusanov per cell side, corrector
    (kernels.py:120-281 restated in oracle/ops.py)."""
    lo, hi, dt = args
    from oracle import ops
    cfg, Q, pde, b = _CPU["cfg"], _CPU["Q"], _CPU["pde"], _CPU["basis"]
    N, d = cfg.cells, cfg.dim
    h = 1.0 / N
    edges = (h,) * d
    t0 = time.perf_counter()
    ops.stable_dt(((h, Q[c]) for c in range(lo, hi)), pde, cfg.order, cfg.cfl, d)
    stores = {c: ops.predictor_picard(Q[c], pde, dt, b, edges) for c in range(lo, hi)}
    strides = [N ** (d - 1 - t) for t in range(d)]
    for c in range(lo, hi):
        idx = [(c // strides[t]) % N for t in range(d)]
        res = {}
        for a in range(d):
            for s in (0, 1):
                j = idx[a] + (1 if s else -1)
                nb = c + ((j % N) - idx[a]) * strides[a]
                other = stores.get(nb, stores[c])
                mine, theirs = stores[c].trace_q[(a, s)], other.trace_q[(a, 1 - s)]
                lo_, hi_ = (mine, theirs) if s == 1 else (theirs, mine)
                res[(a, s)] = ops.rusanov(lo_, hi_, pde, a)
        ops.correct(stores[c], res, b, edges)
    return hi - lo, time.perf_counter() - t0


def cpu_port_rate(cfg_name, cfl, seconds, cores=None, steps=1):
    """DoF-updates/s of the per-cell CPU port on a bounded cell sample; the
    sample is sized for ~`seconds` of wall time per step on `cores` workers."""
    import multiprocessing as mp
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    cfg = cf.CONFIGS[cfg_name] if cfl is None else cf.CONFIGS[cfg_name].with_(cfl=cfl)
    _cpu_init(cfg_name, cfl)
    from oracle import batched
    Q = _CPU["Q"]
    dt = batched.stable_dt_b(Q, 1.0 / cfg.cells, _CPU["pde"], cfg.order, cfg.cfl, cfg.dim)
    cores = cores or os.cpu_count() or 1
    probe = 16
    n_probe, t_probe = _cpu_chunk((0, probe, dt))
    per_cell = t_probe / n_probe
    total = int(max(cores * 4, min(Q.shape[0], seconds * cores / per_cell)))
    chunk = max(1, total // (cores * 4))
    ctx = mp.get_context("fork")
    rates = []
    dof_cell = cfg.m * cfg.n ** cfg.dim
    with ctx.Pool(cores, initializer=_cpu_init, initargs=(cfg_name, cfl)) as pool:
        for k in range(steps):
            start = (k * total) % max(1, Q.shape[0] - total)
            jobs = [(start + i, min(start + i + chunk, start + total), dt) for i in range(0, total, chunk)]
            t0 = time.perf_counter()
            done = sum(n for n, _ in pool.map(_cpu_chunk, jobs))
            rates.append(done * dof_cell / (time.perf_counter() - t0))
    sample = (f"{total} of {Q.shape[0]} cells of step 1 per timed step (per-cell predictor + Rusanov + corrector "
              f"+ dt loop), {cores} worker processes, OPENBLAS_NUM_THREADS=1")
    return rates, cores, sample


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------- reference --

REFARM_FIXTURE = os.path.join(REPO, "tests", "golden", "refarm_{}.npz")


def bench_config(cfg, ncells, ws, steps):
    """The `config` object of both arms (identical by construction)."""
    return {"workload": workload_name(cfg), "cells": ncells, "dof": cf.dof_count(cfg, ncells),
            "cfl_safety": cfg.cfl, "parallelism": f"replicas x{ws} (the path does not shard in this tier)",
            "steps_from_ic": f"1..{steps} (state reset to the initial condition after the warm-up)",
            "l2": ("working set < 126 MB L2: 256 MB write before every timed 2-step chunk (outside the timed "
                   "events)" if l2_flush_needed(cfg) else "working set > 126 MB L2 (state + predictor buffers), no flush")}


def refarm_rate(cfg, steps, seconds_per_step, cores=None, step_ids=None):
    """Reference kernels on stratified samples of trajectory steps (oracle/refarm.py).
    Returns (value, detail) with value = sampled DoF / wall time over the steps."""
    from oracle import refarm
    arm = refarm.RefArm(REFARM_FIXTURE.format(cfg.name), dim=cfg.dim, order=cfg.order, h=1.0 / cfg.cells,
                        cfl=cfg.cfl, cores=cores)
    try:
        per_cell = arm.per_cell_seconds(1)
        total = int(max(arm.cores * 4, seconds_per_step * arm.cores / per_cell))
        dof_cell = cfg.m * cfg.n ** cfg.dim
        ids = list(step_ids if step_ids is not None else range(1, steps + 1))
        cells = its = 0
        wall = 0.0
        for k in ids:
            c, i, w = arm.time_step(k, total)
            cells, its, wall = cells + c, its + i, wall + w
        value = cells * dof_cell / wall
        detail = {"kind": arm.kind, "cores": arm.cores, "picard_iterations_mean": its / cells,
                  "picard_iterations_mean_full_mesh": float(np.mean([arm.mean_iterations(k) for k in ids])),
                  "sample": (f"{total} cells per timed step x {len(ids)} step(s) (trajectory steps "
                             f"{ids[0]}..{ids[-1]}), drawn from tests/golden/refarm_{cfg.name}.npz with each step's "
                             f"Picard-count histogram (largest remainders); per cell: admissible_dt + stp_picard + "
                             f"2d riemann_rusanov + corrector of the "
                             f"{'vendored reference package (oracle/_ref/enclavedg)' if arm.kind == 'reference' else 'numpy port (oracle/ops.py)'}; "
                             f"{arm.cores} worker processes, OPENBLAS_NUM_THREADS=1"),
                  "cpu": cpu_model()}
        return value, detail
    finally:
        arm.close()


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    ncells = cfg.cells ** cfg.dim
    if cfg.kind == "dg" and os.path.exists(REFARM_FIXTURE.format(cfg.name)):
        per_step = max(1.0, min(5.0, 150.0 / max(1, args.steps + args.warmup)))
        # warm-up steps (untimed) on the trajectory's first steps, then the timed ones
        refarm_rate(cfg, args.warmup, 0.5, step_ids=range(1, args.warmup + 1))
        value, det = refarm_rate(cfg, args.steps, per_step)
    elif cfg.kind == "dg":
        per_step = max(1.0, min(5.0, 150.0 / max(1, args.steps + args.warmup)))
        rates, cores, sample = cpu_port_rate(cfg.name, args.cfl, per_step, steps=args.warmup + args.steps)
        value = statistics.median(rates[args.warmup:])
        det = {"kind": "port", "cores": cores, "sample": sample, "cpu": cpu_model()}
    else:
        print(json.dumps({"impl": "reference", "unavailable": "CPU sampler covers the DG configs only"}))
        return
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cf.dof_count(cfg) / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, configs.py)",
        "config": bench_config(cfg, ncells, ws, args.steps),
        "picard_iterations_mean": det.get("picard_iterations_mean"),
        "cpu_baseline": dict(value=value, unit=UNIT, **det),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours --

def l2_flush_needed(cfg):
    """cfg1 (729 cells) and cfg5 (13,121 cells, ~50 MB with the predictor
    buffers) fit in the 126 MB L2; cfg2-4 exceed it several times."""
    return cfg.name in ("cfg1", "cfg5")


def l2_flush_buffer(cfg):
    import torch
    return torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda") if l2_flush_needed(cfg) else None


def measure_device(cfg, steps, warmup, ws, dist, dev, peak64, local):
    """Kernel-resident timing of `steps` consecutive time steps after `warmup`
    steps from the initial state; per-kernel CUDA events on the launching
    stream give the roofline numerators."""
    import torch
    from paper_1806_07984_b200 import solver as S
    solver, Q0, ncells = build_solver(cfg)
    dof = cf.dof_count(cfg, ncells)
    solver.set_state(Q0)
    for _ in range(warmup):
        solver.step()
    # the timed steps are steps 1..K of the stated trajectory
    solver.set_state(Q0)
    torch.cuda.synchronize()
    its0 = int(solver.iter_total.item()) if hasattr(solver, "iter_total") else 0
    timer = S.KernelTimer()
    solver.kernel_timer = timer
    # working sets below the 126 MB L2 (cfg1, cfg5): a 256 MB write evicts L2
    # before every timed chunk, outside the timed events
    flush = l2_flush_buffer(cfg)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)

    def timed(chunks, body):
        if flush is None:
            start.record()
            for _ in range(chunks):
                body()
            stop.record()
            torch.cuda.synchronize()
            return start.elapsed_time(stop)
        total = 0.0
        for _ in range(chunks):
            flush.zero_()
            start.record()
            body()
            stop.record()
            torch.cuda.synchronize()
            total += start.elapsed_time(stop)
        return total

    # pass 1 (eager launches, CUDA events around every hot kernel on the
    # launching stream): the roofline numerators
    # Each eager step starts behind a ~3 ms GPU spin (torch.cuda._sleep) so
    # that the host has enqueued the whole step before its first kernel runs:
    # otherwise, on the small configurations (cfg1, cfg5: tens of us per step)
    # the per-kernel event pairs would include host launch gaps.  The spin is
    # outside every kernel's event pair (ms_eager includes it).
    gate_cycles = int(EAGER_GATE_US * 1965)   # cycles at the 1965 MHz SM clock

    gates = []

    def gated_step():
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record()
        torch.cuda._sleep(gate_cycles)
        g1.record()
        gates.append((g0, g1))
        solver.step()

    ms_eager = max_over_ranks(dist, timed(steps, gated_step), dev)
    # the spins' own durations, measured in place (subtracted for the kernel
    # shares of the step)
    gate_total_ms = sum(g0.elapsed_time(g1) for g0, g1 in gates)
    solver.kernel_timer = None
    tot = timer.totals_ms()
    status = solver.status.cpu().numpy()
    its_timed = int(solver.iter_total.item()) - its0 if hasattr(solver, "iter_total") else 0
    # pass 2 (the production path, DGSolver.run: CUDA-graph replay of the same
    # steps from the same state): the throughput value
    solver.set_state(Q0)
    solver.run(warmup + warmup % 2, graph=True)        # warm-up through the graph itself
    solver.set_state(Q0)
    solver.prepare_graph(2)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        if flush is None:
            ms_graph = timed(1, lambda: solver.run(steps, graph=True))
        else:
            ms_graph = timed(steps // 2, lambda: solver.run(2, graph=True))
            if steps % 2:
                ms_graph += timed(1, lambda: solver.run(1, graph=True))
    if dist:
        dist.barrier()
    ms_max = max_over_ranks(dist, ms_graph, dev)
    ms = ms_eager
    hbm = measured_peaks().get("hbm_gbs")
    kernels, iters_mean = {}, None
    if cfg.kind == "fv":
        n_fv, ms_fv = tot["fv"]
        launches = steps * 2
        cells = cfg.cells ** 3
        ach = costs.fv_cell_bytes(cfg.m) * cells / (ms_fv / n_fv * 1e-3) / 1e9
        kernels["fv_patch"] = {"ms_per_launch": ms_fv / n_fv, "bound": "hbm", "achieved": ach, "unit": "GB/s",
                               "peak": hbm, "frac": ach / hbm if hbm else None,
                               "fp64_tflops": costs.fv_cell_flops("euler") * cells / (ms_fv / n_fv * 1e-3) / 1e12}
        roof = dict(kernels["fv_patch"], kernel="fv_patch")
    else:
        d, n, m = cfg.dim, cfg.n, cfg.m
        its = its_timed
        iters_mean = its / (steps * ncells)
        n_stp, ms_stp = tot["stp"]
        # algorithmic flops: sum over cells of the
        # returned Picard count x the per-iteration count of the reference
        # algorithm, plus the epilogue.  The kernel executes fewer (iteration
        # 1 in its exact reduced form, costs.stp_executed_flops): that rate is
        # reported beside it as executed_tflops / executed_frac.
        flops = its * costs.stp_iter_flops(cfg.pde, d, n, m) + steps * ncells * costs.stp_epilogue_flops(
            cfg.pde, d, n, m)
        flops_exec = costs.stp_executed_flops(cfg.pde, d, n, m, its, steps * ncells)
        ach = flops / (ms_stp * 1e-3) / 1e12
        ach_exec = flops_exec / (ms_stp * 1e-3) / 1e12
        kernels["stp_picard"] = {"ms_per_launch": ms_stp / n_stp, "bound": "fp64", "achieved": ach,
                                 "unit": "TFLOP/s", "peak": peak64, "frac": ach / peak64,
                                 "hbm_gbs": costs.stp_bytes(d, n, m) * ncells / (ms_stp / n_stp * 1e-3) / 1e9,
                                 "flops_per_launch": flops / n_stp,
                                 "executed_tflops": ach_exec, "executed_frac": ach_exec / peak64,
                                 "executed_flops_per_launch": flops_exec / n_stp}
        n_c, ms_c = tot["corrector"]
        cb = costs.corrector_bytes(d, n, m) * ncells / (ms_c / n_c * 1e-3) / 1e9
        kernels["corrector_fused"] = {"ms_per_launch": ms_c / n_c, "bound": "hbm", "achieved": cb, "unit": "GB/s",
                                      "peak": hbm, "frac": cb / hbm if hbm else None}
        # uniform: dt finalize, STP, corrector, 3 ordering kernels; adaptive
        # (cfg5): dt finalize, 2 STP, 2 face solves, restriction, corrector
        launches = steps * (7 if cfg.kind == "dg-amr" else (6 if ncells >= 8192 else 3))
        roof = dict(kernels["stp_picard"], kernel="stp_picard")
    # share of the eager step's GPU time (same pass as the kernel events, spins removed)
    ms_busy = ms_eager - gate_total_ms
    share = {k: v["ms_per_launch"] * steps / ms_busy for k, v in kernels.items()}
    return dict(solver=solver, Q0=Q0, ncells=ncells, dof=dof, ms=ms_max, ms_eager=ms_busy,
                value=dof * steps * ws / (ms_max * 1e-3),
                kernels=kernels, roof=roof, share=share, iters_mean=iters_mean, launches=launches,
                clocks=clocks.summary(), nonfinite_cells=int(status[1]), first_nonfinite_step=int(status[3]) or None)


def run_ours(args, cfg):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = dist_init(ws, "nccl")
    peak64 = fp64_peak_tflops()
    r = measure_device(cfg, args.steps, args.warmup, ws, dist, dev, peak64, local)
    roof = r["roof"]
    traffic = None
    try:
        tr = json.load(open(os.path.join(REPO, "profiles", "traffic.json")))
        traffic = tr.get(cfg.name, {}).get(roof["kernel"])
    except (OSError, ValueError):
        pass
    variant = None
    if cfg.kind != "fv" and cfg.cfl > 0.2 and not args.no_variant:
        v = measure_device(cfg.with_(cfl=0.2), args.steps, args.warmup, ws, dist, dev, peak64, local)
        variant = {"cfl_safety": 0.2, "why": "parity-safe CFL (SURVEY.md section 7 hard part 1)",
                   "value": v["value"], "ms_per_step": v["ms"] / args.steps,
                   "picard_iterations_mean": v["iters_mean"], "nonfinite_cells": v["nonfinite_cells"],
                   "roofline_frac": v["roof"]["frac"], "kernels": v["kernels"]}
        del v
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(r["solver"], r["Q0"], r["dof"], args.steps, ws, dist, dev, args.e2e_slabs)
        if args.e2e_only:
            if rank == 0:
                print(json.dumps({"e2e": e2e, "slabs": args.e2e_slabs}))
            return
    schedule = None
    if cfg.kind == "dg-amr":
        schedule = measure_schedule(cfg, args.steps, args.warmup)
    if schedule and "stp_span_us" in schedule and "stp_picard" in r["kernels"]:
        # the predictor's rate inside the production schedule: both launches'
        # algorithmic flops over their common span (the per-kernel events above
        # time them back to back on one stream)
        k = r["kernels"]["stp_picard"]
        tf = k["flops_per_launch"] / (schedule["stp_span_us"]["median"] * 1e-6) / 1e12
        schedule["stp_two_streams"] = {"achieved": tf, "unit": "TFLOP/s", "peak": peak64, "frac": tf / peak64,
                                       "note": "skeleton + enclave launches overlapped, median span of the launch trace"}
    secondary = None
    if cfg.name == "cfg3" and not args.no_secondary:
        secondary = measure_secondary(ws, dist, dev, peak64, local)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and cfg.kind == "dg":
        if os.path.exists(REFARM_FIXTURE.format(cfg.name)):
            ids = sorted({1, max(1, args.steps // 2), args.steps})
            value, det = refarm_rate(cfg, args.steps, args.cpu_seconds / len(ids), step_ids=ids)
            cpu = dict(value=value, unit=UNIT, **det)
        else:
            rates, cores, sample = cpu_port_rate(cfg.name, args.cfl, args.cpu_seconds, steps=1)
            cpu = {"value": rates[0], "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                   "cpu": cpu_model()}
    if rank == 0:
        line = {
            "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms"] / args.steps,
            "ms_per_step_eager_with_kernel_events": r["ms_eager"] / args.steps,
            "eager_gate_us_per_step": EAGER_GATE_US, "eager_note": "eager pass (per-kernel events) with each step queued behind a GPU spin; spin time removed", "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, configs.py)",
            "config": bench_config(cfg, r["ncells"], ws, args.steps),
            "picard_iterations_mean": r["iters_mean"],
            "nonfinite_cell_results": r["nonfinite_cells"],
            "first_nonfinite_step": r["first_nonfinite_step"],
            "roofline": {"bound": roof["bound"], "achieved": roof["achieved"], "peak": roof["peak"],
                         "unit": roof["unit"], "frac": roof["frac"], "traffic": traffic,
                         "kernel": roof["kernel"],
                         "peak_source": ("fp64: DFMA probe measured in this run (MEASURED_PEAKS.json has no FP64)"
                                         if roof["bound"] == "fp64" else "MEASURED_PEAKS.json hbm_gbs")},
            "kernels": r["kernels"], "kernel_share_of_step": r["share"],
            "fp64_peak_tflops_measured": peak64,
            "gpu_launches": r["launches"],
            "clocks": r["clocks"],
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity_safe_variant": variant,
            "secondary": secondary,
            "schedule": schedule,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def measure_schedule(cfg, steps, warmup):
    """Config 5's schedule: CUDA-graph replay of the two-priority-stream step
    (the production path) against the same steps on one stream, and the
    launch trace of one replayed two-step graph (solver.LaunchTrace): the
    skeleton predictor's head start over the enclave predictor and the
    slack between the end of the skeleton phase (faces + restriction) and the
    end of the enclave predictor (positive = fully hidden)."""
    import torch
    from paper_1806_07984_b200 import solver as S
    out = {}
    flush = l2_flush_buffer(cfg)
    for two in (True, False):
        s, Q0, _ = build_solver(cfg)
        if not two:
            s = S.DGSolver(s.pde, s.order, s.mesh, s.cfl, check_finite=False, two_streams=False)
        s.set_state(Q0)
        s.run(warmup + warmup % 2, graph=True)
        s.set_state(Q0)
        s.prepare_graph(2)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        total = 0.0
        for _ in range(max(1, steps // 2)):
            if flush is not None:
                flush.zero_()
            a.record()
            s.run(2, graph=True)
            b.record()
            torch.cuda.synchronize()
            total += a.elapsed_time(b)
        out["two_streams_ms_per_step" if two else "one_stream_ms_per_step"] = total / (2 * max(1, steps // 2))
        if two:
            s.tracer = S.LaunchTrace()
            s._graph = None
            s.prepare_graph(2)
            heads, slack, spans = [], [], []
            for _ in range(5):
                s.tracer.reset()
                s._graph.replay()
                torch.cuda.synchronize()
                ph = {}
                for ent, _w, sw, t0, t1 in s.tracer.records():
                    ph.setdefault(sw, {})[ent] = (t0, t1)
                for p in ph.values():
                    heads.append((p["EnclaveSTP"][0] - p["SkeletonSTP"][0]) * 1e-3)
                    slack.append((p["EnclaveSTP"][1] - p["Restrict"][1]) * 1e-3)
                    spans.append((max(p["EnclaveSTP"][1], p["SkeletonSTP"][1]) -
                                  min(p["EnclaveSTP"][0], p["SkeletonSTP"][0])) * 1e-3)
            out["skeleton_stp_head_start_us"] = {"min": min(heads), "median": statistics.median(heads)}
            out["skeleton_phase_slack_us"] = {"min": min(slack), "median": statistics.median(slack)}
            # first start to last exit of the two concurrent predictor launches
            # (device clock), with the skeleton faces / restriction running beside them
            out["stp_span_us"] = {"max": max(spans), "median": statistics.median(spans)}
            s.tracer = None
        del s
    out["two_stream_speedup"] = out["one_stream_ms_per_step"] / out["two_streams_ms_per_step"]
    return out


def measure_secondary(ws, dist, dev, peak64, local):
    """BASELINE configs[1] (config 2 at its stated CFL 0.9/(2p+1)) as a line
    item: steps 1..10 from the initial condition, before the reference
    scheme's own blow-up at step 15 (tests/test_gpu_fullsize.py)."""
    cfg = cf.CONFIGS["cfg2"]
    v = measure_device(cfg, 10, 4, ws, dist, dev, peak64, local)
    out = {"workload": workload_name(cfg), "steps_from_ic": "1..10", "value": v["value"], "unit": UNIT,
           "ms_per_step": v["ms"] / 10, "picard_iterations_mean": v["iters_mean"],
           "nonfinite_cell_results": v["nonfinite_cells"], "kernels": v["kernels"],
           "roofline_frac": v["roof"]["frac"]}
    del v
    return out


def pcie_probe(host_a, host_b):
    """This box's host<->device copy rates on the e2e buffers (pinned, up to
    256 MB): H2D alone, D2H alone, and both at once on two streams (GB/s per
    direction) -- the ceiling of the end-to-end number, which moves the whole
    state both ways every step."""
    import torch
    n = min(host_a.numel(), 32 << 20)
    a, b = host_a.reshape(-1)[:n], host_b.reshape(-1)[:n]
    d1 = torch.empty(n, dtype=host_a.dtype, device="cuda")
    d2 = torch.empty(n, dtype=host_a.dtype, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nbytes = n * host_a.element_size()

    def timed(fn, reps=3):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            s1.synchronize()
            s2.synchronize()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        return nbytes / (best * 1e-3) / 1e9

    def h2d():
        with torch.cuda.stream(s1):
            d1.copy_(a, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            b.copy_(d2, non_blocking=True)

    def both():
        h2d()
        d2h()

    saved = b.clone()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    out = {"h2d": timed(h2d), "d2h": timed(d2h), "duplex_per_direction": timed(both), "bytes": nbytes}
    b.copy_(saved)
    torch.cuda.synchronize()
    return out


def measure_e2e(solver, Q0, dof, steps, ws, dist, dev, slabs=None):
    """Public API with host buffers: every step uploads the state from pinned
    host memory (set_state), advances one step, downloads the result."""
    import torch
    host = torch.from_numpy(np.ascontiguousarray(Q0)).pin_memory()
    out = torch.empty_like(host).pin_memory()
    nb = host.numel() * 8
    streamed = hasattr(solver, "step_host") and not getattr(solver, "adaptive", False)

    def one(src, dst):
        if streamed:
            # host state in, host state out, slabs streamed (uploads, kernels
            # and downloads overlapped; dt reduced from the uploaded state)
            solver.step_host(src, dst, **({} if slabs is None else {"slabs": slabs}))
        else:
            solver.set_state(src)
            solver.step()
            dst.copy_(solver.state().reshape(dst.shape), non_blocking=True)

    one(host, out)
    if streamed:
        solver.host_wait()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        one(host, out)
        host, out = out, host
    if streamed:
        solver.host_wait()     # the last step's downloads are inside the timed region
    b.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(dist, a.elapsed_time(b), dev)
    pcie = pcie_probe(host, out)
    api = (f"{type(solver).__name__}.step_host(pinned host in, pinned host out): slab-streamed H2D / kernels / D2H, "
           "dt from the uploaded state" if streamed else
           "set_state(pinned host) + step() + copy to pinned host")
    return {"value": dof * steps * ws / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": nb,
            "d2h_bytes_per_step": nb, "ms_per_step": ms / steps, "api": api, "pcie_gbs": pcie,
            "pcie_floor_ms_per_step": (nb / (pcie["duplex_per_direction"] * 1e9) * 1e3
                                       if pcie and pcie.get("duplex_per_direction") else None)}


def main():
    args = parse()
    if args.lib:
        from paper_1806_07984_b200 import _lib
        _lib.load(args.lib)
    cfg = cf.CONFIGS[args.config]
    if args.cfl is not None:
        cfg = cfg.with_(cfl=args.cfl)
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    run_ours(args, cfg)


if __name__ == "__main__":
    main()
