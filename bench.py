#!/usr/bin/env python
"""bench.py -- Gpoints/s of the acoustic_iso_cd propagator on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--grid 240] [--mode fast|strict|fast_fma] [--radius 4]
                    [--scaling weak|strong] [--propagator acoustic_iso_cd|acoustic_iso]
                    [--tune name=value ...]

N > 1 (torchrun, or spawned by bench.py itself when WORLD_SIZE is unset): one
rank per GPU through the C++ z-slab group (mm_cd_group_run: NCCL halo planes
overlapped with the interior), weak scaling at 240^3 per GPU by default;
--scaling strong --grid 512|1000 fixes the global grid (BASELINE configs[2],
configs[3]) and adds the parallel efficiency of bench.cpp:130-145 against one
GPU on the same grid.

A "step" is one time step of the propagator over the whole grid (the
reference's eng.step(), driver.cpp:104-106).  Workload at N=1: BASELINE.json
configs[1] -- 240^3 grid, 8th order (r=4), CPML nd=27, taper, Ricker source at
the centre, 240^2 surface receivers at k=27, default two-layer model
(synthetic, vp 1500/4500).  Metric: Gpoints/s = n^3 * K / (device time of K
steps), the reference's points_per_s (bench.cpp:184-186).

Timed region (value): K steps of the device-resident loop (mm_cd_run: source
injection from a device wavelet, per-step receiver recording and finiteness
check) bracketed by barrier + synchronize, timed with CUDA events on the
engine's stream, max over ranks.  The working set (3 pressure fields + c +
CPML memory, ~290 MB at 240^3) exceeds the 126 MB L2, so no flush is needed.

e2e: the same K steps driven step by step through the public C ABI with host
buffers: mm_cd_step(amp from host), mm_cd_record, and a D2H copy of that
step's receiver samples into pinned host memory every step.

--impl reference: the reference's own CPU implementation (oracle/_ref, its
sources compiled unmodified; run() with Target::Parallel and all host
threads) on the same workload for a bounded sample of steps.  Under torchrun
only rank 0 runs it.
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

from pathlib import Path

import numpy as np

# before any CUDA context exists (see paper_2007_06048_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Gpoints/s (grid-point updates/sec) acoustic_iso_cd 8th-order"
UNIT = "Gpoints/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)  # configs[1]: 240^3 x 1000 steps
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", type=int, default=None, help="cube edge (default: config per N)")
    ap.add_argument("--mode", default="fast", choices=["fast", "strict", "fast_fma"])
    ap.add_argument("--tune", action="append", default=[],
                    help="name=value tuning parameter (mm_set_tuning), repeatable")
    ap.add_argument("--radius", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-steps", type=int, default=None)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = 240^3 per GPU (grid 240 x 240 x 240 N); strong = the "
                         "--grid^3 global grid (default 1000) cut into N z-slabs")
    ap.add_argument("--no-efficiency", dest="efficiency", action="store_false",
                    help="strong scaling: skip the one-GPU baseline on the same grid")
    ap.add_argument("--propagator", default="acoustic_iso_cd",
                    choices=["acoustic_iso_cd", "acoustic_iso"],
                    help="acoustic_iso: the variable-density engine (SURVEY 8(f) row 4)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ model
def byte_model(n, nd, r=4):
    """Algorithmic bytes per step: 16 B/pt + 16 B per
    damped-axis point (psi and zeta read + write)."""
    N = float(n[0]) * n[1] * n[2]
    damped = sum(N * 2 * nd[a] / n[a] for a in range(3))
    return 16.0 * N + 16.0 * damped, N, damped


def kernel_bytes(n, nd, r=4, nrec=0):
    """Algorithmic bytes per launch of the step kernels:
      cpml     16 B per slab point (p_cur, p_prev, c read; p_next write) + 16 B
               per damped-axis point (psi and zeta read + write): the fused
               one-pass CPML kernel, exactly the byte model's damping share
      inner    16 B per inner-box point (p_cur, p_prev, c read; p_next write)
      epilogue 12 B per receiver (offset read, sample read + write)
    and of the two-pass path (layouts k_cpml does not serve):
      boundary 16 B per slab point + 12 B per damped-axis point (psi or dpsi_z
               read, zeta read + write)
      pass1    8 B per damped-axis point (psi read + write) + 4 B per slab
               point (p_cur read) + 4 B per dpsi_z point written (the z runs
               widened by R planes on both sides)"""
    N = float(n[0]) * n[1] * n[2]
    damped = sum(N * 2 * nd[a] / n[a] for a in range(3))
    inner = float(np.prod([n[a] - 2 * nd[a] for a in range(3)]))
    slab = N - inner
    dpz = 2.0 * (nd[2] + 2 * r) * n[0] * n[1] if nd[2] > 0 else 0.0
    return {"cpml": 16.0 * slab + 16.0 * damped, "inner": 16.0 * inner,
            "epilogue": 12.0 * nrec,
            "boundary": 16.0 * slab + 12.0 * damped,
            "pass1": 8.0 * damped + 4.0 * slab + 4.0 * dpz}


# ------------------------------------------------------------------ clocks
from paper_2007_06048_b200.clocks import ClockSampler  # noqa: E402


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload, kernel):
    """dram read+write bytes per launch of `kernel` from the committed ncu
    summary (profiles/ncu_summary.json, `ncu --set full` captures by
    tools/refresh_profiles.sh); "pass1" sums its x/y and z launches."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text()).get(workload, {})
        if kernel == "pass1" and "pass1_z" in d:
            return sum(d[k]["dram_bytes_per_launch"] for k in ("pass1_z", "pass1_xy") if k in d)
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------ CPU legs
def cpu_reference_run(n, nsteps, nthreads, propagator="acoustic_iso_cd", want_traces=False):
    from oracle.oracle import Oracle, available, nproc
    kind = "reference" if available("reference") else "port"
    o = Oracle(kind)
    vp, vmin, vmax = o.layered_model(n)
    if propagator == "acoustic_iso":
        rho = np.full_like(vp, 1000.0)  # default_layered_model's rho (model.cpp:63-77)
        if kind == "reference":
            out = o.run_vd(n, vp, rho, nsteps=nsteps, nthreads=nthreads)
            threads = nthreads
        else:
            out = o.run_vd(n, vp, rho, nsteps=nsteps, vmax=vmax)
            threads = 1
    elif kind == "reference":
        out = o.run(n, vp, nsteps=nsteps, nthreads=nthreads)
        threads = nthreads
    else:
        out = o.run(n, vp, nsteps=nsteps)
        threads = 1
    gpts = n[0] * n[1] * n[2] * nsteps / out["kernel_seconds"] / 1e9
    if want_traces:
        return gpts, kind, threads, out["kernel_seconds"], out["traces"]
    return gpts, kind, threads, out["kernel_seconds"]


def trace_parity(mm, n, nsteps, ref_traces, mode):
    """The GPU engine's run() (the device loop, mm_run) on the CPU baseline's
    own workload and steps against the reference's trace matrix: rel L2,
    max-abs and bit equality (north_star: rel L2 <= 1e-5, max-abs reported)."""
    cfg = mm.SimConfig(ngrid=n, nsteps=nsteps)
    model = mm.default_layered_model(mm.make_grid(n, cfg.dgrid))
    rec, _ = mm.run(cfg, model, mode=mode)
    got = rec.traces.astype(np.float64)
    want = ref_traces.astype(np.float64)
    diff = np.abs(got - want)
    return {"rel_l2": float(np.linalg.norm(diff) / max(np.linalg.norm(want), 1e-300)),
            "max_abs": float(diff.max()), "steps": nsteps, "receivers": int(want.shape[0]),
            "bitwise": bool(np.array_equal(rec.traces, ref_traces)),
            "vs": "the reference's run() traces (oracle/_ref, full receiver matrix)"}


def cpu_sample_steps(n, requested):
    if requested:
        return requested
    pts = n[0] * n[1] * n[2]
    # ~0.1-0.2 Gpts/s on a multi-core host: aim at ~10-20 s of CPU work
    return max(2, min(100, int(2.0e9 / pts)))


# ------------------------------------------------------------------ our arm
def workload_grid(args, world):
    """BASELINE configs[1] per GPU: 240^3 at N = 1; weak scaling at N > 1 grows
    z, 240 x 240 x 240 N; strong scaling keeps --grid^3 (default 1000^3) for
    every N (the multi-GPU leg in dist.bench_rank uses the same)."""
    if args.scaling == "strong":
        edge = args.grid or 1000
        return (edge, edge, edge)
    edge = args.grid or 240
    return (edge, edge, edge * world)


def run_ours(args):
    rank, world, local = dist_env()
    if world > 1 or os.environ.get("MM_BENCH_ZSLAB") == "1":  # (world 1: the z-slab leg alone)
        from paper_2007_06048_b200 import dist as mmdist
        return mmdist.bench_rank(args, rank, world, local)
    if args.scaling == "strong" and args.grid is None:
        args.grid = 1000  # BASELINE configs[3] at N = 1 (the strong-scaling baseline)
    import torch
    import paper_2007_06048_b200 as mm
    from paper_2007_06048_b200 import _lib

    n = workload_grid(args, world)
    edge = n[0]
    r = args.radius
    nd = (27, 27, 27)
    torch.cuda.set_device(local)
    grid = mm.make_grid(n, (20.0, 20.0, 20.0), r)
    model = mm.default_layered_model(grid)
    dt = mm.cfl_dt(model, grid, 0.8)
    total = args.warmup + args.steps
    w = mm.ricker(25.0, dt, total).samples
    src = tuple(x // 2 for x in n)
    eng = mm.AcousticCdEngine(grid, (0, 0, 0), n, model.vp,
                              mm.EngineOptions(ndamping=nd, taper=True), dt, model.vmax,
                              device=local, mode=args.mode)
    geo = mm.default_receivers(grid, nd)
    eng.set_receivers(geo.receivers, total)
    nrec = geo.nreceivers()
    ext = torch.cuda.ExternalStream(eng.stream_handle(), device=local)

    # clock ramp (untimed): a throw-away engine steps for >= 0.3 s so the SM
    # clocks have left their idle state before the W warm-up steps
    ramp = mm.AcousticCdEngine(grid, (0, 0, 0), n, model.vp,
                               mm.EngineOptions(ndamping=nd, taper=True), dt, model.vmax,
                               device=local, mode=args.mode)
    t_ramp = time.perf_counter()
    while time.perf_counter() - t_ramp < 0.3:
        ramp.run(w[:min(total, 50)], src, record=False, first_sample=0)
        ramp.synchronize()
    del ramp
    # warm-up (untimed) through the same device loop
    eng.run(w[:args.warmup], src, record=True, first_sample=0)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.kernel_launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(ext)
    eng.run(w[args.warmup:total], src, record=True, first_sample=args.warmup)
    t1.record(ext)
    t1.synchronize()
    torch.cuda.synchronize()
    launches = _lib.kernel_launch_count() - launches0
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    pts = float(n[0]) * n[1] * n[2]
    value = pts * args.steps / (ms * 1e-3) / 1e9

    # per-kernel durations inside the real step (the CPML and interior kernels
    # concurrent on their two streams): K more steps of the same device loop,
    # every kernel bracketed by CUDA events on the stream it is launched on
    eng.kernel_timing(True)
    eng.run(w[args.warmup:total], src, record=False)
    kt = eng.kernel_times()
    eng.kernel_timing(False)
    torch.cuda.synchronize()
    kms = {k: v[0] / v[1] for k, v in kt.items() if v[1] > 0}
    klaunch = {k: int(v[1]) for k, v in kt.items()}
    cpml_path = eng.cpml_path()
    # e2e through the public API with host buffers, on the same engine (the
    # wavefield just continues): a second engine would add a second set of
    # streams and allocations, whose placement alone moved a 240^3 step
    # between 137 and 147 us
    eng2 = eng
    host_out = torch.empty((args.steps, nrec), dtype=torch.float32, pin_memory=True).numpy()
    for s in range(args.warmup):
        eng2.step(float(w[s]), src)
        eng2.record(s)
    eng2.synchronize()
    ext2 = torch.cuda.ExternalStream(eng2.stream_handle(), device=local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    e0.record(ext2)
    for s in range(args.warmup, total):
        eng2.step(float(w[s]), src)       # 4 B of input per step (the source sample)
        eng2.record(s)
        eng2.copy_trace_step(s, host_out[s - args.warmup], asynchronous=True)
    e1.record(ext2)
    eng2.synchronize()
    wall = time.perf_counter() - wall0
    e2e_ms = max(e0.elapsed_time(e1), wall * 1e3)
    e2e = pts * args.steps / (e2e_ms * 1e-3) / 1e9
    print(f"e2e: device {e0.elapsed_time(e1):.2f} ms, wall {wall * 1e3:.2f} ms over {args.steps} "
          f"steps", file=sys.stderr)

    peak, peak_src = measured_peak()
    kb = kernel_bytes(n, nd, r, nrec)
    dominant = max(kms, key=kms.get)
    achieved = kb[dominant] / (kms[dominant] * 1e-3) / 1e9
    step_bytes, _, _ = byte_model(n, nd)
    step_gbs = step_bytes * args.steps / (ms * 1e-3) / 1e9
    traffic = ncu_traffic(f"{edge}^3" + ("" if r == 4 else f" r{r}"), dominant)
    per_kernel = {k: {"ms": round(kms[k], 4), "launches": klaunch[k],
                      "algorithmic_bytes": kb.get(k),
                      "achieved_gbs": (round(kb[k] / (kms[k] * 1e-3) / 1e9, 1)
                                       if k in kb else None)} for k in kms}

    from paper_2007_06048_b200.scaling import count_stencil_cost
    cost = count_stencil_cost("acoustic_iso_cd", r)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (default two-layer vp model 1500/4500, Ricker source)",
        "config": {"workload": f"acoustic_iso_cd r={r} {edge}^3 grid, nd=27 CPML, taper, "
                               f"{nrec} surface receivers"
                               + (" (BASELINE configs[1])" if edge == 240 and r == 4 else
                                  " (BASELINE configs[2])" if edge == 512 and r == 4 else
                                  " (BASELINE configs[3] at N = 1)" if edge == 1000 else
                                  " (BASELINE configs[4] radius sweep)" if edge == 512 else ""),
                   "grid": list(n), "radius": r, "ndamping": list(nd), "mode": args.mode,
                   "cpml_path": cpml_path,
                   "flops_per_point": cost.flops_per_point,
                   "arithmetic_intensity": round(cost.arithmetic_intensity, 4),
                   "l2": "working set (3 p fields + c + CPML) > 126 MB L2; no flush"},
        "e2e": {"value": round(e2e, 3), "unit": UNIT, "h2d_bytes_per_step": 4,
                "d2h_bytes_per_step": 4 * nrec},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "kernel": dominant,
                     "algorithmic_bytes_per_launch": kb[dominant],
                     "kernel_ms": round(kms[dominant], 4), "peak_source": peak_src},
        "kernels": per_kernel,
        "step_roofline": {"bytes_per_step_model": step_bytes,
                          "achieved_gbs": round(step_gbs, 1),
                          "frac": round(step_gbs / peak, 4),
                          "roofline_gpts": round(peak * 1e9 / (step_bytes / pts) / 1e9, 1)},
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        ns = cpu_sample_steps(n, args.cpu_sample_steps)
        from oracle.oracle import nproc
        cores = nproc()
        gpts, kind, threads, secs, ref_tr = cpu_reference_run(n, ns, cores, want_traces=True)
        line["cpu_baseline"] = {"value": round(gpts, 5), "unit": UNIT, "cores": threads,
                                "kind": kind,
                                "sample": f"{edge}^3 x {ns} steps from t=0 ({secs:.1f} s), "
                                          "run() Target::Parallel"}
        line["parity"] = trace_parity(mm, n, ns, ref_tr, args.mode)
    print(json.dumps(line), flush=True)
    return 0


VD_METRIC = "Gpoints/s (grid-point updates/sec) acoustic_iso 8th-order"


def vd_kernel_bytes(n, nd):
    """Compulsory bytes per launch of k_vdv / k_vdp (vd_engine.cu): velocity
    reads p, dt/rho, v and writes v (32 B/pt), pressure reads v, dt*bulk, p and
    writes p (24 B/pt); plus 8 B (psi r+w) per damping-layer point and axis."""
    N = n[0] * n[1] * n[2]
    lay = sum(2 * nd[a] * N // n[a] for a in range(3))
    return {"velocity": 32 * N + 8 * lay, "pressure": 24 * N + 8 * lay}


def run_vd(args):
    """The acoustic_iso leg: same contract as run_ours (N = 1)."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    import torch
    import paper_2007_06048_b200 as mm
    from paper_2007_06048_b200 import _lib

    edge = args.grid or 240
    n = (edge, edge, edge)
    nd = (27, 27, 27)
    torch.cuda.set_device(local)
    grid = mm.make_grid(n, (20.0, 20.0, 20.0), args.radius)
    model = mm.default_layered_model(grid)
    dt = mm.cfl_dt(model, grid, 0.8)
    total = args.warmup + args.steps
    w = mm.integrate_wavelet(mm.ricker(25.0, dt, total)).samples
    src = tuple(x // 2 for x in n)
    opts = mm.EngineOptions(ndamping=nd, taper=True)
    geo = mm.default_receivers(grid, nd)
    nrec = geo.nreceivers()
    eng = mm.AcousticVdEngine(grid, model, opts, dt, device=local)
    eng.set_receivers(geo.receivers, total)
    ext = torch.cuda.ExternalStream(eng.stream_handle(), device=local)
    t_ramp = time.perf_counter()
    while time.perf_counter() - t_ramp < 0.3:
        eng.run(w[:min(total, 50)], src, record=False)
        eng.synchronize()
    del eng
    eng = mm.AcousticVdEngine(grid, model, opts, dt, device=local)
    eng.set_receivers(geo.receivers, total)
    ext = torch.cuda.ExternalStream(eng.stream_handle(), device=local)
    eng.run(w[:args.warmup], src, record=True, first_sample=0)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.kernel_launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(ext)
    eng.run(w[args.warmup:total], src, record=True, first_sample=args.warmup)
    t1.record(ext)
    t1.synchronize()
    launches = _lib.kernel_launch_count() - launches0
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    pts = float(n[0]) * n[1] * n[2]
    value = pts * args.steps / (ms * 1e-3) / 1e9
    # per-kernel durations (CUDA events on the engine stream)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    for s in range(args.steps):
        ev[s][0].record(ext)
        eng.update_velocity()
        ev[s][1].record(ext)
        eng.update_pressure()
        ev[s][2].record(ext)
        eng.inject_source(float(w[s % total]), src)
    torch.cuda.synchronize()
    kms = {k: statistics.mean(e[i].elapsed_time(e[i + 1]) for e in ev)
           for i, k in enumerate(("velocity", "pressure"))}
    # e2e through the public API with host buffers
    eng2 = mm.AcousticVdEngine(grid, model, opts, dt, device=local)
    eng2.set_receivers(geo.receivers, total)
    host_out = torch.empty((args.steps, nrec), dtype=torch.float32, pin_memory=True).numpy()
    for s in range(args.warmup):
        eng2.step(float(w[s]), src)
        eng2.record(s)
    eng2.synchronize()
    ext2 = torch.cuda.ExternalStream(eng2.stream_handle(), device=local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    e0.record(ext2)
    for s in range(args.warmup, total):
        eng2.step(float(w[s]), src)
        eng2.record(s)
        eng2.copy_trace_step(s, host_out[s - args.warmup], asynchronous=True)
    e1.record(ext2)
    eng2.synchronize()
    wall = time.perf_counter() - wall0
    e2e_ms = max(e0.elapsed_time(e1), wall * 1e3)
    e2e = pts * args.steps / (e2e_ms * 1e-3) / 1e9

    peak, peak_src = measured_peak()
    kb = vd_kernel_bytes(n, nd)
    dominant = max(kms, key=kms.get)
    achieved = kb[dominant] / (kms[dominant] * 1e-3) / 1e9
    ref_model = 40 * pts  # the reference's fused cost model (bench.cpp:97)
    step_gbs = ref_model * args.steps / (ms * 1e-3) / 1e9
    line = {
        "metric": VD_METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (default two-layer model: vp 1500/4500, rho 1000; integrated Ricker)",
        "config": {"workload": f"acoustic_iso r={args.radius} {edge}^3 grid, nd=27 CPML, taper, "
                               f"{nrec} surface receivers", "grid": list(n),
                   "radius": args.radius, "ndamping": list(nd),
                   "l2": "working set (p, v, dt/rho, dt*bulk, CPML) > 126 MB L2; no flush"},
        "e2e": {"value": round(e2e, 3), "unit": UNIT, "h2d_bytes_per_step": 4,
                "d2h_bytes_per_step": 4 * nrec},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": ncu_traffic(f"vd_{edge}^3", dominant), "kernel": dominant, "algorithmic_bytes_per_launch": kb[dominant],
                     "kernel_ms": round(kms[dominant], 4), "peak_source": peak_src},
        "kernels": {k: {"ms": round(kms[k], 4), "algorithmic_bytes": kb[k],
                        "achieved_gbs": round(kb[k] / (kms[k] * 1e-3) / 1e9, 1)} for k in kms},
        "step_roofline": {"bytes_per_step_model": ref_model,
                          "model": "reference cost model 40 B/pt (bench.cpp:97)",
                          "achieved_gbs": round(step_gbs, 1), "frac": round(step_gbs / peak, 4),
                          "roofline_gpts": round(peak / 40, 1)},
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        ns = cpu_sample_steps(n, args.cpu_sample_steps)
        from oracle.oracle import nproc
        gpts, kind, threads, secs = cpu_reference_run(n, ns, nproc(), "acoustic_iso")
        line["cpu_baseline"] = {"value": round(gpts, 5), "unit": UNIT, "cores": threads,
                                "kind": kind,
                                "sample": f"{edge}^3 x {ns} steps from t=0 ({secs:.1f} s), "
                                          "run(AcousticIso) Target::Parallel"}
    print(json.dumps(line), flush=True)
    return 0


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    n = workload_grid(args, world)
    from oracle.oracle import nproc
    cores = nproc()
    ns = max(1, min(args.steps, cpu_sample_steps(n, args.cpu_sample_steps)))
    # warm-up: one short run (page in, thread start-up)
    cpu_reference_run(n, max(1, min(args.warmup, 2)), cores, args.propagator)
    gpts, kind, threads, secs = cpu_reference_run(n, ns, cores, args.propagator)
    vd = args.propagator == "acoustic_iso"
    line = {
        "impl": "reference", "metric": VD_METRIC if vd else METRIC, "value": round(gpts, 5), "unit": UNIT,
        "n_gpus": world, "steps": ns, "warmup": args.warmup,
        "ms_per_step": secs * 1e3 / ns, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (default two-layer model)",
        "config": {"workload": f"{args.propagator} r=4 {n[0]}x{n[1]}x{n[2]} grid, nd=27 CPML, "
                               f"taper (bounded sample: {ns} steps from t=0)", "grid": list(n)},
        "cpu_baseline": {"value": round(gpts, 5), "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{n[0]}x{n[1]}x{n[2]} x {ns} steps, run("
                                   f"{'AcousticIso' if vd else 'AcousticIsoCd'}) Target::Parallel"},
        "e2e": {"value": round(gpts, 5), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` started without torchrun: launch N ranks (one per
    GPU) through torch.distributed.run on this node and relay their output."""
    import socket
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        have = 0
    if args.impl == "ours" and have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but {have} CUDA device(s) visible", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.gpus > 1:
        # NCCL init lines (ranks, transports) on stderr; stdout keeps the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.tune:
        from paper_2007_06048_b200 import _lib
        for kv in args.tune:
            k, v = kv.split("=")
            _lib.set_tuning(k, int(v))
    if args.impl == "reference":
        return run_reference(args)
    if args.propagator == "acoustic_iso":
        return run_vd(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
