"""Metric definitions of the reference's scaling study.

ref: bench.cpp:87-107 count_stencil_cost, :109-128 weak_scaling_plan,
:130-145 compute_efficiency, :162-195 run_scaling (bench.hpp:40-100).  Pure
host arithmetic: bench.py reports these beside the measured Gpoints/s.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

from ._lib import ConfigError


@dataclass
class KernelCostModel:  # ref: bench.hpp:40-44
    flops_per_point: int
    bytes_per_point: int
    arithmetic_intensity: float


def count_stencil_cost(propagator: str, radius: int) -> KernelCostModel:
    """ref: bench.cpp:87-107 (the counted replays of bench.cpp:22-79).

    acoustic_iso_cd: per axis and tap `acc += w * (p + p - two * c)` = 5
    operations; the three axes summed (2); `2 pc - pp + dt2 vp vp lap` (6):
    15 r + 8.  acoustic_iso: staggered taps `acc += w * (f - f)` = 3 per tap on
    6 derivatives, `dt / rho` (1), three `v += inv_rho * d` (6), `rho vp vp`
    (2), `p += dt bulk (dx + dy + dz)` (5): 18 r + 14.  Bytes: one access per
    array touched, 16 and 40 B/pt (bench.cpp:93,97)."""
    if radius < 1 or radius > 8:
        raise ConfigError("stencil radius must be in [1, 8]")
    if propagator == "acoustic_iso_cd":
        flops, nbytes = 3 * 5 * radius + 2 + 6, 16
    elif propagator == "acoustic_iso":
        flops, nbytes = 6 * 3 * radius + 1 + 6 + 2 + 5, 40
    else:
        raise ConfigError(f"no cost model for propagator {propagator!r}")
    return KernelCostModel(flops, nbytes, flops / nbytes)


def weak_scaling_plan(base: int, ranks: Sequence[int], mode: str = "ideal"
                      ) -> List[Tuple[int, Tuple[int, int, int]]]:
    """ref: bench.cpp:109-128.  ideal: (r base, base, base); practical: a cube
    of r x the baseline volume, side rounded up to a multiple of 64 (the
    baseline itself never rounded)."""
    if base < 1:
        raise ConfigError("weak-scaling base size must be >= 1")
    plan = []
    for r in ranks:
        if r < 1:
            raise ConfigError("rank counts must be >= 1")
        if mode == "ideal":
            plan.append((r, (r * base, base, base)))
        elif r == 1:
            plan.append((r, (base, base, base)))
        else:
            side = base * (r ** (1.0 / 3.0))
            rounded = int(math.ceil(side / 64.0)) * 64
            plan.append((r, (rounded, rounded, rounded)))
    return plan


@dataclass
class ScalingRun:  # ref: bench.hpp:60-74
    ranks: int
    n: Tuple[int, int, int]
    nsteps: int
    kernel_s: float = 0.0
    modeling_s: float = 0.0
    points_per_s: float = 0.0
    efficiency_pct: float = 0.0
    ok: bool = True
    error: str = ""
    run_id: str = ""


@dataclass
class ScalingResult:
    mode: str = "strong"  # "strong" | "weak_ideal" | "weak_practical"
    runs: List[ScalingRun] = field(default_factory=list)


def compute_efficiency(result: ScalingResult) -> None:
    """ref: bench.cpp:130-145 -- against runs[0]:
    strong: t0 r0 / (ti ri); weak: t0 points_i / (ti ri points_0).  Failed runs
    keep 0."""
    if not result.runs:
        return
    b = result.runs[0]
    if not b.ok or b.kernel_s <= 0.0:
        return
    pts0 = float(b.n[0]) * b.n[1] * b.n[2]
    for run in result.runs:
        if not run.ok or run.kernel_s <= 0.0:
            continue
        pts = float(run.n[0]) * run.n[1] * run.n[2]
        if result.mode == "strong":
            eff = b.kernel_s * b.ranks / (run.kernel_s * run.ranks)
        else:
            eff = b.kernel_s * pts / (run.kernel_s * run.ranks * pts0)
        run.efficiency_pct = 100.0 * eff


def run_scaling(plan, nsteps: int, mode: str,
                executor: Callable[[Tuple[int, int, int], int], Tuple[float, float]]
                ) -> ScalingResult:
    """ref: bench.cpp:162-195 -- run each (ranks, n) of the plan through
    `executor(n, ranks) -> (kernel_s, modeling_s)`, record failures and keep
    sweeping, then compute the efficiencies."""
    res = ScalingResult(mode=mode)
    for ranks, n in plan:
        run = ScalingRun(ranks=ranks, n=tuple(n), nsteps=nsteps,
                         run_id=f"r{ranks}_{n[0]}x{n[1]}x{n[2]}")
        try:
            k, m = executor(tuple(n), ranks)
            run.kernel_s, run.modeling_s = k, m
            if k > 0:
                run.points_per_s = float(n[0]) * n[1] * n[2] * nsteps / k
        except Exception as e:  # noqa: BLE001 -- recorded, as the reference does
            run.ok = False
            run.error = str(e)
        res.runs.append(run)
    compute_efficiency(res)
    return res
