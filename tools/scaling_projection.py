"""Projected strong / weak scaling from single-GPU measurements (no multi-GPU
box was available in this run; these are NOT multi-GPU measurements).

For each N and global grid: the cost-weighted legal z cuts of bench.py
--gpus N; every rank's slab timed alone on this GPU as an engine with its
global offset (its own CPML share, ghost planes zero), K steps of the device
loop; t_N = max over ranks.  The schedule overhead of the multi-rank C++ group
(edge planes on their own stream, halo transfer, interior) is measured on this
GPU too: N in-process ranks stepping together (mm_cd_group_step_local) against
one engine on the same grid -- both run all the work on one GPU, so their
ratio is the schedule's cost, not a communication time.  NVLink time for the
halo planes (r planes of nx*ny floats per neighbour, 16 MB at 1000^2) is
overlapped with the interior in the schedule and is reported separately at
the measured 770 GB/s peer bandwidth (B200_PROFILING.md).

    python tools/scaling_projection.py [--grids 512,1000] [--ranks 2,4,8] [--steps 10]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import paper_2007_06048_b200 as mm  # noqa: E402
from paper_2007_06048_b200 import dist as D  # noqa: E402
from paper_2007_06048_b200.propagator import ZSlabGroup, step_local  # noqa: E402
from paper_2007_06048_b200.scaling import ScalingResult, ScalingRun, compute_efficiency  # noqa: E402


def time_engine(n_glob, z0, nz, steps, nd=(27, 27, 27), r=4):
    grid = mm.make_grid(n_glob, (20.0, 20.0, 20.0), r)
    lg = mm.make_grid((n_glob[0], n_glob[1], nz), (20.0, 20.0, 20.0), r)
    dt = float(np.float32(D.cfl_dt_vmax(4500.0, grid, 0.8)))
    vp = D.layered_slice(n_glob, z0, nz, r)
    e = mm.AcousticCdEngine(lg, (0, 0, z0), n_glob, vp, mm.EngineOptions(ndamping=nd, taper=True),
                            dt, 4500.0)
    w = np.zeros(steps, np.float32)
    e.run(w[:3], None, record=False)
    ms = e.run(w, None, record=False)
    e.close()
    return ms / steps


def time_inprocess(n_glob, cuts, steps, nd=(27, 27, 27), r=4):
    import torch
    grid = mm.make_grid(n_glob, (20.0, 20.0, 20.0), r)
    dt = float(np.float32(D.cfl_dt_vmax(4500.0, grid, 0.8)))
    opts = mm.EngineOptions(ndamping=nd, taper=True)
    gs = [ZSlabGroup(grid, cuts, k, None, opts, dt, 4500.0,
                     vp_local=D.layered_slice(n_glob, cuts[k], cuts[k + 1] - cuts[k], r))
          for k in range(len(cuts) - 1)]
    for _ in range(3):
        step_local(gs, 0.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        step_local(gs, 0.0)
    for g in gs:
        g.engine.synchronize()
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) * 1e3 / steps
    for g in gs:
        g.close()
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grids", default="512,1000")
    ap.add_argument("--ranks", default="2,4,8")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    out = {"note": "projection from single-GPU timings, not a multi-GPU measurement"}
    for edge in [int(x) for x in a.grids.split(",")]:
        n = (edge, edge, edge)
        t1 = time_engine(n, 0, edge, a.steps)
        ent = {"one_gpu_ms_per_step": round(t1, 4), "ranks": {}}
        for N in [int(x) for x in a.ranks.split(",")]:
            cuts = D.weighted_cuts(n, (27, 27, 27), 4, N)
            per = [time_engine(n, cuts[k], cuts[k + 1] - cuts[k], a.steps) for k in range(N)]
            tN = max(per)
            # schedule overhead: N in-process ranks vs one engine, same grid, one GPU
            tl = time_inprocess(n, cuts, a.steps) if edge <= 512 else None
            ov = tl / t1 if tl else None
            halo_us = 2 * 4 * edge * edge * 4 / 770e9 * 1e6  # both neighbours, r = 4 planes
            res = ScalingResult("strong", [ScalingRun(1, n, 1, kernel_s=t1),
                                           ScalingRun(N, n, 1, kernel_s=tN)])
            compute_efficiency(res)
            ent["ranks"][N] = {"cuts": cuts, "rank_ms_per_step": [round(x, 4) for x in per],
                               "t_N_ms": round(tN, 4),
                               "projected_gpts": round(edge ** 3 / (tN * 1e-3) / 1e9, 1),
                               "projected_strong_efficiency_pct": round(res.runs[1].efficiency_pct, 1),
                               "in_process_schedule_over_one_engine": (round(ov, 4) if ov else None),
                               "halo_transfer_us_at_770GBps_overlapped": round(halo_us, 1)}
            print(edge, N, ent["ranks"][N], flush=True)
        out[f"{edge}^3"] = ent
    print(json.dumps(out))


if __name__ == "__main__":
    main()
