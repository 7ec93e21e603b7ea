"""Per-phase device times of one engine step (CUDA events on the engine stream).

    python tools/phase_times.py [--grid 240] [--steps 50] [--mode fast] [--radius 4]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=240)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--radius", type=int, default=4)
    ap.add_argument("--nd", type=int, default=27)
    ap.add_argument("--debug", action="store_true", help="sync after each phase, report faults")
    a = ap.parse_args()
    import torch
    import paper_2007_06048_b200 as mm
    n = (a.grid,) * 3
    nd = (a.nd,) * 3
    grid = mm.make_grid(n, (20.0, 20.0, 20.0), a.radius)
    model = mm.default_layered_model(grid)
    dt = mm.cfl_dt(model, grid, 0.8)
    w = mm.ricker(25.0, dt, 2 * a.steps + 10).samples
    e = mm.AcousticCdEngine(grid, (0, 0, 0), n, model.vp, mm.EngineOptions(ndamping=nd, taper=True),
                            dt, model.vmax, mode=a.mode)
    src = tuple(x // 2 for x in n)
    if a.debug:
        for nm, fn in (("pass1", e.update_boundary_psi), ("inner", e.update_inner),
                       ("boundary", e.update_boundary)):
            fn()
            try:
                e.synchronize()
                print("ok", nm, flush=True)
            except Exception as ex:  # noqa: BLE001
                print("FAULT in", nm, ex, flush=True)
                return
        return
    for s in range(10):
        e.step(float(w[s]), src)
    e.synchronize()
    ext = torch.cuda.ExternalStream(e.stream_handle())
    names = ["pass1", "inner", "boundary", "inject+rotate"]
    evs = []
    for s in range(a.steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(ext)
        e.update_boundary_psi()
        ev[1].record(ext)
        e.update_inner()
        ev[2].record(ext)
        e.update_boundary()
        ev[3].record(ext)
        e.inject_source(float(w[s + 10]), src)
        e.rotate()
        ev[4].record(ext)
        evs.append(ev)
    torch.cuda.synchronize()
    out = {}
    for k, nm in enumerate(names):
        out[nm] = statistics.mean(ev[k].elapsed_time(ev[k + 1]) for ev in evs)
    # fused step
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(ext)
    for s in range(a.steps):
        e.step(float(w[s + 10]), src)
    t1.record(ext)
    torch.cuda.synchronize()
    out["step"] = t0.elapsed_time(t1) / a.steps
    pts = float(a.grid) ** 3
    out["gpts_step"] = pts / (out["step"] * 1e-3) / 1e9
    inner_pts = float(a.grid - 2 * a.nd) ** 3
    out["inner_gpts"] = inner_pts / (out["inner"] * 1e-3) / 1e9
    out["inner_GBps_16B"] = inner_pts * 16 / (out["inner"] * 1e-3) / 1e9
    out["boundary_gpts"] = (pts - inner_pts) / (out["boundary"] * 1e-3) / 1e9
    print(json.dumps({k: round(v, 4) for k, v in out.items()}))


if __name__ == "__main__":
    main()
