"""Where the host-driven (e2e) loop loses time against the device loop:
per-step wall and CUDA-event time of step / step+record / step+record+copy."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2007_06048_b200 as mm  # noqa: E402


def main():
    edge = int(sys.argv[1]) if len(sys.argv) > 1 else 240
    n = (edge,) * 3
    nd = (27, 27, 27)
    grid = mm.make_grid(n, (20.0, 20.0, 20.0), 4)
    model = mm.default_layered_model(grid)
    dt = mm.cfl_dt(model, grid, 0.8)
    steps = 600
    w = mm.ricker(25.0, dt, steps + 20).samples
    src = tuple(x // 2 for x in n)
    eng = mm.AcousticCdEngine(grid, (0, 0, 0), n, model.vp,
                              mm.EngineOptions(ndamping=nd, taper=True), dt, model.vmax)
    geo = mm.default_receivers(grid, nd)
    eng.set_receivers(geo.receivers, steps + 20)
    out = torch.empty((steps, geo.nreceivers()), dtype=torch.float32, pin_memory=True).numpy()
    ext = torch.cuda.ExternalStream(eng.stream_handle())
    for s in range(20):
        eng.step(float(w[s]), src)
    eng.synchronize()
    for variant in ("run", "step", "step+record", "step+record+copy", "step", "run"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(ext)
        if variant == "run":
            eng.run(w[:steps], src, record=True, first_sample=0)
        else:
            for s in range(steps):
                eng.step(float(w[s]), src)
                if "record" in variant:
                    eng.record(s)
                if "copy" in variant:
                    eng.copy_trace_step(s, out[s], asynchronous=True)
        t_host = time.perf_counter() - t0
        e1.record(ext)
        eng.synchronize()
        wall = time.perf_counter() - t0
        dev = e0.elapsed_time(e1)
        print(f"{variant:18s} host-issue {t_host / steps * 1e6:7.1f} us/step  wall "
              f"{wall / steps * 1e6:7.1f}  device {dev / steps * 1e3:7.1f}")


if __name__ == "__main__":
    main()
