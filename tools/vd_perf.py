"""Device time of the acoustic_iso (VD) step: Gpts/s and achieved GB/s.

    python tools/vd_perf.py [edge ...]

Bytes per step (compulsory, this design): 56 B/pt (velocity: p, dt/rho,
v r+w; pressure: v, dtb, p r+w) + 16 B/pt of CPML psi traffic (r+w, one
array per pass) on each damping-layer point and axis.
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2007_06048_b200 as mm  # noqa: E402


def bytes_per_step(n, nd):
    N = n[0] * n[1] * n[2]
    lay = sum(2 * nd[a] * N // n[a] for a in range(3))
    return 56 * N + 16 * lay


def main(edges):
    for edge in edges:
        n = (edge, edge, edge)
        g = mm.make_grid(n, (20.0, 20.0, 20.0))
        m = mm.default_layered_model(g)
        nd = (27, 27, 27)
        e = mm.AcousticVdEngine(g, m, mm.EngineOptions(ndamping=nd), 1e-3)
        steps = 200 if edge <= 256 else 40
        amps = np.zeros(steps, np.float32)
        e.run(amps[:10], (edge // 2,) * 3, record=False)
        ms = e.run(amps, (edge // 2,) * 3, record=False)
        t = ms / steps
        N = edge ** 3
        B = bytes_per_step(n, nd)
        # per-kernel device times (sub-phases back to back, CUDA events)
        import torch
        ext = torch.cuda.ExternalStream(e.stream_handle())
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        kv = kp = 0.0
        reps = 20
        for _ in range(reps):
            ev[0].record(ext)
            e.update_velocity()
            ev[1].record(ext)
            e.update_pressure()
            ev[2].record(ext)
            torch.cuda.synchronize()
            kv += ev[0].elapsed_time(ev[1]) / reps
            kp += ev[1].elapsed_time(ev[2]) / reps
        print(f"{edge}^3: {t*1e3:.1f} us/step  {N/t/1e6:.1f} Gpts/s  "
              f"{B/t/1e6:.0f} GB/s (model {B/N:.1f} B/pt)  velocity {kv*1e3:.1f} us  "
              f"pressure {kp*1e3:.1f} us")
        e.close()


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [240, 512])
