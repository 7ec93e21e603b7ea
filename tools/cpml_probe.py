"""Per-kernel times of the acoustic_iso_cd step under tuning variants.

    python tools/cpml_probe.py --grid 240 --steps 100 [--tune name=value ...]
           [--variants "overlap=0;cpml_zt=24,overlap=0"]

For each variant (";"-separated lists of name=value, "," inside one variant):
device ms/step of the mm_cd_run loop, Gpts/s, and the mean duration of every
kernel inside the step (CUDA events on the launching stream)."""
import argparse
import os
import sys
from pathlib import Path

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2007_06048_b200 as mm  # noqa: E402
from paper_2007_06048_b200 import _lib  # noqa: E402


def parse_kv(s):
    out = {}
    for kv in filter(None, (x.strip() for x in s.split(","))):
        k, v = kv.split("=")
        out[k] = int(v)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=240)
    ap.add_argument("--nz", type=int, default=0)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--radius", type=int, default=4)
    ap.add_argument("--nd", type=int, default=27)
    ap.add_argument("--variants", default="")
    ap.add_argument("--mode", default="fast")
    a = ap.parse_args()
    n = (a.grid, a.grid, a.nz or a.grid)
    grid = mm.make_grid(n, (20.0, 20.0, 20.0), a.radius)
    model = mm.default_layered_model(grid)
    dt = mm.cfl_dt(model, grid, 0.8)
    w = mm.ricker(25.0, dt, a.steps).samples
    src = tuple(x // 2 for x in n)
    opts = mm.EngineOptions(ndamping=(a.nd,) * 3, taper=True)
    for var in (a.variants.split(";") if a.variants else [""]):
        kv = parse_kv(var)
        _lib.reset_tuning()
        for k, v in kv.items():
            _lib.set_tuning(k, v)
        e = mm.AcousticCdEngine(grid, (0, 0, 0), n, model.vp, opts, dt, model.vmax,
                                mode=a.mode)
        e.run(w[:10], src, record=False)
        ms = e.run(w, src, record=False)
        e.kernel_timing(True)
        e.run(w, src, record=False)
        kt = e.kernel_times()
        e.kernel_timing(False)
        pts = n[0] * n[1] * n[2]
        per = ", ".join(f"{k} {v[0] / v[1] * 1e3:.1f} us" for k, v in sorted(kt.items()))
        print(f"[{var or 'default'}] path={e.cpml_path()} {ms / a.steps * 1e3:.1f} us/step "
              f"{pts * a.steps / (ms * 1e-3) / 1e9:.1f} Gpts/s | {per}", flush=True)
        e.close()
    _lib.reset_tuning()


if __name__ == "__main__":
    main()
