"""Step a fast and a strict engine side by side and report the first step and
the points where they differ (debugging aid for the fast kernels)."""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2007_06048_b200 as mm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs=3, default=[24, 28, 32])
    ap.add_argument("--nd", type=int, nargs=3, default=[5, 6, 7])
    ap.add_argument("--radius", type=int, default=4)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--fs", action="store_true")
    a = ap.parse_args()
    n, nd = tuple(a.n), tuple(a.nd)
    grid = mm.make_grid(n, (20.0, 20.0, 20.0), radius=a.radius)
    model = mm.random_model(grid, seed=3)
    opts = mm.EngineOptions(ndamping=nd, taper=True, free_surface=a.fs)
    dt = 1.2e-3
    w = mm.ricker(25.0, dt, a.steps).samples
    src = tuple(x // 2 for x in n)
    eng = {m: mm.AcousticCdEngine(grid, (0, 0, 0), n, model.vp, opts, dt, model.vmax, mode=m)
           for m in ("fast", "strict")}
    for s in range(a.steps):
        for e in eng.values():
            e.step(float(w[s]), src)
        pf, ps = eng["fast"].pressure(), eng["strict"].pressure()
        bad = np.argwhere(pf != ps)
        if len(bad):
            print(f"step {s}: {len(bad)} mismatches")
            for i, j, k in bad[:20]:
                kind = ("X" if i < nd[0] or i >= n[0] - nd[0] else
                        "Y" if j < nd[1] or j >= n[1] - nd[1] else
                        "Z" if k < nd[2] or k >= n[2] - nd[2] else "inner")
                print(f"  ({i},{j},{k}) {kind} fast={pf[i, j, k]!r} strict={ps[i, j, k]!r}")
            xs, ys, zs = bad[:, 0], bad[:, 1], bad[:, 2]
            print("  x", np.unique(xs), "\n  y", np.unique(ys), "\n  z", np.unique(zs))
            return
    print("no mismatch")


if __name__ == "__main__":
    main()
