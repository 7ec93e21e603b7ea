"""Tiny / degenerate grids: fast, strict and the oracle side by side
(debugging aid; on a CPU-only host only the oracle port vs reference leg runs)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2007_06048_b200 as mm
from oracle.oracle import Oracle, available

CASES = [((5, 7, 9), (1, 2, 3), 4, True), ((5, 7, 9), (1, 2, 3), 4, False),
         ((9, 9, 9), (4, 4, 4), 4, True), ((9, 9, 9), (4, 4, 4), 4, False),
         ((1, 40, 33), (0, 6, 5), 2, True), ((37, 1, 12), (8, 0, 2), 4, True),
         ((20, 18, 2), (4, 3, 0), 8, True), ((40, 12, 40), (6, 5, 6), 4, False)]


def main():
    gpu = "--gpu" in sys.argv
    orc = {k: Oracle(k) for k in ("port", "reference") if available(k)}
    for n, nd, r, fs in CASES:
        grid = mm.make_grid(n, (20.0, 15.0, 10.0), r)
        m = mm.random_model(grid, seed=2)
        w = mm.ricker(25.0, 1e-3, 15).samples
        src = tuple(x // 2 for x in n)
        engs = {k: o.engine(n, m.vp, d=(20.0, 15.0, 10.0), radius=r, ndamping=nd,
                            free_surface=fs, taper=True, dt=1e-3, vmax=m.vmax)
                for k, o in orc.items()}
        if gpu:
            opts = mm.EngineOptions(ndamping=nd, taper=True, free_surface=fs)
            for md in ("fast", "strict"):
                engs[md] = mm.AcousticCdEngine(grid, (0, 0, 0), n, m.vp, opts, 1e-3, m.vmax,
                                               mode=md)
        for s in range(15):
            for e in engs.values():
                e.step(float(w[s]) * 1e3, src)
        ps = {k: np.asarray(e.pressure()).reshape(grid_shape(n, r)) for k, e in engs.items()}
        base = "reference" if "reference" in ps else "port"
        line = []
        for k, p in ps.items():
            d = np.argwhere(p != ps[base])
            line.append(f"{k}: {len(d)} diff" + (f" first {tuple(d[0])}" if len(d) else ""))
        print(n, nd, r, fs, "|", "; ".join(line))


def grid_shape(n, r):
    return tuple(x + 2 * r for x in n)


if __name__ == "__main__":
    main()
