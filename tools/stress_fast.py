"""Stress the fast acoustic_iso_cd step under concurrency (diagnostics).

    MODES=fast[,strict|,fast] BUSY=0|1 FS=0|1 [N=nx,ny,nz ND=a,b,c R=4] \
        python tools/stress_fast.py ITERATIONS

Runs the odd-extent free-surface configuration of test_gpu_parity for
ITERATIONS fresh engines, optionally interleaved with other engines (MODES)
or with unrelated GPU work on another stream (BUSY=1), and reports engines
whose final field differs from the first one.  Combine with MM_BND_CTAS=<n>
(few boundary CTAs) and MM_DEBUG_SYNC=kernels (name the faulting kernel).
"""
import os, sys, numpy as np
sys.path.insert(0,'.')
import paper_2007_06048_b200 as mm
def _t(k, d):
    v = os.environ.get(k)
    return tuple(int(x) for x in v.split(",")) if v else d
n = _t("N", (61, 47, 53))
nd = _t("ND", (9, 7, 11))
radius = int(os.environ.get("R", "4"))
src = tuple(x // 2 for x in n)
fs = os.environ.get("FS", "1") == "1"
modes = os.environ.get("MODES", "fast,strict").split(",")
steps, dt = 60, 1.0e-3
grid = mm.make_grid(n, (20.0, 15.0, 10.0), radius)
m = mm.random_model(grid, seed=11)
w = mm.ricker(25.0, dt, steps).samples
opts = mm.EngineOptions(ndamping=nd, taper=True, free_surface=fs)
bad = 0
busy = os.environ.get("BUSY") == "1"
if busy:
    import torch
    bs = torch.cuda.Stream()
    X = torch.randn(2048, 2048, device="cuda")
for it in range(int(sys.argv[1])):
    eng = {f"{md}{i}": mm.AcousticCdEngine(grid, (0, 0, 0), n, m.vp, opts, dt, m.vmax, mode=md)
           for i, md in enumerate(modes)}
    for s in range(steps):
        for e in eng.values():
            e.step(float(w[s]), src)
        if busy:
            with torch.cuda.stream(bs):
                for _ in range(2):
                    Y = X @ X
    ps = [e.pressure() for e in eng.values()]
    if it == 0:
        ref = ps[0]
    if not all(np.array_equal(x, ref) for x in ps): bad += 1
    for e in eng.values(): e.close()
print(os.environ.get("TAG",""), "iterations", sys.argv[1], "mismatches", bad, flush=True)
