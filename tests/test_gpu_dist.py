"""GPU z-slab path: the overlap schedule (edges -> halo transfer || interior ->
finish) through the C-ABI plane pointers, several ranks in one process on one
device (device-to-device halo copies stand in for NCCL), bit-identical to the
single engine -- the reference's own guarantee (test_dist.cpp:107-118)."""
import numpy as np
import pytest

from paper_2007_06048_b200 import dist as D

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,fs,src_z,parts", [
    ("fast", False, 32, 3),
    ("fast", True, 25, 2),      # source inside an edge plane of a cut
    ("strict", False, 40, 2),
])
def test_zslab_overlap_schedule_bitwise(mm, mode, fs, src_z, parts):
    n, nd, steps, dt = (40, 36, 64), (5, 6, 7), 40, 1.2e-3
    grid = mm.make_grid(n, (20.0, 20.0, 20.0))
    model = mm.random_model(grid, seed=5)
    opts = mm.EngineOptions(ndamping=nd, taper=True, free_surface=fs)
    w = mm.ricker(25.0, dt, steps).samples
    src = (20, 18, src_z)
    whole = mm.AcousticCdEngine(grid, (0, 0, 0), n, model.vp, opts, dt, model.vmax, mode=mode)
    for s in range(steps):
        whole.step(float(w[s]), src)
    full = whole.pressure()
    cuts = D.weighted_cuts(n, nd, 4, parts)
    if src_z == 25:
        cuts = [0, 27, 64]  # put the source 2 planes below the cut (an edge plane)
        D.validate_cuts(cuts, 64, 7, 4)
    ranks = []
    for r in range(parts):
        info = D.SlabInfo(r, parts, cuts)
        lg = mm.make_grid((n[0], n[1], info.nz), grid.d)
        e = mm.AcousticCdEngine(lg, (0, 0, info.z0), n, D.local_vp(model.vp, 4, info.z0, info.nz),
                                opts, dt, model.vmax, mode=mode)
        ranks.append(D.ZSlabRank(e, info, None, src))
    for s in range(steps):
        D.step_local(ranks, float(w[s]))
    for rk in ranks:
        z0, nz = rk.info.z0, rk.info.nz
        got = rk.e.pressure()[:, :, 4:-4]
        assert np.array_equal(got, full[:, :, 4 + z0:4 + z0 + nz]), (rk.info.rank, cuts)
