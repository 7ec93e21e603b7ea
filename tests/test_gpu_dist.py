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


# ------------------------------------------------------------ C++ group (mm_cd_group_*)
def _layered(mm, n, r=4):
    grid = mm.make_grid(n, (20.0, 20.0, 20.0), r)
    return grid, mm.default_layered_model(grid)


@pytest.mark.parametrize("fs,with_comm", [(False, False), (True, True)])
def test_group_world1_equals_single_engine(mm, fs, with_comm):
    """The C++ group with one rank (no halo partner) runs the group schedule
    (pass 1, edge-free interior with the interior kernel on its side stream,
    epilogue with the slab-centre check) and equals one engine bitwise --
    device loop and host-driven steps, receivers included."""
    from paper_2007_06048_b200.propagator import ZSlabGroup
    n, nd, steps = (48, 44, 56), (6, 7, 8), 40
    grid, model = _layered(mm, n)
    dt = float(np.float32(mm.cfl_dt(model, grid, 0.8)))
    opts = mm.EngineOptions(ndamping=nd, taper=True, free_surface=fs)
    w = mm.ricker(25.0, dt, steps).samples
    src = (20, 22, 30)
    geo = mm.default_receivers(grid, nd)
    one = mm.AcousticCdEngine(grid, (0, 0, 0), n, model.vp, opts, dt, model.vmax)
    one.set_receivers(geo.receivers, steps)
    one.run(w, src, record=True)
    nid = None
    if with_comm:  # a one-rank NCCL communicator (ncclCommInitRank / CommDestroy)
        from paper_2007_06048_b200.propagator import nccl_unique_id
        nid = nccl_unique_id()
    g = ZSlabGroup(grid, [0, n[2]], 0, model.vp, opts, dt, model.vmax, nccl_id=nid)
    g.engine.set_receivers(geo.receivers, steps)
    g.run(w[:25], src, record=True)
    for s in range(25, steps):                # host-driven steps continue the run
        g.step(float(w[s]), src)
        g.engine.record(s)
    assert np.array_equal(g.engine.pressure(), one.pressure())
    assert np.array_equal(g.engine.pressure_prev(), one.pressure_prev())
    assert np.array_equal(g.engine.traces(steps), one.traces(steps))
    g.close()


def test_group_reports_rank_instability(mm):
    """Per-rank finiteness check of the slab centre every step (dist.cpp:222-224)."""
    from paper_2007_06048_b200.propagator import ZSlabGroup
    n = (24, 24, 24)
    grid = mm.make_grid(n, (20.0, 20.0, 20.0))
    vp = grid.field(4000.0)
    g = ZSlabGroup(grid, [0, 24], 0, vp, mm.EngineOptions(), 5e-3, 4000.0)  # far past CFL
    with pytest.raises(mm.InstabilityError) as ei:
        g.run(np.ones(400, np.float32), (12, 12, 12), record=False)
    assert 1 <= ei.value.step <= 400 and "rank 0" in str(ei.value)
    g.close()


def _nccl_worker(rank, world, cuts, n, nd, steps, idq, q):
    import paper_2007_06048_b200 as mm
    from paper_2007_06048_b200 import dist as D
    from paper_2007_06048_b200.propagator import ZSlabGroup
    try:
        if rank == 0:
            from paper_2007_06048_b200.propagator import nccl_unique_id
            nid = nccl_unique_id()
            for _ in range(world - 1):
                idq.put(nid)
        else:
            nid = idq.get(timeout=120)
        grid = mm.make_grid(n, (20.0, 20.0, 20.0))
        vp = D.layered_slice(n, cuts[rank], cuts[rank + 1] - cuts[rank], 4)
        dt = D.cfl_dt_vmax(4500.0, grid, 0.8)
        w = mm.ricker(25.0, dt, steps).samples
        g = ZSlabGroup(grid, cuts, rank, None, mm.EngineOptions(ndamping=nd, taper=True),
                       float(np.float32(dt)), 4500.0, nccl_id=nid, device=rank, vp_local=vp)
        g.run(w, (n[0] // 2, n[1] // 2, n[2] // 2), record=False)
        q.put(("ok", rank, g.engine.pressure()[:, :, 4:-4].copy()))
        g.close()
    except Exception as e:  # noqa: BLE001
        q.put(("err", rank, repr(e)))


def test_group_nccl_world2_equals_single_engine(mm):
    """Two ranks on two GPUs through NCCL == one engine on the whole grid,
    bitwise (the reference's decomposition invariance, test_dist.cpp:107-118).
    Needs two devices: NCCL does not put two ranks on one GPU."""
    if mm.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    n, nd, steps = (64, 60, 96), (8, 8, 8), 30
    cuts = D.weighted_cuts(n, nd, 4, 2)
    ctx = mp.get_context("spawn")
    idq, qs = ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, cuts, n, nd, steps, idq, qs))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [qs.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[0] == "ok" for r in res), res
    grid, model = _layered(mm, n)
    dt = float(np.float32(D.cfl_dt_vmax(4500.0, grid, 0.8)))
    one = mm.AcousticCdEngine(grid, (0, 0, 0), n, model.vp,
                              mm.EngineOptions(ndamping=nd, taper=True), dt, 4500.0)
    one.run(mm.ricker(25.0, D.cfl_dt_vmax(4500.0, grid, 0.8), steps).samples,
            (n[0] // 2, n[1] // 2, n[2] // 2), record=False)
    full = one.pressure()[:, :, 4:-4]
    for _, rank, field in sorted(res, key=lambda t: t[1]):
        assert np.array_equal(field, full[:, :, cuts[rank]:cuts[rank + 1]]), rank


@pytest.mark.parametrize("mode,fs,src_z,cuts", [
    ("fast", False, 32, None),          # cost-weighted cuts, 3 ranks
    ("fast", True, 25, [0, 27, 64]),    # source 2 planes below a cut (an edge plane)
    ("strict", False, 40, [0, 22, 43, 64]),
])
def test_cpp_group_multirank_in_process_bitwise(mm, mode, fs, src_z, cuts):
    """The C++ group schedule with several ranks (edge planes on their own
    stream, halo transfer, interior, epilogue, rotation), ranks in one process
    on one GPU through mm_cd_group_step_local (device-to-device copies in place
    of NCCL): every slab equals one engine on the whole grid, bitwise."""
    from paper_2007_06048_b200.propagator import ZSlabGroup, step_local
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
    cuts = cuts or D.weighted_cuts(n, nd, 4, 3)
    D.validate_cuts(cuts, n[2], nd[2], 4)
    groups = [ZSlabGroup(grid, cuts, r, model.vp, opts, dt, model.vmax, mode=mode)
              for r in range(len(cuts) - 1)]
    for s in range(steps):
        step_local(groups, float(w[s]), src)
    for g in groups:
        got = g.engine.pressure()[:, :, 4:-4]
        assert np.array_equal(got, full[:, :, 4 + g.z0:4 + g.z0 + g.nz]), (g.rank, cuts)
    for g in groups:
        g.close()
