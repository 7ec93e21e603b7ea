"""acoustic_iso (variable density) on the GPU, SURVEY.md §8(f) row 4.

The CUDA engine (csrc/vd_engine.cu, through the C ABI) against the pinned
oracle and the reference-generated fixtures: bit-identical pressure and
velocities.  Also the reference's own VD property tests
(test_propagator.cpp:47-71, :118-133) and the driver path (run() with
Propagator::AcousticIso, driver.cpp:122-128).
"""
import numpy as np

from paper_2007_06048_b200._lib import tuned
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _model(mm, n, r, seed, d=(20.0, 20.0, 20.0)):
    g = mm.make_grid(n, d, r)
    rng = np.random.default_rng(seed)
    vp, rho = g.field(), g.field()
    g.inner(vp)[...] = rng.uniform(1500.0, 4500.0, n).astype(np.float32)
    g.inner(rho)[...] = rng.uniform(1000.0, 2500.0, n).astype(np.float32)
    return g, mm.validate_model(mm.EarthModel(g, vp, rho=rho))


@pytest.mark.parametrize("name", ["vd_cpml", "vd_r2_fs", "vd_r8"])
def test_vd_engine_matches_reference_fixture(mm, name):
    gd = load_golden(name)
    n, r = tuple(int(x) for x in gd["n"]), int(gd["radius"])
    g = mm.make_grid(n, (20.0, 20.0, 20.0), r)
    m = mm.validate_model(mm.EarthModel(g, gd["vp"].copy(), rho=gd["rho"].copy()))
    opts = mm.EngineOptions(ndamping=tuple(int(x) for x in gd["ndamping"]),
                            free_surface=bool(gd["free_surface"]), taper=bool(gd["taper"]))
    src = tuple(int(x) for x in gd["src"])
    nd2 = int(gd["ndamping"][2])
    with mm.AcousticVdEngine(g, m, opts, float(gd["dt"])) as e:
        for s in range(int(gd["steps"])):
            e.step(float(gd["wavelet"][s]), src)
            if s % 7 == 0 or s == int(gd["steps"]) - 1:
                assert np.array_equal(e.pressure()[r:-r, r:-r, r + nd2], gd["surface"][s]), s
        assert np.array_equal(e.pressure(), gd["p"])
        for ax, key in enumerate(("vx", "vy", "vz")):
            assert np.array_equal(e.velocity(ax), gd[key]), key


@pytest.mark.parametrize("n,r,nd,fs,taper,d", [
    ((33, 29, 41), 4, (6, 5, 7), False, True, (20.0, 12.5, 7.25)),
    ((40, 36, 30), 3, (0, 8, 4), True, False, (10.0, 10.0, 10.0)),
    ((27, 45, 38), 1, (4, 0, 9), True, True, (15.0, 20.0, 5.0)),
    ((50, 20, 24), 6, (7, 3, 0), False, False, (20.0, 20.0, 20.0)),
])
def test_vd_engine_matches_oracle(mm, oracle_port, n, r, nd, fs, taper, d):
    g, m = _model(mm, n, r, seed=sum(n), d=d)
    dt = 7e-4
    src = (n[0] // 3, n[1] // 2, n[2] // 2)
    o = oracle_port.vd_engine(n, m.vp, m.rho, d=d, radius=r, ndamping=nd, free_surface=fs,
                              taper=taper, dt=dt, vmax=m.vmax)
    w = mm.integrate_wavelet(mm.ricker(25.0, dt, 30)).samples
    with mm.AcousticVdEngine(g, m, mm.EngineOptions(ndamping=nd, free_surface=fs, taper=taper),
                             dt) as e:
        for s in range(30):
            e.step(float(w[s]), src)
            o.step(float(w[s]), src)
        assert np.array_equal(e.pressure(), o.pressure())
        for ax in range(3):
            assert np.array_equal(e.velocity(ax), o.velocity(ax)), ax
        assert np.abs(o.pressure()).max() > 0


def test_vd_subphases_and_device_loop(mm):
    """step == velocity -> pressure -> source -> free surface
    (propagator_impl.hpp:275-295); the graph-captured loop == per-step calls."""
    n, r = (30, 28, 32), 4
    g, m = _model(mm, n, r, seed=3)
    opts = mm.EngineOptions(ndamping=(5, 5, 5), free_surface=True)
    dt = 1e-3
    w = mm.integrate_wavelet(mm.ricker(25.0, dt, 24)).samples
    src = (15, 14, 10)
    rec = np.array([[i, j, 5] for i in range(n[0]) for j in range(0, n[1], 3)], np.int32)
    with mm.AcousticVdEngine(g, m, opts, dt) as a, mm.AcousticVdEngine(g, m, opts, dt) as b, \
            mm.AcousticVdEngine(g, m, opts, dt) as c:
        a.set_receivers(rec, 24)
        for s in range(24):
            a.step(float(w[s]), src)
            a.record(s)
            b.update_velocity()
            b.update_pressure()
            b.inject_source(float(w[s]), src)
            b.apply_free_surface()
        c.set_receivers(rec, 24)
        c.run(w, src)
        for x, y in ((a, b), (a, c)):
            assert np.array_equal(x.pressure(), y.pressure())
            for ax in range(3):
                assert np.array_equal(x.velocity(ax), y.velocity(ax))
        assert np.array_equal(a.traces(), c.traces())
        assert c.steps_taken() == 24


def test_vd_zero_state_and_constant_pressure(mm):
    """test_propagator.cpp:47-71 (zero stays zero) and :118-133 (a spatially
    constant pressure, ghosts included, is left untouched)."""
    g = mm.make_grid((14, 14, 14), (10.0, 10.0, 10.0))
    m = mm.constant_model(g, 1500.0, rho=1000.0)
    with mm.AcousticVdEngine(g, m, mm.EngineOptions(ndamping=(3, 3, 3)), 1e-3) as e:
        for _ in range(3):
            e.step(0.0, None)
        assert not e.pressure().any()
        assert not any(e.velocity(ax).any() for ax in range(3))
    with mm.AcousticVdEngine(g, m, mm.EngineOptions(ndamping=(4, 4, 4)), 1e-3) as e:
        e.set_pressure(np.full(g.shape, 0.75, np.float32))
        for _ in range(5):
            e.step(0.0, None)
        for ax in range(3):
            assert not e.velocity(ax).any()
        assert (g.inner(e.pressure()) == 0.75).all()


def test_vd_source_injection_scale(mm):
    """p[src] += dt * (rho vp vp) * amp after one step from rest."""
    g = mm.make_grid((16, 16, 16), (10.0, 10.0, 10.0))
    m = mm.constant_model(g, 1500.0, rho=1000.0)
    with mm.AcousticVdEngine(g, m, mm.EngineOptions(), 1e-3) as e:
        e.step(1.0, (8, 8, 8))
        p = e.pressure()
        expect = np.float32(np.float32(1e-3) * np.float32(np.float32(1000.0 * 1500.0) * 1500.0))
        assert p[12, 12, 12] == expect
        assert np.count_nonzero(p) == 1


def test_vd_run_matches_reference_fixture(mm):
    gd = load_golden("run_vd_layered_32")
    n = tuple(int(x) for x in gd["n"])
    cfg = mm.SimConfig(propagator="acoustic_iso", ngrid=n, nsteps=int(gd["nsteps"]),
                       ndamping=tuple(int(x) for x in gd["ndamping"]),
                       ntaper=tuple(int(x) for x in gd["ntaper"]))
    rec, rep = mm.run(cfg, mm.default_layered_model(mm.make_grid(n, cfg.dgrid)))
    assert rep.dt == float(gd["dt"])
    assert np.array_equal(rec.traces, gd["traces"])


def test_vd_run_matches_reference_live(mm, oracle_ref):
    n = (40, 36, 44)
    cfg = mm.SimConfig(propagator="acoustic_iso", ngrid=n, nsteps=50, ndamping=(8, 7, 9),
                       free_surface=True, receiver_increment=(2, 3))
    model = mm.default_layered_model(mm.make_grid(n, cfg.dgrid))
    rec, rep = mm.run(cfg, model)
    ref = oracle_ref.run_vd(n, model.vp, model.rho, nsteps=50, ndamping=(8, 7, 9),
                            free_surface=True)
    pick = np.array([i * n[1] + j for i in range(0, n[0], 2) for j in range(0, n[1], 3)])
    assert rep.dt == ref["dt"]
    assert np.array_equal(rec.traces, ref["traces"][pick])


def test_vd_large_grid_against_oracle(mm, oracle_port):
    """A BASELINE-class shape (nd 27 slabs) for a few steps: bit-identical."""
    n, r = (128, 120, 136), 4
    g, m = _model(mm, n, r, seed=77)
    nd = (27, 27, 27)
    dt = 1e-3
    w = mm.integrate_wavelet(mm.ricker(25.0, dt, 6)).samples
    o = oracle_port.vd_engine(n, m.vp, m.rho, radius=r, ndamping=nd, dt=dt, vmax=m.vmax)
    with mm.AcousticVdEngine(g, m, mm.EngineOptions(ndamping=nd), dt) as e:
        for s in range(6):
            e.step(float(w[s]) * 1e6, (30, 60, 100))
            o.step(float(w[s]) * 1e6, (30, 60, 100))
        assert np.array_equal(e.pressure(), o.pressure())
        assert np.array_equal(e.velocity(2), o.velocity(2))


def test_vd_cli_model_run(mm, tmp_path, oracle_ref):
    """`minimod model --propagator acoustic_iso` (tools/cli.cpp:256-272)."""
    import io
    from paper_2007_06048_b200.__main__ import main
    out, err = io.StringIO(), io.StringIO()
    n = (60, 56, 64)  # default ndamping 27 needs n > 54
    rc = main(["model", "--propagator", "acoustic_iso", "--ngrid", ",".join(map(str, n)),
               "--nsteps", "30", "--output", str(tmp_path / "shot.bin")], out, err)
    assert rc == 0, err.getvalue()
    assert "Time Kernel" in out.getvalue()
    rec = mm.load_record(tmp_path / "shot.bin")
    model = mm.default_layered_model(mm.make_grid(n, (20.0, 20.0, 20.0)))
    ref = oracle_ref.run_vd(n, model.vp, model.rho, nsteps=30)
    assert np.array_equal(rec.traces, ref["traces"])


def test_vd_kernel_families_agree(mm, monkeypatch):
    """The TMA kernels (default) and the plain one-thread-per-point restatement
    (tuning vd_simple=1, read at engine creation) are bit-identical."""
    n, r = (70, 66, 75), 4
    g, m = _model(mm, n, r, seed=11)
    opts = mm.EngineOptions(ndamping=(9, 10, 11), free_surface=True, taper=True)
    dt = 1e-3
    w = mm.integrate_wavelet(mm.ricker(25.0, dt, 40)).samples
    fast = mm.AcousticVdEngine(g, m, opts, dt)
    with tuned(vd_simple=1):
        plain = mm.AcousticVdEngine(g, m, opts, dt)
    for s in range(40):
        fast.step(float(w[s]) * 1e6, (20, 30, 40))
        plain.step(float(w[s]) * 1e6, (20, 30, 40))
    assert np.array_equal(fast.pressure(), plain.pressure())
    for ax in range(3):
        assert np.array_equal(fast.velocity(ax), plain.velocity(ax))
    fast.close()
    plain.close()


@pytest.mark.parametrize("ctas", [1, 7])
def test_vd_few_ctas(mm, ctas):
    """Long item sequences per CTA through the TMA rings (tuning vd_ctas, read
    at engine creation) on an odd free-surface grid: still bit-identical to
    the plain kernels."""
    n = (61, 47, 53)
    g = mm.make_grid(n, (20.0, 15.0, 10.0), 4)
    rng = np.random.default_rng(5)
    vp, rho = g.field(), g.field()
    g.inner(vp)[...] = rng.uniform(1500, 4500, n).astype(np.float32)
    g.inner(rho)[...] = rng.uniform(1000, 2500, n).astype(np.float32)
    m = mm.validate_model(mm.EarthModel(g, vp, rho=rho))
    o = mm.EngineOptions(ndamping=(9, 7, 11), taper=True, free_surface=True)
    w = mm.integrate_wavelet(mm.ricker(25.0, 1e-3, 40)).samples
    with tuned(vd_ctas=ctas):
        fast = mm.AcousticVdEngine(g, m, o, 1e-3)
    with tuned(vd_simple=1):
        plain = mm.AcousticVdEngine(g, m, o, 1e-3)
    for s in range(40):
        fast.step(float(w[s]) * 1e6, (30, 23, 26))
        plain.step(float(w[s]) * 1e6, (30, 23, 26))
    assert np.array_equal(fast.pressure(), plain.pressure())
    assert all(np.array_equal(fast.velocity(a), plain.velocity(a)) for a in range(3))


@pytest.mark.slow
def test_vd_large_grid_families_agree(mm, monkeypatch):
    """1000 x 1000 x 120 (byte offsets past 2^32 per field, 32 x 32 tiles with
    a partial last column): TMA kernels == plain kernels after a few steps
    from a random pressure field with every damping run active."""
    n = (1000, 1000, 120)
    g = mm.make_grid(n, (20.0, 20.0, 20.0), 4)
    model = mm.default_layered_model(g)
    opts = mm.EngineOptions(ndamping=(27, 27, 27), free_surface=True)
    rng = np.random.default_rng(8)
    p0 = g.field()
    g.inner(p0)[...] = rng.standard_normal(n).astype(np.float32)
    fast = mm.AcousticVdEngine(g, model, opts, 1e-3)
    with tuned(vd_simple=1):
        plain = mm.AcousticVdEngine(g, model, opts, 1e-3)
    for e in (fast, plain):
        e.set_pressure(p0)
        for s in range(3):
            e.step(1.0, (500, 500, 60))
    assert np.array_equal(fast.pressure(), plain.pressure())
    assert np.array_equal(fast.velocity(0), plain.velocity(0))
    fast.close()
    plain.close()


@pytest.mark.parametrize("n,r,nd,fs", [
    ((5, 7, 9), 4, (1, 2, 3), True),     # smaller than one tile, thinner than the halo
    ((5, 7, 9), 4, (1, 2, 3), False),    # both z layers active and within R
    ((1, 40, 33), 2, (0, 6, 5), True),   # a single x column
    ((37, 1, 12), 3, (8, 0, 2), True),   # a single y row
    ((20, 18, 2), 8, (4, 3, 0), True),   # two z planes, r = 8
    ((9, 9, 9), 4, (4, 4, 4), False),    # inner box of one point
    ((40, 12, 40), 4, (6, 5, 6), False),  # y layers 2 apart
])
def test_vd_tiny_and_degenerate_grids(mm, oracle_port, n, r, nd, fs):
    g, m = _model(mm, n, r, seed=sum(n) + r)
    dt = 5e-4
    src = tuple(x // 2 for x in n)
    w = mm.integrate_wavelet(mm.ricker(25.0, dt, 12)).samples
    o = oracle_port.vd_engine(n, m.vp, m.rho, radius=r, ndamping=nd, free_surface=fs,
                              dt=dt, vmax=m.vmax)
    with mm.AcousticVdEngine(g, m, mm.EngineOptions(ndamping=nd, free_surface=fs), dt) as e:
        for s in range(12):
            e.step(float(w[s]) * 1e6, src)
            o.step(float(w[s]) * 1e6, src)
        assert np.array_equal(e.pressure(), o.pressure())
        for ax in range(3):
            assert np.array_equal(e.velocity(ax), o.velocity(ax)), ax


@pytest.mark.parametrize("src_z", [0, 2, 9])
def test_vd_step_epilogue_edge_placements(mm, oracle_port, src_z):
    """acoustic_iso's k_epilogue (injection, free surface, receiver sample in
    one launch): receivers on the source point, on and near the surface, a
    source on the surface and within R of it; run() and step()+record() both
    equal the oracle's inject -> free surface -> record order."""
    n, nd, steps, dt = (26, 22, 24), (5, 4, 6), 12, 5e-4
    g, m = _model(mm, n, 4, seed=7)
    w = mm.integrate_wavelet(mm.ricker(25.0, dt, steps)).samples * 1e6
    src = (13, 11, src_z)
    rec = np.array([src, (13, 11, 0), (12, 11, 0), (13, 11, 1), (13, 11, 3), (0, 0, 0),
                    (25, 21, 23), (14, 11, src_z)])
    o = oracle_port.vd_engine(n, m.vp, m.rho, radius=4, ndamping=nd, free_surface=True, dt=dt,
                              vmax=m.vmax)
    want = np.zeros((len(rec), steps), np.float32)
    for s in range(steps):
        o.step(float(w[s]), src)
        p = np.asarray(o.pressure()).reshape(g.shape)
        want[:, s] = [p[i + 4, j + 4, k + 4] for i, j, k in rec]
    assert (np.abs(want).max() > 0) == (src_z != 0)  # a source on the surface is zeroed
    opts = mm.EngineOptions(ndamping=nd, free_surface=True)
    for use_loop in (False, True):
        with mm.AcousticVdEngine(g, m, opts, dt) as e:
            e.set_receivers(rec, steps)
            if use_loop:
                e.run(w, src)
            else:
                for s in range(steps):
                    e.step(float(w[s]), src)
                    e.record(s)
            assert np.array_equal(e.pressure(), o.pressure()), use_loop
            assert np.array_equal(e.traces(), want), use_loop
