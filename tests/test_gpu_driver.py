"""GPU parity of the driver path run() (ref: driver.cpp:83-144) against the
reference's golden traces and checksums, plus the device-loop contract."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_run_layered_32_golden(mm, mode):
    g = load_golden("run_layered_32")
    n = tuple(int(x) for x in g["n"])
    cfg = mm.SimConfig(ngrid=n, nsteps=int(g["nsteps"]), ndamping=tuple(g["ndamping"]),
                       ntaper=tuple(g["ntaper"]))
    model = mm.default_layered_model(mm.make_grid(n, cfg.dgrid))
    rec, rep = mm.run(cfg, model, mode=mode)
    assert rep.dt == float(g["dt"]) and rep.steps_run == cfg.nsteps
    assert rep.kernel_seconds > 0 and rep.kernel_seconds <= rep.modeling_seconds
    if mode == "strict":
        assert np.array_equal(rec.traces, g["traces"])
    else:
        assert rel_l2(rec.traces, g["traces"]) <= 1e-5


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_run_oracle_config_100(mm, mode):
    """C1: 100^3 x 100 steps, layered, nd 27, taper on (BASELINE configs[0])."""
    g = load_golden("run_layered_100")
    cfg = mm.SimConfig(ngrid=(100, 100, 100), nsteps=100)
    model = mm.default_layered_model(mm.make_grid(cfg.ngrid, cfg.dgrid))
    rec, rep = mm.run(cfg, model, mode=mode)
    got = rec.traces[g["pick"]]
    if mode == "strict":
        assert np.array_equal(got, g["traces"])
        # (float64 norm: summation order differs across hosts, hence 1e-12)
        assert abs(np.linalg.norm(rec.traces.astype(np.float64)) / g["trace_norm"] - 1) < 1e-12
    else:
        assert rel_l2(got, g["traces"]) <= 1e-5
        assert abs(np.linalg.norm(rec.traces.astype(np.float64)) / g["trace_norm"] - 1) < 1e-5


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_final_field_checksums_100(mm, mode):
    """Final p_cur of C1 against the reference checksums."""
    g = load_golden("run_layered_100")
    grid = mm.make_grid((100, 100, 100), (20.0, 20.0, 20.0))
    model = mm.default_layered_model(grid)
    dt = mm.cfl_dt(model, grid, 0.8)
    w = mm.ricker(25.0, dt, 100).samples
    e = mm.AcousticCdEngine(grid, (0, 0, 0), grid.n, model.vp,
                            mm.EngineOptions(ndamping=(27, 27, 27), taper=True), dt, model.vmax,
                            mode=mode)
    e.set_receivers(np.array([[0, 0, 27]]), 100)
    e.run(w, (50, 50, 50))
    p = grid.inner(e.pressure()).astype(np.float64)
    assert abs(np.sqrt((p ** 2).sum()) / g["p_norm"] - 1) < 1e-6
    assert abs(np.abs(p).max() / g["p_max"] - 1) < 1e-6


def test_device_loop_equals_host_loop(mm):
    """mm_cd_run (device wavelet/counter/recording) == step()+record() calls."""
    g = load_golden("eng_cpml_aniso")
    n = tuple(int(x) for x in g["n"])
    grid = mm.make_grid(n, (20.0, 20.0, 20.0))
    opts = mm.EngineOptions(ndamping=tuple(int(x) for x in g["ndamping"]), taper=True)
    rec = np.array([[i, j, 7] for i in range(n[0]) for j in range(0, n[1], 3)])
    out = []
    for use_loop in (False, True):
        e = mm.AcousticCdEngine(grid, (0, 0, 0), n, g["vp"], opts, float(g["dt"]),
                                float(g["vmax"]), mode="strict")
        e.set_receivers(rec, int(g["steps"]))
        src = tuple(int(x) for x in g["src"])
        if use_loop:
            e.run(g["wavelet"], src)
        else:
            for s in range(int(g["steps"])):
                e.step(float(g["wavelet"][s]), src)
                e.record(s)
        out.append((e.pressure(), e.traces()))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[1][0], g["p_cur"])


def test_cli_model_shot_record_matches_reference(mm, tmp_path, oracle_ref):
    """`python -m paper_2007_06048_b200 model` (tools/cli.cpp:264-272): the
    parameter block, the run and the shot record in the reference's format --
    traces bit-identical to the reference's own run() of the same command."""
    import io
    from paper_2007_06048_b200 import driver, shotio
    from paper_2007_06048_b200.__main__ import main as cli_main
    n, nsteps = (64, 60, 62), 20
    out, err = io.StringIO(), io.StringIO()
    argv = ["model", "--ngrid", ",".join(map(str, n)), "--nsteps", str(nsteps),
            "--output", str(tmp_path / "shot.bin")]
    assert cli_main(argv, out, err) == 0, err.getvalue()
    cfg = mm.SimConfig(ngrid=n, nsteps=nsteps)
    model = mm.default_layered_model(mm.make_grid(n, cfg.dgrid))
    text = out.getvalue()
    assert text.startswith(driver.render_parameter_block(cfg, model))
    assert "Time Kernel" in text and "Time Modeling" in text
    rec = shotio.load_record(tmp_path / "shot.bin")
    vp, _, _ = oracle_ref.layered_model(n)
    ref = oracle_ref.run(n, vp, nsteps=nsteps, nthreads=8)
    assert rec.dt == ref["dt"] and rec.nsteps == nsteps
    assert np.array_equal(rec.traces, ref["traces"])


@pytest.mark.parametrize("mode", ["fast", "strict"])
@pytest.mark.parametrize("src_z", [0, 2, 9])
def test_step_epilogue_edge_placements(mm, oracle_port, mode, src_z):
    """k_epilogue forms injection, free surface and receiver sampling in one
    launch: a receiver on the source point, receivers on the surface plane and
    within R of it, a source on the surface (zeroed by it) and within R of it
    (mirrored) -- run() and step()+record() both equal the oracle's
    inject -> free surface -> record order (propagator_impl.hpp:166-172,
    source.cpp:61-66)."""
    n, nd, steps = (26, 22, 24), (5, 4, 6), 14
    h = (20.0, 20.0, 20.0)
    grid = mm.make_grid(n, h)
    m = mm.random_model(grid, seed=11)
    dt = 1e-3
    w = mm.ricker(25.0, dt, steps).samples * 1e3
    src = (13, 11, src_z)
    rec = np.array([src, (13, 11, 0), (12, 11, 0), (13, 11, 1), (13, 11, 3), (0, 0, 0),
                    (25, 21, 23), (14, 11, src_z)])
    ref = oracle_port.engine(n, m.vp, d=h, ndamping=nd, free_surface=True, taper=True, dt=dt,
                             vmax=m.vmax)
    want = np.zeros((len(rec), steps), np.float32)
    for s in range(steps):
        ref.step(float(w[s]), src)
        p = ref.pressure().reshape(grid.shape)
        want[:, s] = [p[i + 4, j + 4, k + 4] for i, j, k in rec]
    assert (np.abs(want).max() > 0) == (src_z != 0)  # a source on the surface is zeroed
    opts = mm.EngineOptions(ndamping=nd, taper=True, free_surface=True)
    for use_loop in (False, True):
        e = mm.AcousticCdEngine(grid, (0, 0, 0), n, m.vp, opts, dt, m.vmax, mode=mode)
        e.set_receivers(rec, steps)
        if use_loop:
            e.run(w, src)
        else:
            for s in range(steps):
                e.step(float(w[s]), src)
                e.record(s)
        assert np.array_equal(e.pressure(), ref.pressure().reshape(grid.shape)), use_loop
        assert np.array_equal(e.traces(), want), use_loop
