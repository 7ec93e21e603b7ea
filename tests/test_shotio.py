"""On-disk formats and the report, pinned against the reference's own writers
(SURVEY.md §8(f)): save_record (source.cpp:68-95), load_model / save_model
(model.cpp:64-190), render_parameter_block / render_timing (driver.cpp:150-215),
and the `minimod model` command line (tools/cli.cpp:256-272)."""
import io
import json
import os

import numpy as np
import pytest

from paper_2007_06048_b200 import driver, numerics, shotio
from paper_2007_06048_b200.__main__ import main as cli_main
from paper_2007_06048_b200._lib import ConfigError


def _record(nrec=5, nsteps=7, dt=1.6101529682055116e-3, src=(3, 4, 5), inc=(2, 1), seed=0):
    rng = np.random.default_rng(seed)
    geo = numerics.AcquisitionGeometry(src, np.zeros((nrec, 3), np.int32), inc)
    return numerics.ShotRecord(nsteps, dt, geo,
                               rng.standard_normal((nrec, nsteps)).astype(np.float32))


def test_record_matches_reference_writer(tmp_path, oracle_ref):
    rec = _record()
    ours, theirs = tmp_path / "ours.bin", tmp_path / "ref.bin"
    shotio.save_record(rec, ours)
    oracle_ref.save_record(rec.traces, rec.dt, theirs, source_loc=rec.geometry.source_loc,
                           receiver_increment=rec.geometry.receiver_increment)
    assert ours.read_bytes() == theirs.read_bytes()          # raw f32, trace-major
    a = json.loads((tmp_path / "ours.bin.json").read_text())
    b = json.loads((tmp_path / "ref.bin.json").read_text())
    assert a == b and sorted(a) == sorted(b)
    # nothing left behind by the tmp + rename protocol
    assert sorted(os.listdir(tmp_path)) == ["ours.bin", "ours.bin.json", "ref.bin",
                                            "ref.bin.json"]


def test_record_round_trip(tmp_path):
    rec = _record(nrec=3, nsteps=11, seed=4)
    shotio.save_record(rec, tmp_path / "t.bin")
    back = shotio.load_record(tmp_path / "t.bin")
    assert back.nsteps == rec.nsteps and back.dt == rec.dt
    assert np.array_equal(back.traces, rec.traces)
    assert tuple(back.geometry.source_loc) == rec.geometry.source_loc
    assert back.at(2, 10) == float(rec.traces[2, 10])


def test_record_shape_and_path_errors(tmp_path):
    rec = _record()
    rec.traces = rec.traces[:, :3]
    with pytest.raises(ConfigError):
        shotio.save_record(rec, tmp_path / "x.bin")
    with pytest.raises(ConfigError):
        shotio.save_record(_record(), "")
    (tmp_path / "y.bin").write_bytes(b"\0" * 8)
    (tmp_path / "y.bin.json").write_text(json.dumps(
        {"dt": 1.0, "nsteps": 7, "nreceivers": 5, "source_loc": [0, 0, 0],
         "receiver_increment": [1, 1], "nshots": 1}))
    with pytest.raises(ConfigError, match="size mismatch"):
        shotio.load_record(tmp_path / "y.bin")


def test_model_matches_reference_writer_and_reader(tmp_path, oracle_ref):
    n, r = (6, 7, 9), 4
    grid = numerics.make_grid(n, (20.0, 20.0, 20.0), r)
    model = numerics.random_model(grid, seed=2)
    (tmp_path / "ours").mkdir()
    (tmp_path / "ref").mkdir()
    shotio.save_model(model, tmp_path / "ours" / "m.json")
    oracle_ref.save_model(model.vp, n, grid.d, r, tmp_path / "ref" / "m.json")
    assert ((tmp_path / "ours" / "vp.f32").read_bytes() ==
            (tmp_path / "ref" / "vp.f32").read_bytes())
    assert ((tmp_path / "ours" / "m.json").read_text() ==
            (tmp_path / "ref" / "m.json").read_text())
    # both readers on the reference's files: same validated, ghost-filled vp
    rn, rd, rvp, rvmin, rvmax = oracle_ref.load_model(tmp_path / "ref" / "m.json")
    m = shotio.load_model(tmp_path / "ref" / "m.json")
    assert tuple(m.grid.n) == rn and tuple(m.grid.d) == rd
    assert np.array_equal(m.vp, rvp)
    assert (m.vmin, m.vmax) == (rvmin, rvmax)


def test_model_manifest_errors(tmp_path):
    grid = numerics.make_grid((4, 4, 4), (10.0, 10.0, 10.0))
    shotio.save_model(numerics.constant_model(grid, 2000.0), tmp_path / "m.json")
    j = json.loads((tmp_path / "m.json").read_text())
    for key, val, msg in (("dtype", "f64le", "dtype"), ("order", "x-fastest", "order")):
        bad = dict(j, **{key: val})
        (tmp_path / "b.json").write_text(json.dumps(bad))
        with pytest.raises(ConfigError, match=msg):
            shotio.load_model(tmp_path / "b.json")
    (tmp_path / "vp.f32").write_bytes(b"\0" * 12)
    with pytest.raises(ConfigError, match="size mismatch"):
        shotio.load_model(tmp_path / "m.json")
    (tmp_path / "c.json").write_text("{not json")
    with pytest.raises(ConfigError, match="malformed"):
        shotio.load_model(tmp_path / "c.json")
    with pytest.raises(ConfigError, match="cannot open"):
        shotio.load_model(tmp_path / "missing.json")


@pytest.mark.parametrize("ngrid,nd,src,nthreads", [
    ((240, 240, 240), (27, 27, 27), None, 1),
    ((100, 120, 90), (10, 12, 9), (50, 60, 45), 8),
])
def test_report_matches_reference(oracle_ref, ngrid, nd, src, nthreads):
    cfg = driver.SimConfig(ngrid=ngrid, dgrid=(20.0, 12.5, 7.25), nsteps=300, fmax=17.5,
                           cfl=0.7, ndamping=nd, ntaper=(3, 2, 1), source_loc=src,
                           receiver_increment=(2, 3))
    model = numerics.EarthModel(numerics.make_grid(ngrid, cfg.dgrid), None, 1500.0, 4512.5)
    rep = driver.RunReport(1e-3, 12.3456, 13.0049, 300)
    ours = driver.render_parameter_block(cfg, model, nthreads=nthreads) + driver.render_timing(rep)
    ref = oracle_ref.render_report(
        ngrid=ngrid, dgrid=cfg.dgrid, nsteps=300, fmax=17.5, cfl=0.7, radius=4, ndamping=nd,
        ntaper=(3, 2, 1), source_loc=src, receiver_increment=(2, 3),
        source_increment=(1, 1, 0), nshots=1, time_rec=0.0, nthreads=nthreads, vmin=1500.0,
        vmax=4512.5, kernel_s=12.3456, modeling_s=13.0049)
    assert ours == ref


@pytest.mark.parametrize("argv", [
    [], ["dist"], ["model", "--ngrid", "10,10"], ["model", "--nsteps", "0"],
    ["model", "--fmax", "-1"], ["model", "--propagator", "elastic_iso"],
    ["model", "--dgrid", "1,a,1"], ["model", "--bogus"],
])
def test_cli_config_errors_exit_2(argv):
    out, err = io.StringIO(), io.StringIO()
    assert cli_main(argv, out, err) == 2
    assert err.getvalue().startswith("error: ")


def test_cli_help():
    out = io.StringIO()
    assert cli_main(["--help"], out, io.StringIO()) == 0
    assert "model" in out.getvalue()


def test_model_with_rho_matches_reference(tmp_path, oracle_ref, mm):
    """save_model / load_model with a density volume (model.cpp:122-184): the
    acoustic_iso engine's model files."""
    n = (5, 6, 7)
    g = mm.make_grid(n, (10.0, 12.0, 14.0))
    rng = np.random.default_rng(9)
    vp, rho = g.field(), g.field()
    g.inner(vp)[...] = rng.uniform(1500, 4000, n).astype(np.float32)
    g.inner(rho)[...] = rng.uniform(900, 2600, n).astype(np.float32)
    model = mm.validate_model(mm.EarthModel(g, vp, rho=rho))
    (tmp_path / "ours").mkdir()
    (tmp_path / "ref").mkdir()
    shotio.save_model(model, tmp_path / "ours" / "m.json")
    oracle_ref.save_model_rho(model.vp, model.rho, n, g.d, 4, tmp_path / "ref" / "m.json")
    for f in ("vp.f32", "rho.f32", "m.json"):
        assert (tmp_path / "ours" / f).read_bytes() == (tmp_path / "ref" / f).read_bytes(), f
    back = shotio.load_model(tmp_path / "ref" / "m.json")
    assert np.array_equal(back.rho, oracle_ref.load_model_rho(tmp_path / "ref" / "m.json", n))
    assert np.array_equal(back.rho, model.rho) and np.array_equal(back.vp, model.vp)
    (tmp_path / "ours" / "rho.f32").write_bytes(b"\0" * 8)
    with pytest.raises(ConfigError, match="size mismatch"):
        shotio.load_model(tmp_path / "ours" / "m.json")
