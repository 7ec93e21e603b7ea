"""acoustic_iso (variable density), SURVEY.md §8(f) row 4 -- CPU side.

Pins the oracle's restatement of AcousticVdEngine<float> (oracle/
minimod_oracle.c, ref: propagator_impl.hpp:175-295) against fixtures the
reference build generated (tests/golden/make_golden.py vd) and against the
reference itself, and the product's host numerics for this engine
(staggered weights stencil.cpp:76-97, integrate_wavelet source.cpp:30-38)
against the reference.  The GPU engine is checked in test_gpu_vd.py.
"""
import numpy as np
import pytest

from conftest import load_golden

VD_GOLDEN = ["vd_cpml", "vd_r2_fs", "vd_r8"]


@pytest.mark.parametrize("name", VD_GOLDEN)
def test_oracle_vd_matches_golden(oracle_port, name):
    g = load_golden(name)
    n, r = tuple(g["n"]), int(g["radius"])
    e = oracle_port.vd_engine(n, g["vp"], g["rho"], radius=r, ndamping=tuple(g["ndamping"]),
                              free_surface=bool(g["free_surface"]), taper=bool(g["taper"]),
                              dt=float(g["dt"]))
    src = tuple(g["src"])
    nd2 = int(g["ndamping"][2])
    for s in range(int(g["steps"])):
        e.step(float(g["wavelet"][s]), src)
        assert np.array_equal(e.pressure()[r:-r, r:-r, r + nd2], g["surface"][s]), s
    assert np.array_equal(e.pressure(), g["p"])
    for ax, key in enumerate(("vx", "vy", "vz")):
        assert np.array_equal(e.velocity(ax), g[key]), key
    assert np.abs(g["p"]).max() > 0


def test_oracle_vd_run_matches_golden(oracle_port):
    g = load_golden("run_vd_layered_32")
    n = tuple(g["n"])
    vp, _, vmax = oracle_port.layered_model(n)
    rho = np.full_like(vp, 1000.0)
    out = oracle_port.run_vd(n, vp, rho, nsteps=int(g["nsteps"]), ndamping=tuple(g["ndamping"]),
                             ntaper=tuple(g["ntaper"]), vmax=vmax)
    assert out["dt"] == float(g["dt"])
    assert np.array_equal(out["traces"], g["traces"])


@pytest.mark.parametrize("r", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("h", [1.0, 7.25, 20.0])
def test_staggered_coeffs_match_reference(mm, oracle_ref, oracle_port, r, h):
    ref = oracle_ref.staggered_first_derivative_coeffs(r, h)
    assert np.array_equal(mm.staggered_first_derivative_coeffs(r, h).c, ref)
    assert np.array_equal(oracle_port.staggered_first_derivative_coeffs(r, h), ref)


def test_staggered_coeffs_known_values(mm):
    # r = 2, h = 1: the classic (9/8, -1/24) staggered pair
    c = mm.staggered_first_derivative_coeffs(2, 1.0).c
    assert c[0] == pytest.approx(9.0 / 8.0, rel=1e-15)
    assert c[1] == pytest.approx(-1.0 / 24.0, rel=1e-15)
    with pytest.raises(mm.ConfigError):
        mm.staggered_first_derivative_coeffs(9, 1.0)


def test_integrate_wavelet_matches_reference(mm, oracle_ref):
    dt = 1.6101529682055116e-3
    w = mm.ricker(25.0, dt, 700)
    ours = mm.integrate_wavelet(w).samples
    assert np.array_equal(ours, oracle_ref.integrate_wavelet(w.samples, dt))
    assert abs(float(ours[-1])) < 1e-6  # a Ricker integrates to ~0


@pytest.mark.parametrize("fs,taper,r,nd", [(False, False, 4, (3, 2, 4)), (True, True, 4, (3, 2, 4)),
                                           (True, False, 2, (0, 3, 2)), (False, True, 8, (2, 0, 0))])
def test_oracle_vd_matches_reference_live(oracle_port, oracle_ref, fs, taper, r, nd):
    n = (14, 12, 17)
    rng = np.random.default_rng(5)
    sh = tuple(x + 2 * r for x in n)
    vp = np.zeros(sh, np.float32)
    rho = np.zeros(sh, np.float32)
    vp[r:-r, r:-r, r:-r] = rng.uniform(1500, 3000, n)
    rho[r:-r, r:-r, r:-r] = rng.uniform(800, 2500, n)
    vp = oracle_port.fill_ghosts_replicate(vp, n, r)
    rho = oracle_port.fill_ghosts_replicate(rho, n, r)
    kw = dict(d=(10.0, 12.0, 9.0), radius=r, ndamping=nd, free_surface=fs, taper=taper, dt=1e-3)
    a = oracle_port.vd_engine(n, vp, rho, **kw)
    b = oracle_ref.vd_engine(n, vp, rho, **kw)
    for s in range(10):
        amp = float(np.sin(0.7 * s))
        a.step(amp, (6, 5, 8))
        b.step(amp, (6, 5, 8))
    assert np.array_equal(a.pressure(), b.pressure())
    for ax in range(3):
        assert np.array_equal(a.velocity(ax), b.velocity(ax))


def test_oracle_vd_zero_and_constant_states(oracle_port):
    """test_propagator.cpp:47-71 and :118-133 on the oracle."""
    n, r = (14, 14, 14), 4
    vp = np.full(tuple(x + 2 * r for x in n), 1500.0, np.float32)
    rho = np.full_like(vp, 1000.0)
    e = oracle_port.vd_engine(n, vp, rho, d=(10.0, 10.0, 10.0), ndamping=(4, 4, 4), dt=1e-3)
    for _ in range(3):
        e.step(0.0, None)
    assert not e.pressure().any() and not any(e.velocity(a).any() for a in range(3))
    e.pressure_view()[...] = 0.75
    for _ in range(5):
        e.step(0.0, None)
    assert not any(e.velocity(a).any() for a in range(3))
    assert (e.pressure()[r:-r, r:-r, r:-r] == 0.75).all()


def test_vd_engine_rejects_missing_rho_without_gpu(mm):
    """propagator_impl.hpp:186-187 (checked before any device work)."""
    g = mm.make_grid((12, 12, 12), (10, 10, 10))
    m = mm.constant_model(g, 1500.0)
    assert not m.has_rho()
    with pytest.raises(mm.ValidationError, match="rho"):
        mm.AcousticVdEngine(g, m)
    cfg = mm.SimConfig(propagator="acoustic_iso", ngrid=(12, 12, 12), nsteps=3,
                       ndamping=(2, 2, 2))
    with pytest.raises(mm.ValidationError, match="rho"):
        mm.run(cfg, m)
    with pytest.raises(mm.ConfigError, match="propagator"):
        mm.run(mm.SimConfig(propagator="elastic_iso", ngrid=(12, 12, 12)), m)


def test_vd_model_validation(mm):
    g = mm.make_grid((6, 6, 6), (10, 10, 10))
    m = mm.default_layered_model(g)
    assert m.has_rho() and (m.rho == 1000.0).all()  # model.cpp:63-77, ghosts included
    bad = mm.EarthModel(g, g.field(1500.0), rho=g.field(1000.0))
    g.inner(bad.rho)[1, 2, 3] = -1.0
    with pytest.raises(mm.ValidationError, match="rho"):
        mm.validate_model(bad)
    rho = np.pad(np.full(g.n, 900.0, np.float32), g.radius)  # zero ghosts
    ok = mm.validate_model(mm.EarthModel(g, g.field(1500.0), rho=rho))
    assert (ok.rho == 900.0).all()  # ghosts replicated
