"""Host-side setup numerics of the product library (C++ behind the C ABI) equal
the pinned oracle bit for bit.  CPU only (no device calls)."""
import numpy as np
import pytest

from oracle.oracle import ghosted_shape


@pytest.mark.parametrize("radius", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("h", [1.0, 0.85, 10.0, 20.0])
def test_coefficients_bitwise(mm, oracle_port, radius, h):
    s = mm.second_derivative_coeffs(radius, h)
    c, center = oracle_port.second_derivative_coeffs(radius, h)
    assert np.array_equal(s.c, c) and s.center == center
    assert np.array_equal(mm.central_first_derivative_coeffs(radius, h).c,
                          oracle_port.central_first_derivative_coeffs(radius, h))


def test_coefficient_errors(mm):
    with pytest.raises(mm.ConfigError):
        mm.second_derivative_coeffs(0, 1.0)
    with pytest.raises(mm.ConfigError):
        mm.second_derivative_coeffs(9, 1.0)
    with pytest.raises(mm.ConfigError):
        mm.central_first_derivative_coeffs(4, 0.0)


def test_monomial_exactness(mm):
    # acceptance.cpp:34-68 (criterion 1): exact on x^q, q <= 2r
    x0, h = 0.37, 0.85
    for radius in (1, 2, 4):
        s2 = mm.second_derivative_coeffs(radius, h)
        s1 = mm.central_first_derivative_coeffs(radius, h)
        for q in range(2 * radius + 1):
            d2 = s2.center * x0 ** q + sum(
                s2.c[m - 1] * ((x0 + m * h) ** q + (x0 - m * h) ** q) for m in range(1, radius + 1))
            d1 = sum(s1.c[m - 1] * ((x0 + m * h) ** q - (x0 - m * h) ** q)
                     for m in range(1, radius + 1))
            w2 = 0.0 if q < 2 else q * (q - 1) * x0 ** (q - 2)
            w1 = 0.0 if q < 1 else q * x0 ** (q - 1)
            assert abs(d2 - w2) / max(1.0, abs(w2)) < 1e-8
            assert abs(d1 - w1) / max(1.0, abs(w1)) < 1e-8


@pytest.mark.parametrize("radius", [1, 2, 4, 8])
def test_cfl_dt_bitwise(mm, oracle_port, radius):
    g = mm.make_grid((10, 10, 10), (20.0, 15.0, 10.0), radius)
    m = mm.constant_model(g, 4500.0)
    assert mm.cfl_dt(m, g, 0.8) == oracle_port.cfl_dt(4500.0, radius, (20.0, 15.0, 10.0), 0.8)
    with pytest.raises(mm.ConfigError):
        mm.cfl_dt(m, g, 1.5)


def test_ricker_bitwise(mm, oracle_port):
    for dt in (1.61015297e-3, 1e-3, 1.7777777777e-3):
        assert np.array_equal(mm.ricker(25.0, dt, 777).samples, oracle_port.ricker(25.0, dt, 777))
    with pytest.raises(mm.ConfigError):
        mm.ricker(25.0, 0.05, 10)  # dt > 1/(2 fmax)
    with pytest.raises(mm.ConfigError):
        mm.ricker(0.0, 1e-3, 10)


@pytest.mark.parametrize("fs", [False, True])
def test_profile_bitwise(mm, oracle_port, fs):
    n, h, nd = (60, 70, 80), (20.0, 15.0, 10.0), (12, 0, 9)
    dt = float(np.float32(1.2e-3))
    prof = mm.build_profile(n, h, nd, 25.0, 4500.0, dt, 1e-3, fs)
    vp = np.full(ghosted_shape(n, 4), 4500.0, np.float32)
    e = oracle_port.engine(n, vp, d=h, ndamping=nd, free_surface=fs, dt=1.2e-3, vmax=4500.0)
    for ax in range(3):
        assert np.array_equal(prof.axis[ax].a, e.profile_array(0, ax))
        assert np.array_equal(prof.axis[ax].b, e.profile_array(1, ax))
        assert np.array_equal(prof.axis[ax].inv_kappa, e.profile_array(2, ax))
        assert prof.d0[ax] == e.d0(ax)
    with pytest.raises(mm.ConfigError):
        mm.build_profile(n, h, nd, 25.0, 4500.0, dt, 1.0, fs)


def test_taper_and_models_bitwise(mm, oracle_port):
    n = (30, 34, 38)
    g = mm.make_grid(n, (20, 20, 20))
    rng = np.random.default_rng(3)
    vp = g.field()
    g.inner(vp)[...] = rng.uniform(1500, 4500, size=n)
    vp = oracle_port.fill_ghosts_replicate(vp, n, 4)
    for nt, off, gn in [((3, 3, 3), (0, 0, 0), n), ((2, 4, 1), (0, 0, 10), (30, 34, 60)),
                        ((3, 3, 3), (0, 0, 5), (30, 34, 43))]:
        a = mm.taper_material(vp.copy(), nt, off, gn, g)
        b = oracle_port.taper_material(vp, n, 4, nt, off, gn)
        assert np.array_equal(a, b)
    m = mm.default_layered_model(g)
    vp2, lo, hi = oracle_port.layered_model(n)
    assert np.array_equal(m.vp, vp2) and (m.vmin, m.vmax) == (lo, hi) == (1500.0, 4500.0)
    f = vp.copy()
    f[:4] = 0
    assert np.array_equal(mm.fill_ghosts_replicate(f, g), vp)


def test_validation_errors(mm):
    g = mm.make_grid((8, 8, 8), (1, 1, 1))
    vp = g.field(1500.0)
    g.inner(vp)[2, 2, 2] = -1.0
    with pytest.raises(mm.ValidationError):
        mm.validate_model(mm.EarthModel(g, vp))
    with pytest.raises(mm.ConfigError):
        mm.make_grid((0, 10, 10), (1, 1, 1))
    with pytest.raises(mm.ConfigError, match="y"):
        mm.partition_regions(mm.make_grid((100, 100, 100), (20, 20, 20)), (10, 50, 10))


def test_partition_and_receivers(mm):
    # test_grid.cpp:54-63 and test_source.cpp:103-114
    g = mm.make_grid((240, 240, 240), (20, 20, 20))
    p = mm.partition_regions(g, (27, 27, 27))
    assert p.inner.lo == (27, 27, 27) and p.inner.hi == (213, 213, 213)
    assert sum(s.volume() for s in p.slabs) == 240 ** 3 - 186 ** 3
    geo = mm.default_receivers(g, (27, 27, 27))
    assert geo.nreceivers() == 57600 and tuple(geo.receivers[1]) == (0, 1, 27)
    assert geo.source_loc == (120, 120, 120)
