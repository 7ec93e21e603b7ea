"""Physics acceptance criteria of the reference on the GPU engine (fast mode).

The reference's acceptance binary (tests/acceptance.cpp) pins the hot path
with end-to-end physics checks besides the bitwise oracles; these restate
criteria 2, 3 and 10 on the B200 engine:

* 2: a free-space Ricker pulse matches the analytic solution
  p(t) = h^3 w(t - r/v) / (4 pi r) within 5 % of its peak, and the misfit
  shrinks with the grid spacing (acceptance.cpp:104-139);
* 3: CPML reflections <= 1 % of the direct arrival while a hard truncation
  reflects >= 30 % (acceptance.cpp:143-172);
* 10: 2000 steps stay finite and the energy leaves the box
  (acceptance.cpp:428-455);
* 9 (acoustic_iso vs acoustic_iso_cd): the variable-density engine's pulse
  arrives within one sample of the constant-density one
  (acceptance.cpp:370-425).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run_point(mm, n, h, nd, cfl, nsteps, src, rcv, vp_val=1500.0):
    """acceptance.cpp:74-93 run_cd_point: constant model, Ricker at src, the
    post-step pressure at rcv every step (device receiver, one column/step)."""
    g = mm.make_grid((n, n, n), (h, h, h))
    m = mm.constant_model(g, vp_val)
    dt = mm.cfl_dt(m, g, cfl)
    w = mm.ricker(25.0, dt, nsteps).samples
    with mm.AcousticCdEngine(g, (0, 0, 0), g.n, m.vp, mm.EngineOptions(ndamping=(nd, nd, nd)),
                             dt, vp_val) as e:
        e.set_receivers(np.array([rcv], np.int32), nsteps)
        e.run(w, src)
        return e.traces(nsteps)[0].astype(np.float64), dt


def ricker_continuous(t, fmax=25.0):
    fp = fmax / 2.5
    tau = math.pi * fp * (t - 1.5 / fp)
    a = tau * tau
    return (1.0 - 2.0 * a) * math.exp(-a)


def analytic_misfit(trace, dt, h, dist, window):
    err = ref_max = 0.0
    for s, v in enumerate(trace):
        t = (s + 1) * dt  # sample s holds the post-step field
        if t >= window:
            break
        ref = h ** 3 * ricker_continuous(t - dist / 1500.0) / (4.0 * math.pi * dist)
        ref_max = max(ref_max, abs(ref))
        err = max(err, abs(v - ref))
    return err / ref_max


def test_free_space_pulse_matches_analytic_and_converges(mm):
    window = 0.45
    _, dt_f = run_point(mm, 120, 10.0, 0, 0.4, 1, (60, 60, 60), (80, 60, 60))
    fine, _ = run_point(mm, 120, 10.0, 0, 0.4, int(window / dt_f) + 2, (60, 60, 60),
                        (80, 60, 60))
    _, dt_c = run_point(mm, 60, 20.0, 0, 0.4, 1, (30, 30, 30), (40, 30, 30))
    coarse, _ = run_point(mm, 60, 20.0, 0, 0.4, int(window / dt_c) + 2, (30, 30, 30),
                          (40, 30, 30))
    mis_f = analytic_misfit(fine, dt_f, 10.0, 200.0, window)
    mis_c = analytic_misfit(coarse, dt_c, 20.0, 200.0, window)
    assert mis_f <= 0.05, mis_f
    assert mis_f < mis_c, (mis_f, mis_c)


def test_cpml_absorbs_boundary_reflections(mm):
    h, window = 20.0, 1.25
    _, dt = run_point(mm, 100, h, 0, 0.8, 4, (50, 50, 50), (50, 50, 15))
    nsteps = int(window / dt) + 2
    ref, _ = run_point(mm, 160, h, 0, 0.8, nsteps, (80, 80, 80), (80, 80, 45))
    cpml, _ = run_point(mm, 100, h, 10, 0.8, nsteps, (50, 50, 50), (50, 50, 15))
    hard, _ = run_point(mm, 100, h, 0, 0.8, nsteps, (50, 50, 50), (50, 50, 15))
    peak = np.abs(ref).max()
    r_cpml = np.abs(cpml - ref).max() / peak
    r_hard = np.abs(hard - ref).max() / peak
    assert r_cpml <= 0.01, r_cpml
    assert r_hard >= 0.30, r_hard


def test_long_run_stays_finite_and_loses_energy(mm):
    cfg = mm.SimConfig(ngrid=(48, 48, 48), nsteps=2000, ndamping=(8, 8, 8))
    model = mm.default_layered_model(mm.make_grid(cfg.ngrid, cfg.dgrid))
    rec, rep = mm.run(cfg, model)
    inject = rep.dt * rep.dt * model.vmax * model.vmax  # unit-amplitude source scale
    a = np.abs(rec.traces)
    assert np.isfinite(a).all() and a.max() > 0.0
    assert a[:, -100:].max() <= 10.0 * inject


def best_lag(a, b, max_lag):
    """acceptance.cpp:370-390: the lag maximising the normalised correlation."""
    n = min(len(a), len(b))
    best, arg = -1.0, -max_lag - 1
    for lag in range(-max_lag, max_lag + 1):
        i = np.arange(n)
        j = i + lag
        ok = (j >= 0) & (j < n)
        x, y = a[i[ok]], b[j[ok]]
        corr = abs(float(np.dot(x, y))) / math.sqrt(float(np.dot(x, x)) * float(np.dot(y, y)))
        if corr > best:
            best, arg = corr, lag
    return arg


def test_vd_arrives_in_phase_with_cd(mm):
    """Criterion 9 (acceptance.cpp:392-425) for the engines this repo serves:
    the first-order acoustic_iso pulse (integrated Ricker) arrives within one
    sample of the second-order acoustic_iso_cd one."""
    g = mm.make_grid((50, 50, 50), (20.0, 20.0, 20.0))
    m = mm.constant_model(g, 1500.0, rho=1000.0)
    dt = mm.cfl_dt(m, g, 0.8)
    nsteps, src, rcv = 500, (25, 25, 25), np.array([[25, 25, 38]], np.int32)
    w = mm.ricker(25.0, dt, nsteps)
    wi = mm.integrate_wavelet(w).samples
    opts = mm.EngineOptions(ndamping=(10, 10, 10))
    with mm.AcousticCdEngine(g, (0, 0, 0), g.n, m.vp, opts, dt, 1500.0) as cd, \
            mm.AcousticVdEngine(g, m, opts, dt) as vd:
        cd.set_receivers(rcv, nsteps)
        vd.set_receivers(rcv, nsteps)
        cd.run(w.samples, src)
        vd.run(wi, src)
        t_cd = cd.traces(nsteps)[0].astype(np.float64)
        t_vd = vd.traces(nsteps)[0].astype(np.float64)
    assert abs(best_lag(t_cd, t_vd, 20)) <= 1
