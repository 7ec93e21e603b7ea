"""The CPU oracle is pinned: golden fixtures (made by the reference build) and,
where oracle/_ref exists, the live reference agree with the C restatement bit
for bit.  CPU only."""
import numpy as np
import pytest

from conftest import load_golden
from oracle.oracle import ghosted_shape

ENGINE_CASES = ["eng_plain_20", "eng_cpml_aniso", "eng_cpml_fs", "eng_r2_fs", "eng_r8",
                "eng_nd_0x", "eng_nd_0y"]


def run_oracle_case(o, g):
    n = tuple(int(x) for x in g["n"])
    r = int(g["radius"])
    nd = tuple(int(x) for x in g["ndamping"])
    e = o.engine(n, g["vp"], radius=r, ndamping=nd, free_surface=bool(g["free_surface"]),
                 taper=bool(g["taper"]), dt=float(g["dt"]), vmax=float(g["vmax"]))
    src = tuple(int(x) for x in g["src"])
    surf = []
    for s in range(int(g["steps"])):
        e.step(float(g["wavelet"][s]), src)
        surf.append(e.pressure()[r:-r, r:-r, r + nd[2]].copy())
    return e, np.stack(surf)


@pytest.mark.parametrize("name", ENGINE_CASES)
def test_port_matches_reference_golden_bitwise(oracle_port, name):
    g = load_golden(name)
    e, surf = run_oracle_case(oracle_port, g)
    assert np.array_equal(e.pressure(), g["p_cur"])
    assert np.array_equal(e.pressure_prev(), g["p_prev"])
    assert np.array_equal(surf, g["surface"])
    assert np.abs(g["p_cur"]).max() > 0


def test_port_degenerate_cpml_golden(oracle_port):
    g = load_golden("eng_degenerate")
    n = (20, 20, 20)
    vp = np.full(ghosted_shape(n, 4), 2000.0, np.float32)
    a = oracle_port.engine(n, vp, ndamping=(5, 5, 5), dt=1e-3, vmax=2000.0)
    for ax in range(3):
        a.profile_array(0, ax)[:] = 0.0
        a.profile_array(1, ax)[:] = 1.0
        a.profile_array(2, ax)[:] = 1.0
    b = oracle_port.engine(n, vp, dt=1e-3, vmax=2000.0)
    a.set_state(g["p0"], g["p1"])
    b.set_state(g["p0"], g["p1"])
    for _ in range(5):
        a.step(0.0, None)
        b.step(0.0, None)
    assert np.array_equal(a.pressure(), g["p_cur"])
    assert np.array_equal(b.pressure(), g["p_cur"])  # test_cpml.cpp:134-177


def test_port_run_golden(oracle_port):
    g = load_golden("run_layered_32")
    n = tuple(int(x) for x in g["n"])
    vp, _, vmax = oracle_port.layered_model(n)
    out = oracle_port.run(n, vp, nsteps=int(g["nsteps"]), ndamping=tuple(g["ndamping"]),
                          ntaper=tuple(g["ntaper"]))
    assert out["dt"] == float(g["dt"])
    assert np.array_equal(out["traces"], g["traces"])


def test_known_answers(oracle_port):
    # test_cpml.cpp:11-23: d0 = 3*4500*ln(1000)/(2*540) = 86.3469
    n = (60, 60, 60)
    vp = np.full(ghosted_shape(n, 4), 4500.0, np.float32)
    e = oracle_port.engine(n, vp, ndamping=(27, 27, 27), dt=1e-3, vmax=4500.0)
    want = 3.0 * 4500.0 * np.log(1000.0) / (2.0 * 540.0)
    assert abs(want - 86.3469) < 1e-3
    for ax in range(3):
        assert abs(e.d0(ax) - want) <= 1e-12 * want
    # test_propagator.cpp:73-83: injection dt^2 vp^2 = 2.25 at one point
    n = (16, 16, 16)
    vp = np.full(ghosted_shape(n, 4), 1500.0, np.float32)
    e = oracle_port.engine(n, vp, d=(10, 10, 10), dt=1e-3, vmax=1500.0)
    e.step(1.0, (8, 8, 8))
    p = e.pressure()
    assert abs(p[12, 12, 12] - 2.25) < 2.25e-6
    assert np.count_nonzero(p) == 1
    # Appendix A constants
    c, center = oracle_port.second_derivative_coeffs(4, 1.0)
    assert np.allclose(c, [1.6, -0.2, 8 / 315, -1 / 560], rtol=0, atol=1e-15)
    dt = oracle_port.cfl_dt(4500.0, 4, (20.0, 20.0, 20.0), 0.8)
    assert abs(dt - 1.61015297e-3) < 1e-11
    # cfl radius 1 = 1/sqrt(3) (test_driver.cpp:24-31)
    assert abs(oracle_port.cfl_dt(1.0, 1, (1.0, 1.0, 1.0), 1.0) - 1 / np.sqrt(3)) < 1e-12


def test_port_vs_live_reference_random_cases(oracle_port, oracle_ref):
    """Extra configurations straight against the reference build (when present)."""
    rng = np.random.default_rng(5)
    cases = [((30, 26, 34), 4, (6, 5, 7), True, True, (3, 2, 1)),
             ((22, 30, 26), 3, (4, 7, 5), False, True, (2, 2, 2)),
             ((28, 28, 28), 1, (6, 6, 6), True, False, (3, 3, 3))]
    for n, r, nd, fs, taper, ntaper in cases:
        vp = np.zeros(ghosted_shape(n, r), np.float32)
        vp[r:-r, r:-r, r:-r] = rng.uniform(1500, 4500, size=n)
        vp = oracle_port.fill_ghosts_replicate(vp, n, r)
        kw = dict(radius=r, ndamping=nd, free_surface=fs, taper=taper, ntaper=ntaper,
                  dt=1.1e-3, vmax=4500.0)
        a = oracle_port.engine(n, vp, **kw)
        b = oracle_ref.engine(n, vp, **kw)
        w = oracle_port.ricker(25.0, 1.1e-3, 60)
        for s in range(60):
            a.step(w[s], (n[0] // 3, n[1] // 2, n[2] // 2))
            b.step(w[s], (n[0] // 3, n[1] // 2, n[2] // 2))
        assert np.array_equal(a.pressure(), b.pressure()), (n, r)


def test_port_distributed_slab_equals_single(oracle_port):
    """z-slab engines with offsets + ghost exchange reproduce the single engine
    bitwise (test_dist.cpp:107-118 restated for z cuts)."""
    n, r, nd = (24, 24, 40), 4, (4, 4, 4)
    vp, _, vmax = oracle_port.layered_model(n)
    w = oracle_port.ricker(25.0, 1.61e-3, 30)
    src = (12, 12, 20)
    whole = oracle_port.engine(n, vp, ndamping=nd, taper=True, ntaper=(2, 2, 2), dt=1.61e-3,
                               vmax=vmax)
    cuts = [0, 18, 40]  # legal: >= nd + r = 8 from both faces
    parts = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        sub = vp[:, :, lo:hi + 2 * r].copy()
        parts.append(oracle_port.engine((n[0], n[1], hi - lo), sub, offset=(0, 0, lo),
                                        global_n=n, ndamping=nd, taper=True, ntaper=(2, 2, 2),
                                        dt=1.61e-3, vmax=vmax))
    for s in range(30):
        whole.step(w[s], src)
        # exchange p_cur ghosts (face only), then step every part
        cur = [p.pressure() for p in parts]
        prev = [p.pressure_prev() for p in parts]
        lo_p, hi_p = cur
        lo_p[:, :, -r:] = hi_p[:, :, r:2 * r]
        hi_p[:, :, :r] = lo_p[:, :, -2 * r:-r]
        for p, c, q in zip(parts, cur, prev):
            p.set_state(q, c)
        for (lo, hi), p in zip(zip(cuts[:-1], cuts[1:]), parts):
            owns = lo <= src[2] < hi
            p.step(w[s], (src[0], src[1], src[2] - lo) if owns else None)
    full = whole.pressure()
    for (lo, hi), p in zip(zip(cuts[:-1], cuts[1:]), parts):
        assert np.array_equal(p.pressure()[:, :, r:-r], full[:, :, r + lo:r + hi])
