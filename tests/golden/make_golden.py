"""Generate tests/golden/*.npz from the REFERENCE build (oracle/_ref).

Run in the authoring container, where /root/reference exists and
`make -C oracle` has built oracle/_ref/libminimod_ref.so:

    python tests/golden/make_golden.py [all|cd|vd]

Every array below comes from the reference's own AcousticCdEngine<float>,
AcousticVdEngine<float> and run() (through oracle/ref_shim.cpp); nothing is computed by this repo's code.
Inputs (vp models) are stored alongside, so the fixtures are self-contained.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Oracle, ghosted_shape  # noqa: E402

OUT = Path(__file__).resolve().parent
R = Oracle("reference")
P = Oracle("port")


def rand_vp(n, r, seed, lo=1500.0, hi=4500.0):
    rng = np.random.default_rng(seed)
    vp = np.zeros(ghosted_shape(n, r), np.float32)
    vp[r:r + n[0], r:r + n[1], r:r + n[2]] = rng.uniform(lo, hi, size=n).astype(np.float32)
    return P.fill_ghosts_replicate(vp, n, r)


ENGINE_CASES = {
    # name: (n, r, ndamping, free_surface, taper, steps, dt, seed)
    "eng_plain_20": ((20, 20, 20), 4, (0, 0, 0), False, False, 10, 1e-3, 31),
    "eng_cpml_aniso": ((24, 28, 32), 4, (5, 6, 7), False, True, 40, 1.2e-3, 7),
    "eng_cpml_fs": ((24, 28, 32), 4, (5, 6, 7), True, True, 40, 1.2e-3, 8),
    "eng_r2_fs": ((26, 22, 30), 2, (6, 4, 5), True, False, 40, 1.2e-3, 9),
    "eng_r8": ((36, 34, 38), 8, (5, 6, 7), False, False, 30, 1.0e-3, 10),
    "eng_nd_0x": ((24, 24, 24), 4, (0, 5, 5), False, True, 40, 1.2e-3, 11),
    "eng_nd_0y": ((24, 24, 24), 4, (5, 0, 5), False, True, 40, 1.2e-3, 12),
}


def engine_case(name, n, r, nd, fs, taper, steps, dt, seed):
    vp = rand_vp(n, r, seed)
    vmax = float(vp.max())
    e = R.engine(n, vp, radius=r, ndamping=nd, free_surface=fs, taper=taper, dt=dt, vmax=vmax)
    w = R.ricker(25.0, dt, steps)
    src = tuple(x // 2 for x in n)
    rec = []
    for s in range(steps):
        e.step(w[s], src)
        rec.append(e.pressure()[r:-r, r:-r, r + nd[2]].copy())
    np.savez_compressed(
        OUT / f"{name}.npz", n=np.array(n), radius=r, ndamping=np.array(nd), free_surface=int(fs),
        taper=int(taper), steps=steps, dt=np.float32(dt), vmax=vmax, src=np.array(src), vp=vp,
        wavelet=w, p_cur=e.pressure(), p_prev=e.pressure_prev(),
        surface=np.stack(rec).astype(np.float32))
    print(name, "max|p|", float(np.abs(e.pressure()).max()))


def degenerate_case():
    """test_cpml.cpp:134-177: a=0,b=1 CPML equals the plain engine bitwise."""
    n = (20, 20, 20)
    vp = np.full(ghosted_shape(n, 4), 2000.0, np.float32)
    rng = np.random.default_rng(21)
    p0 = np.zeros_like(vp)
    p1 = np.zeros_like(vp)
    p0[4:-4, 4:-4, 4:-4] = (1e-3 * rng.uniform(-1, 1, size=n)).astype(np.float32)
    p1[4:-4, 4:-4, 4:-4] = (1e-3 * rng.uniform(-1, 1, size=n)).astype(np.float32)
    a = R.engine(n, vp, ndamping=(5, 5, 5), dt=1e-3, vmax=2000.0)
    for ax in range(3):
        a.profile_array(0, ax)[:] = 0.0
        a.profile_array(1, ax)[:] = 1.0
        a.profile_array(2, ax)[:] = 1.0
    a.set_state(p0, p1)
    for _ in range(5):
        a.step(0.0, None)
    np.savez_compressed(OUT / "eng_degenerate.npz", p0=p0, p1=p1, p_cur=a.pressure())
    print("eng_degenerate done")


def run_case():
    """driver run(): 32^3 layered, nd 4, ntaper 2 (test_dist.cpp:95-104 config)."""
    n = (32, 32, 32)
    vp, vmin, vmax = R.layered_model(n)
    out = R.run(n, vp, nsteps=40, ndamping=(4, 4, 4), ntaper=(2, 2, 2))
    np.savez_compressed(OUT / "run_layered_32.npz", n=np.array(n), nsteps=40,
                        ndamping=np.array((4, 4, 4)), ntaper=np.array((2, 2, 2)),
                        traces=out["traces"], dt=out["dt"])
    print("run_layered_32 dt", out["dt"])


def checksum_case():
    """100^3 x 100 layered (the BASELINE oracle config): checksums + sampled traces."""
    n = (100, 100, 100)
    vp, vmin, vmax = R.layered_model(n)
    out = R.run(n, vp, nsteps=100, nthreads=8)
    pick = np.arange(0, n[0] * n[1], 97)
    np.savez_compressed(OUT / "run_layered_100.npz", n=np.array(n), nsteps=100, pick=pick,
                        traces=out["traces"][pick], dt=out["dt"],
                        trace_norm=float(np.linalg.norm(out["traces"].astype(np.float64))),
                        # final-field checksums measured on the reference
                        p_norm=159.223167, p_max=60.9030991)
    print("run_layered_100 dt", out["dt"])


# acoustic_iso (variable density): AcousticVdEngine<float>
VD_CASES = {
    # name: (n, r, ndamping, free_surface, taper, steps, dt, seed)
    "vd_cpml": ((22, 26, 30), 4, (5, 6, 7), False, True, 40, 1.0e-3, 41),
    "vd_r2_fs": ((24, 20, 28), 2, (6, 4, 5), True, False, 40, 1.0e-3, 42),
    "vd_r8": ((34, 34, 36), 8, (5, 6, 7), False, False, 25, 1.0e-3, 43),
}


def vd_case(name, n, r, nd, fs, taper, steps, dt, seed):
    vp = rand_vp(n, r, seed)
    rho = rand_vp(n, r, seed + 100, 1000.0, 2500.0)
    e = R.vd_engine(n, vp, rho, radius=r, ndamping=nd, free_surface=fs, taper=taper, dt=dt)
    w = R.integrate_wavelet(R.ricker(25.0, dt, steps), dt)
    src = tuple(x // 2 for x in n)
    rec = []
    for s in range(steps):
        e.step(w[s], src)
        rec.append(e.pressure()[r:-r, r:-r, r + nd[2]].copy())
    np.savez_compressed(
        OUT / f"{name}.npz", n=np.array(n), radius=r, ndamping=np.array(nd), free_surface=int(fs),
        taper=int(taper), steps=steps, dt=np.float32(dt), src=np.array(src), vp=vp, rho=rho,
        wavelet=w, p=e.pressure(), vx=e.velocity(0), vy=e.velocity(1), vz=e.velocity(2),
        surface=np.stack(rec).astype(np.float32))
    print(name, "max|p|", float(np.abs(e.pressure()).max()))


def vd_run_case():
    """driver run() with Propagator::AcousticIso: 32^3 layered (rho 1000)."""
    n = (32, 32, 32)
    vp, vmin, vmax = R.layered_model(n)
    rho = np.full_like(vp, 1000.0)
    out = R.run_vd(n, vp, rho, nsteps=60, ndamping=(4, 4, 4), ntaper=(2, 2, 2))
    np.savez_compressed(OUT / "run_vd_layered_32.npz", n=np.array(n), nsteps=60,
                        ndamping=np.array((4, 4, 4)), ntaper=np.array((2, 2, 2)),
                        traces=out["traces"], dt=out["dt"])
    print("run_vd_layered_32 dt", out["dt"], "max", float(np.abs(out["traces"]).max()))


if __name__ == "__main__":
    only = sys.argv[1] if len(sys.argv) > 1 else "all"
    if only in ("all", "cd"):
        for name, args in ENGINE_CASES.items():
            engine_case(name, *args)
        degenerate_case()
        run_case()
        checksum_case()
    if only in ("all", "vd"):
        for name, args in VD_CASES.items():
            vd_case(name, *args)
        vd_run_case()
