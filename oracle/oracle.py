"""ctypes front-end for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two back ends with the same Python surface:

* ``Oracle("port")`` -- ``oracle/libminimod_oracle.so``, the plain-C
  restatement in ``oracle/minimod_oracle.c`` (travels to the GPU box).
* ``Oracle("reference")`` -- ``oracle/_ref/libminimod_ref.so``, the
  reference's own sources compiled by ``oracle/build_ref.sh`` (built in the
  authoring container where /root/reference exists; the built .so travels).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  The product package never does.

Fields use the reference layout: ghosted, z fastest, numpy shape
``(nx+2r, ny+2r, nz+2r)`` (ref: grid.hpp:61-65).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "libminimod_oracle.so"
REF_LIB = HERE / "_ref" / "libminimod_ref.so"

_i3 = C.c_int * 3
_d3 = C.c_double * 3
_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)


def _f32(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_fp)


def ghosted_shape(n, r):
    return tuple(int(x) + 2 * r for x in n)


def available(kind: str = "port") -> bool:
    return (PORT_LIB if kind == "port" else REF_LIB).exists()


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not path.exists():
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        self.lib = C.CDLL(str(path))
        p = "mo_" if kind == "port" else "ref_"
        self.p = p
        L = self.lib
        self._err = getattr(L, p + "last_error")
        self._err.restype = C.c_char_p
        for name in ("engine_pressure", "engine_pressure_prev"):
            f = getattr(L, p + name)
            f.restype = _fp
            f.argtypes = [C.c_void_p]
        f = getattr(L, p + "engine_profile")
        f.restype = _fp
        f.argtypes = [C.c_void_p, C.c_int, C.c_int]
        f = getattr(L, p + "engine_d0")
        f.restype = C.c_double
        f.argtypes = [C.c_void_p, C.c_int]
        getattr(L, p + "engine_destroy").argtypes = [C.c_void_p]
        getattr(L, p + "engine_step").argtypes = [C.c_void_p, C.c_float, C.c_void_p]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err().decode())

    # ---- setup helpers --------------------------------------------------
    def second_derivative_coeffs(self, radius, h):
        c = (C.c_double * 8)()
        center = C.c_double()
        self._check(getattr(self.lib, self.p + "second_derivative_coeffs")(
            C.c_int(radius), C.c_double(h), c, C.byref(center)))
        return np.array(c[:radius]), center.value

    def central_first_derivative_coeffs(self, radius, h):
        c = (C.c_double * 8)()
        self._check(getattr(self.lib, self.p + "central_first_derivative_coeffs")(
            C.c_int(radius), C.c_double(h), c))
        return np.array(c[:radius])

    def ricker(self, fmax, dt, nsteps):
        out = np.zeros(nsteps, np.float32)
        self._check(getattr(self.lib, self.p + "ricker")(
            C.c_double(fmax), C.c_double(dt), C.c_int(nsteps), _f32(out)))
        return out

    def layered_model(self, n, r=4, d=(20.0, 20.0, 20.0)):
        vp = np.zeros(ghosted_shape(n, r), np.float32)
        vmin, vmax = C.c_float(), C.c_float()
        if self.kind == "port":
            self.lib.mo_layered_model(_i3(*n), C.c_int(r), _f32(vp), C.byref(vmin), C.byref(vmax))
        else:
            self._check(self.lib.ref_layered_model(_i3(*n), _d3(*d), C.c_int(r), _f32(vp),
                                                   C.byref(vmin), C.byref(vmax)))
        return vp, vmin.value, vmax.value

    def cfl_dt(self, vmax, radius, d, cfl):
        dt = C.c_double()
        if self.kind != "port":
            raise NotImplementedError("use cfl_dt_model on the reference back end")
        self._check(self.lib.mo_cfl_dt(C.c_double(vmax), C.c_int(radius), _d3(*d),
                                       C.c_double(cfl), C.byref(dt)))
        return dt.value

    def taper_material(self, vp, n, r, ntaper, offset=(0, 0, 0), global_n=None):
        f = np.ascontiguousarray(vp, dtype=np.float32).copy()
        gn = n if global_n is None else global_n
        if self.kind == "port":
            self.lib.mo_taper_material(_f32(f), _i3(*n), C.c_int(r), _i3(*ntaper), _i3(*offset),
                                       _i3(*gn))
        else:
            self._check(self.lib.ref_taper_material(_f32(f), _i3(*n), C.c_int(r), _i3(*ntaper),
                                                    _i3(*offset), _i3(*gn)))
        return f

    def fill_ghosts_replicate(self, f, n, r):
        f = np.ascontiguousarray(f, dtype=np.float32).copy()
        if self.kind != "port":
            raise NotImplementedError
        self.lib.mo_fill_ghosts_replicate(_f32(f), _i3(*n), C.c_int(r))
        return f

    # ---- driver ---------------------------------------------------------
    def run(self, n, vp, *, d=(20.0, 20.0, 20.0), radius=4, nsteps=100, fmax=25.0, cfl=0.8,
            ndamping=(27, 27, 27), ntaper=(3, 3, 3), taper=True, free_surface=False,
            r_target=1e-3, src=None, vmax=None, nthreads=1, want_field=False):
        """minimod::run() for acoustic_iso_cd (ref: driver.cpp:83-144).

        Returns dict(traces [nrec x nsteps], dt, kernel_seconds[, p])."""
        n = tuple(int(x) for x in n)
        vp = np.ascontiguousarray(vp, dtype=np.float32)
        nrec = n[0] * n[1]
        traces = np.zeros((nrec, nsteps), np.float32)
        dt = C.c_double()
        ks = C.c_double()
        srcp = _i3(*src) if src is not None else None
        if self.kind == "port":
            if vmax is None:
                vmax = float(vp[radius:radius + n[0], radius:radius + n[1],
                                radius:radius + n[2]].max())
            p = np.zeros(ghosted_shape(n, radius), np.float32) if want_field else None
            self._check(self.lib.mo_run(
                _i3(*n), _d3(*d), C.c_int(radius), C.c_int(nsteps), C.c_double(fmax),
                C.c_double(cfl), _i3(*ndamping), _i3(*ntaper), C.c_int(int(taper)),
                C.c_int(int(free_surface)), C.c_double(r_target), srcp, _f32(vp),
                C.c_float(vmax), _f32(traces), _f32(p) if p is not None else None,
                C.byref(dt), C.byref(ks)))
            out = dict(traces=traces, dt=dt.value, kernel_seconds=ks.value)
            if want_field:
                out["p"] = p
            return out
        ms = C.c_double()
        self._check(self.lib.ref_run(
            _i3(*n), _d3(*d), C.c_int(radius), C.c_int(nsteps), C.c_double(fmax),
            C.c_double(cfl), _i3(*ndamping), _i3(*ntaper), C.c_int(int(taper)),
            C.c_int(int(free_surface)), C.c_double(r_target), srcp, _f32(vp),
            C.c_int(nthreads), _f32(traces), C.byref(dt), C.byref(ks), C.byref(ms)))
        return dict(traces=traces, dt=dt.value, kernel_seconds=ks.value,
                    modeling_seconds=ms.value)

    # ---- acoustic_iso (variable density) --------------------------------
    def staggered_first_derivative_coeffs(self, radius, h):
        c = (C.c_double * 8)()
        self._check(getattr(self.lib, self.p + "staggered_first_derivative_coeffs")(
            C.c_int(radius), C.c_double(h), c))
        return np.array(c[:radius])

    def integrate_wavelet(self, w, dt):
        w = np.ascontiguousarray(w, dtype=np.float32)
        out = np.zeros_like(w)
        fn = getattr(self.lib, self.p + "integrate_wavelet")
        rc = fn(_f32(w), C.c_int(w.size), C.c_double(dt), _f32(out))
        if self.kind != "port":
            self._check(rc)
        return out

    def vd_engine(self, n, vp, rho, *, d=(20.0, 20.0, 20.0), radius=4, ndamping=(0, 0, 0),
                  fmax=25.0, r_target=1e-3, free_surface=False, taper=False, ntaper=(3, 3, 3),
                  dt=1e-3, vmax=None, nthreads=1):
        return OracleVdEngine(self, n, vp, rho, d=d, radius=radius, ndamping=ndamping,
                              fmax=fmax, r_target=r_target, free_surface=free_surface,
                              taper=taper, ntaper=ntaper, dt=dt, vmax=vmax, nthreads=nthreads)

    def run_vd(self, n, vp, rho, *, d=(20.0, 20.0, 20.0), radius=4, nsteps=100, fmax=25.0,
               cfl=0.8, ndamping=(27, 27, 27), ntaper=(3, 3, 3), taper=True,
               free_surface=False, r_target=1e-3, src=None, vmax=None, nthreads=1):
        """minimod::run() for acoustic_iso (ref: driver.cpp:83-144, :122-128)."""
        n = tuple(int(x) for x in n)
        vp = np.ascontiguousarray(vp, dtype=np.float32)
        rho = np.ascontiguousarray(rho, dtype=np.float32)
        traces = np.zeros((n[0] * n[1], nsteps), np.float32)
        dt, ks = C.c_double(), C.c_double()
        srcp = _i3(*src) if src is not None else None
        common = (_i3(*n), _d3(*d), C.c_int(radius), C.c_int(nsteps), C.c_double(fmax),
                  C.c_double(cfl), _i3(*ndamping), _i3(*ntaper), C.c_int(int(taper)),
                  C.c_int(int(free_surface)), C.c_double(r_target), srcp, _f32(vp), _f32(rho))
        if self.kind == "port":
            if vmax is None:
                r = radius
                vmax = float(vp[r:r + n[0], r:r + n[1], r:r + n[2]].max())
            self._check(self.lib.mo_run_vd(*common, C.c_float(vmax), _f32(traces), C.byref(dt),
                                           C.byref(ks)))
            return dict(traces=traces, dt=dt.value, kernel_seconds=ks.value)
        ms = C.c_double()
        self._check(self.lib.ref_run_vd(*common, C.c_int(nthreads), _f32(traces), C.byref(dt),
                                        C.byref(ks), C.byref(ms)))
        return dict(traces=traces, dt=dt.value, kernel_seconds=ks.value,
                    modeling_seconds=ms.value)

    # ---- on-disk formats and report (reference back end only) -----------
    def _ref_only(self):
        if self.kind != "reference":
            raise NotImplementedError("the reference back end writes the reference formats")

    def save_record(self, traces, dt, path, *, source_loc=(0, 0, 0), receiver_increment=(1, 1),
                    nshots=1):
        """save_record (source.cpp:68-95): traces [nreceivers x nsteps]."""
        self._ref_only()
        t = np.ascontiguousarray(traces, dtype=np.float32)
        self._check(self.lib.ref_save_record(
            _f32(t), C.c_int(t.shape[0]), C.c_int(t.shape[1]), C.c_double(dt), _i3(*source_loc),
            (C.c_int * 2)(*receiver_increment), C.c_int(nshots), str(path).encode()))

    def save_model(self, vp, n, d, radius, manifest):
        """save_model (model.cpp:160-190) of a ghosted vp field."""
        self._ref_only()
        v = np.ascontiguousarray(vp, dtype=np.float32)
        self._check(self.lib.ref_save_model(_i3(*n), _d3(*d), C.c_int(radius), _f32(v),
                                            str(manifest).encode()))

    def load_model(self, manifest, radius=4):
        """load_model (model.cpp:64-99): (n, d, ghosted vp of radius 4, vmin, vmax)."""
        self._ref_only()
        n, d = _i3(), _d3()
        vmin, vmax = C.c_float(), C.c_float()
        self._check(self.lib.ref_load_model(str(manifest).encode(), n, d, None, C.byref(vmin),
                                            C.byref(vmax)))
        vp = np.zeros(ghosted_shape(tuple(n), radius), np.float32)
        self._check(self.lib.ref_load_model(str(manifest).encode(), n, d, _f32(vp),
                                            C.byref(vmin), C.byref(vmax)))
        return tuple(n), tuple(d), vp, vmin.value, vmax.value

    def save_model_rho(self, vp, rho, n, d, radius, manifest):
        """save_model (model.cpp:157-184) of a model with a density volume."""
        self._ref_only()
        v = np.ascontiguousarray(vp, dtype=np.float32)
        r = np.ascontiguousarray(rho, dtype=np.float32)
        self._check(self.lib.ref_save_model_rho(_i3(*n), _d3(*d), C.c_int(radius), _f32(v),
                                                _f32(r), str(manifest).encode()))

    def load_model_rho(self, manifest, n, radius=4):
        """rho of load_model (model.cpp:122-155), or None."""
        self._ref_only()
        rho = np.zeros(ghosted_shape(tuple(n), radius), np.float32)
        has = C.c_int()
        self._check(self.lib.ref_load_model_rho(str(manifest).encode(), _f32(rho), C.byref(has)))
        return rho if has.value else None

    def render_report(self, *, ngrid, dgrid, nsteps, fmax, cfl, radius, ndamping, ntaper,
                      source_loc, receiver_increment, source_increment, nshots, time_rec,
                      nthreads, vmin, vmax, kernel_s, modeling_s):
        """render_parameter_block + render_timing (driver.cpp:150-215)."""
        self._ref_only()
        buf = C.create_string_buffer(1 << 14)
        self.lib.ref_render_report.argtypes = None
        self._check(self.lib.ref_render_report(
            _i3(*ngrid), _d3(*dgrid), C.c_int(nsteps), C.c_double(fmax), C.c_double(cfl),
            C.c_int(radius), _i3(*ndamping), _i3(*ntaper),
            _i3(*source_loc) if source_loc is not None else None,
            (C.c_int * 2)(*receiver_increment), _i3(*source_increment), C.c_int(nshots),
            C.c_double(time_rec), C.c_int(nthreads), C.c_float(vmin), C.c_float(vmax),
            C.c_double(kernel_s), C.c_double(modeling_s), buf, C.c_int(len(buf))))
        return buf.value.decode()

    # ---- engine ---------------------------------------------------------
    def engine(self, n_local, vp_local, *, d=(20.0, 20.0, 20.0), radius=4, offset=(0, 0, 0),
               global_n=None, ndamping=(0, 0, 0), fmax=25.0, r_target=1e-3,
               free_surface=False, taper=False, ntaper=(3, 3, 3), dt=1e-3, vmax=None,
               nthreads=1):
        return OracleEngine(self, n_local, vp_local, d=d, radius=radius, offset=offset,
                            global_n=global_n, ndamping=ndamping, fmax=fmax, r_target=r_target,
                            free_surface=free_surface, taper=taper, ntaper=ntaper, dt=dt,
                            vmax=vmax, nthreads=nthreads)


class OracleEngine:
    """AcousticCdEngine<float> (ref: propagator.hpp:93-140) on the CPU."""

    def __init__(self, o: Oracle, n_local, vp_local, *, d, radius, offset, global_n, ndamping,
                 fmax, r_target, free_surface, taper, ntaper, dt, vmax, nthreads):
        self.o = o
        self.n = tuple(int(x) for x in n_local)
        self.r = radius
        self.global_n = tuple(global_n) if global_n is not None else self.n
        vp_local = np.ascontiguousarray(vp_local, dtype=np.float32)
        assert vp_local.shape == ghosted_shape(self.n, radius), vp_local.shape
        if vmax is None:
            r = radius
            vmax = float(vp_local[r:-r, r:-r, r:-r].max())
        h = C.c_void_p()
        args = [_i3(*self.n), _d3(*d), C.c_int(radius), _i3(*offset), _i3(*self.global_n),
                _f32(vp_local), _i3(*ndamping), C.c_double(fmax), C.c_double(r_target),
                C.c_int(int(free_surface)), C.c_int(int(taper)), _i3(*ntaper), C.c_float(dt),
                C.c_double(vmax)]
        if o.kind == "port":
            o._check(o.lib.mo_engine_create(*args, C.byref(h)))
        else:
            o._check(o.lib.ref_engine_create(*args, C.c_int(nthreads), C.byref(h)))
        self.h = h
        self.shape = ghosted_shape(self.n, radius)
        self.size = int(np.prod(self.shape))

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            getattr(self.o.lib, self.o.p + "engine_destroy")(h)
            self.h = None

    def step(self, amp, src=None):
        srcp = _i3(*src) if src is not None else None
        self.o._check(getattr(self.o.lib, self.o.p + "engine_step")(self.h, C.c_float(amp),
                                                                    srcp))

    def _view(self, ptr):
        return np.ctypeslib.as_array(ptr, shape=(self.size,)).reshape(self.shape)

    def pressure(self):
        return self._view(getattr(self.o.lib, self.o.p + "engine_pressure")(self.h)).copy()

    def pressure_prev(self):
        return self._view(getattr(self.o.lib, self.o.p + "engine_pressure_prev")(self.h)).copy()

    def profile_array(self, which, axis):
        """Mutable view of a CPML table (which 0=a, 1=b, 2=inv_kappa)."""
        ptr = getattr(self.o.lib, self.o.p + "engine_profile")(self.h, which, axis)
        return np.ctypeslib.as_array(ptr, shape=(self.global_n[axis],))

    def d0(self, axis):
        return getattr(self.o.lib, self.o.p + "engine_d0")(self.h, axis)

    def set_state(self, p_prev, p_cur):
        a = np.ascontiguousarray(p_prev, dtype=np.float32)
        b = np.ascontiguousarray(p_cur, dtype=np.float32)
        fn = getattr(self.o.lib, self.o.p + "engine_set_state")
        rc = fn(self.h, _f32(a), _f32(b))
        if self.o.kind != "port":
            self.o._check(rc)


class OracleVdEngine:
    """AcousticVdEngine<float> (ref: propagator.hpp:147-176) on the CPU."""

    def __init__(self, o: Oracle, n, vp, rho, *, d, radius, ndamping, fmax, r_target,
                 free_surface, taper, ntaper, dt, vmax, nthreads):
        self.o = o
        self.n = tuple(int(x) for x in n)
        self.r = radius
        vp = np.ascontiguousarray(vp, dtype=np.float32)
        rho = None if rho is None else np.ascontiguousarray(rho, dtype=np.float32)
        self.shape = ghosted_shape(self.n, radius)
        self.size = int(np.prod(self.shape))
        h = C.c_void_p()
        common = [_i3(*self.n), _d3(*d), C.c_int(radius), _f32(vp),
                  _f32(rho) if rho is not None else None, _i3(*ndamping), C.c_double(fmax),
                  C.c_double(r_target), C.c_int(int(free_surface)), C.c_int(int(taper)),
                  _i3(*ntaper), C.c_float(dt)]
        if o.kind == "port":
            if vmax is None:
                r = radius
                vmax = float(vp[r:-r, r:-r, r:-r].max())
            o._check(o.lib.mo_vd_create(*common, C.c_float(vmax), C.byref(h)))
        else:
            o._check(o.lib.ref_vd_create(*common, C.c_int(nthreads), C.byref(h)))
        self.h = h
        for name in ("vd_pressure",):
            getattr(o.lib, o.p + name).restype = _fp
        getattr(o.lib, o.p + "vd_velocity").restype = _fp
        getattr(o.lib, o.p + "vd_destroy").argtypes = [C.c_void_p]
        getattr(o.lib, o.p + "vd_step").argtypes = [C.c_void_p, C.c_float, C.c_void_p]

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            getattr(self.o.lib, self.o.p + "vd_destroy")(h)
            self.h = None

    def step(self, amp, src=None):
        srcp = _i3(*src) if src is not None else None
        self.o._check(getattr(self.o.lib, self.o.p + "vd_step")(self.h, C.c_float(amp), srcp))

    def _view(self, ptr):
        return np.ctypeslib.as_array(ptr, shape=(self.size,)).reshape(self.shape)

    def pressure_view(self):
        """Mutable view (the reference's pressure() returns a reference)."""
        fn = getattr(self.o.lib, self.o.p + "vd_pressure")
        fn.argtypes = [C.c_void_p]
        return self._view(fn(self.h))

    def pressure(self):
        return self.pressure_view().copy()

    def velocity(self, axis):
        fn = getattr(self.o.lib, self.o.p + "vd_velocity")
        fn.argtypes = [C.c_void_p, C.c_int]
        return self._view(fn(self.h, axis)).copy()


def nproc() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1
