"""AcousticCdEngine -- Python mirror of minimod::AcousticCdEngine<float>.

ref: propagator.hpp:93-140 (interface), propagator_impl.hpp:53-173
(implementation).  Every call goes through the C ABI
(include/minimod_b200.h) into the CUDA library; there is no CPU path.

Differences from the C++ reference that callers may notice:
* ``pressure()`` / ``pressure_prev()`` return host copies (the fields live in
  HBM); write back with ``set_state``.
* ``profile()`` returns a copy of the CPML tables; apply edits with
  ``set_profile`` (accepted before the first step, as the reference tests
  use it: test_cpml.cpp:148-153).
* ``runner`` arguments are accepted and ignored (the GPU is the runner).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import MM_MODE_FAST, MM_MODE_FAST_FMA, MM_MODE_STRICT, check, lib
from .numerics import AxisCpml, CpmlProfile, Grid3D, make_grid

_i3 = C.c_int * 3


def _fptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_float))


@dataclass
class EngineOptions:  # ref: propagator.hpp:23-30 (same defaults)
    ndamping: tuple = (0, 0, 0)
    fmax: float = 25.0
    r_target: float = 1e-3
    free_surface: bool = False
    taper: bool = False
    ntaper: tuple = (3, 3, 3)

    def to_c(self) -> _lib.mm_engine_options:
        o = _lib.mm_engine_options()
        o.ndamping[:] = [int(x) for x in self.ndamping]
        o.fmax = float(self.fmax)
        o.r_target = float(self.r_target)
        o.free_surface = int(bool(self.free_surface))
        o.taper = int(bool(self.taper))
        o.ntaper[:] = [int(x) for x in self.ntaper]
        return o


_MODES = {"fast": MM_MODE_FAST, "strict": MM_MODE_STRICT, "fast_fma": MM_MODE_FAST_FMA}


class AcousticCdEngine:
    """Second-order constant-density acoustic propagator with CPML on the GPU."""

    def __init__(self, grid: Grid3D, offset: Sequence[int], global_n: Sequence[int],
                 vp_local: np.ndarray, opts: Optional[EngineOptions] = None,
                 dt: float = 1e-3, vmax_global: Optional[float] = None, *, device: int = 0,
                 mode: str = "fast"):
        opts = opts or EngineOptions()
        self._h = None
        self._grid = grid
        self.offset = tuple(int(x) for x in offset)
        self.global_n = tuple(int(x) for x in global_n)
        vp = np.ascontiguousarray(vp_local, dtype=np.float32)
        if vp.shape != grid.shape:
            raise ValueError(f"vp_local shape {vp.shape} != ghosted grid shape {grid.shape}")
        if vmax_global is None:
            vmax_global = float(grid.inner(vp).max())
        g = _lib.mm_grid()
        g.n[:] = list(grid.n)
        g.d[:] = list(grid.d)
        g.radius = grid.radius
        h = C.c_void_p()
        self.mode = mode
        check(lib().mm_cd_create(C.byref(g), _i3(*self.offset), _i3(*self.global_n), _fptr(vp),
                                 C.byref(opts.to_c()), C.c_float(dt), float(vmax_global),
                                 int(device), _MODES[mode], C.byref(h)))
        self._h = h
        self.device = device
        self.options = opts
        self._nrec = 0
        self._cap = 0

    @classmethod
    def _view(cls, handle, grid: Grid3D, offset, global_n, opts, device, mode):
        """A non-owning wrapper of an engine another object owns (the slab
        engine of a ZSlabGroup)."""
        self = cls.__new__(cls)
        self._h = handle
        self._grid = grid
        self.offset = tuple(int(x) for x in offset)
        self.global_n = tuple(int(x) for x in global_n)
        self.mode = mode
        self.device = device
        self.options = opts
        self._nrec = 0
        self._cap = 0
        self._owned = False
        return self

    # -- lifetime ---------------------------------------------------------
    def close(self):
        if self._h and getattr(self, "_owned", True):
            lib().mm_cd_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    # -- reference interface ---------------------------------------------
    def step(self, source_amplitude: float, src: Optional[Sequence[int]] = None, runner=None):
        """ref: propagator.hpp:103-104."""
        check(lib().mm_cd_step(self._h, C.c_float(source_amplitude),
                               _i3(*src) if src is not None else None))

    def grid(self) -> Grid3D:
        return self._grid

    def dt(self) -> float:
        v = C.c_float()
        check(lib().mm_cd_get_dt(self._h, C.byref(v)))
        return v.value

    def pressure(self) -> np.ndarray:
        out = self._grid.field()
        check(lib().mm_cd_get_pressure(self._h, _fptr(out)))
        return out

    def pressure_prev(self) -> np.ndarray:
        out = self._grid.field()
        check(lib().mm_cd_get_pressure_prev(self._h, _fptr(out)))
        return out

    def velocity(self) -> np.ndarray:
        """The (tapered) vp copy the engine steps with."""
        out = self._grid.field()
        check(lib().mm_cd_get_velocity(self._h, _fptr(out)))
        return out

    def set_state(self, p_prev: np.ndarray, p_cur: np.ndarray):
        """ref: propagator.hpp:116-120."""
        a = np.ascontiguousarray(p_prev, dtype=np.float32)
        b = np.ascontiguousarray(p_cur, dtype=np.float32)
        if a.shape != self._grid.shape or b.shape != self._grid.shape:
            raise ValueError("set_state fields must have the ghosted grid shape")
        check(lib().mm_cd_set_state(self._h, _fptr(a), _fptr(b)))

    def profile(self) -> CpmlProfile:
        """Copy of the CPML tables (ref: propagator.hpp:112-114)."""
        axes = []
        for ax in range(3):
            n = self.global_n[ax]
            a, b, k = (np.zeros(n, np.float32) for _ in range(3))
            check(lib().mm_cd_get_profile(self._h, ax, _fptr(a), _fptr(b), _fptr(k)))
            axes.append(AxisCpml(a, b, k))
        d0 = (C.c_double * 3)()
        check(lib().mm_cd_get_d0(self._h, d0))
        return CpmlProfile(axes, tuple(self.options.ndamping), tuple(d0))

    def set_profile(self, prof: CpmlProfile):
        for ax in range(3):
            A = prof.axis[ax]
            a = np.ascontiguousarray(A.a, np.float32)
            b = np.ascontiguousarray(A.b, np.float32)
            k = np.ascontiguousarray(A.inv_kappa, np.float32)
            check(lib().mm_cd_set_profile(self._h, ax, _fptr(a), _fptr(b), _fptr(k)))

    # -- sub-phases (ref: propagator_impl.hpp:154-173) --------------------
    def update_boundary_psi(self):
        check(lib().mm_cd_update_boundary_psi(self._h))

    def update_inner(self):
        check(lib().mm_cd_update_inner(self._h))

    def update_boundary(self):
        check(lib().mm_cd_update_boundary(self._h))

    def update_planes(self, z_lo: int, z_hi: int):
        check(lib().mm_cd_update_planes(self._h, int(z_lo), int(z_hi)))

    def update_plane_ranges(self, ranges):
        """p_next on the union of plane ranges [(z_lo, z_hi), ...] in one launch per
        kernel (the z-slab schedule's edge planes)."""
        flat = [int(v) for r in ranges for v in r]
        arr = (C.c_int * max(1, len(flat)))(*flat)
        check(lib().mm_cd_update_plane_ranges(self._h, arr, len(flat) // 2))

    def inject_source(self, amp: float, src: Optional[Sequence[int]]):
        check(lib().mm_cd_inject_source(self._h, C.c_float(amp),
                                        _i3(*src) if src is not None else None))

    def apply_free_surface(self):
        check(lib().mm_cd_apply_free_surface(self._h))

    def rotate(self):
        check(lib().mm_cd_rotate(self._h))

    def synchronize(self):
        check(lib().mm_cd_synchronize(self._h))

    def steps_taken(self) -> int:
        v = C.c_longlong()
        check(lib().mm_cd_steps_taken(self._h, C.byref(v)))
        return v.value

    # -- receivers / device loop -----------------------------------------
    def set_receivers(self, ijk: np.ndarray, capacity: int):
        ijk = np.ascontiguousarray(ijk, dtype=np.int32).reshape(-1, 3)
        check(lib().mm_cd_set_receivers(self._h, ijk.ctypes.data_as(C.POINTER(C.c_int)),
                                        ijk.shape[0], int(capacity)))
        self._nrec, self._cap = ijk.shape[0], int(capacity)

    def record(self, step: int):
        check(lib().mm_cd_record(self._h, int(step)))

    def traces(self, nsteps: Optional[int] = None) -> np.ndarray:
        nsteps = self._cap if nsteps is None else nsteps
        out = np.zeros((self._nrec, nsteps), np.float32)
        check(lib().mm_cd_get_traces(self._h, _fptr(out), int(nsteps)))
        return out

    def copy_trace_step(self, step: int, out: np.ndarray, asynchronous: bool = False):
        """Receiver samples of one recorded step into `out` (nreceivers float32)."""
        assert out.dtype == np.float32 and out.size >= self._nrec
        check(lib().mm_cd_copy_trace_step(self._h, int(step), _fptr(out), int(asynchronous)))

    def run(self, amps: np.ndarray, src: Optional[Sequence[int]] = None, record: bool = True,
            first_sample: int = 0) -> float:
        """Device-resident loop over len(amps) steps; returns device milliseconds."""
        amps = np.ascontiguousarray(amps, dtype=np.float32)
        ms = C.c_float()
        check(lib().mm_cd_run(self._h, _fptr(amps), amps.size,
                              _i3(*src) if src is not None else None, int(record),
                              int(first_sample), C.byref(ms)))
        return ms.value

    def cpml_path(self) -> str:
        """Kernels of a full step's damping-slab update: "cpml" (fused one-pass),
        "two-pass" or "strict"."""
        buf = C.create_string_buffer(32)
        check(lib().mm_cd_cpml_path(self._h, buf, 32))
        return buf.value.decode()

    # -- per-kernel timing (bench evidence) ------------------------------
    def kernel_timing(self, on: bool = True):
        """Bracket every kernel of the following steps with CUDA events on its
        own stream (steps issue eagerly while on); clears the totals."""
        check(lib().mm_cd_kernel_timing(self._h, int(bool(on))))

    def kernel_times(self) -> dict:
        """{kernel name: (total ms, launches)} since kernel_timing(True)."""
        n = C.c_int()
        check(lib().mm_cd_kernel_times(self._h, 0, None, None, None, C.byref(n)))
        k = n.value
        names = (C.c_char * 32 * max(k, 1))()
        ms = (C.c_double * max(k, 1))()
        cnt = (C.c_longlong * max(k, 1))()
        check(lib().mm_cd_kernel_times(self._h, k, C.cast(names, C.c_void_p), ms, cnt,
                                       C.byref(n)))
        return {names[i].value.decode(): (ms[i], cnt[i]) for i in range(k)}

    # -- multi-GPU plumbing ----------------------------------------------
    def stream_handle(self) -> int:
        s = C.c_void_p()
        check(lib().mm_cd_stream(self._h, C.byref(s)))
        return s.value or 0

    def halo_planes(self, side: int, which: int, next_field: bool = False):
        """(device pointer, bytes) of the r contiguous z-planes (see the C ABI)."""
        p = C.c_void_p()
        n = C.c_size_t()
        fn = lib().mm_cd_next_halo_planes if next_field else lib().mm_cd_halo_planes
        check(fn(self._h, int(side), int(which), C.byref(p), C.byref(n)))
        return p.value, n.value


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (mm_nccl_get_unique_id), made by rank 0 and
    shared with the other ranks by the host runtime."""
    buf = (C.c_ubyte * 128)()
    check(lib().mm_nccl_get_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def validate_cuts_native(cuts, nz: int, nd_z: int, radius: int) -> None:
    """mm_zslab_validate_cuts (ref: dist.cpp:119-132)."""
    arr = (C.c_int * len(cuts))(*cuts)
    check(lib().mm_zslab_validate_cuts(arr, len(cuts) - 1, int(nz), int(nd_z), int(radius)))


class ZSlabGroup:
    """One rank of the multi-GPU z-slab run (mm_cd_group_*, group.cu): its slab
    engine and NCCL halo exchange, driven from C++.

    ref: run_distributed_rank (dist.cpp:144-267) with dims {1, 1, P}."""

    def __init__(self, grid: Grid3D, cuts, rank: int, vp_global: Optional[np.ndarray],
                 opts: Optional[EngineOptions], dt: float, vmax: float, *,
                 nccl_id: Optional[bytes] = None, device: int = 0, mode: str = "fast",
                 vp_local: Optional[np.ndarray] = None):
        opts = opts or EngineOptions()
        world = len(cuts) - 1
        r = grid.radius
        z0, z1 = int(cuts[rank]), int(cuts[rank + 1])
        # the rank's ghosted slice of the ghosted global model (dist.cpp:171-180)
        if vp_local is None:
            vp_local = vp_global[:, :, z0:z1 + 2 * r]
        vp_loc = np.ascontiguousarray(vp_local, dtype=np.float32)
        if vp_loc.shape != (grid.shape[0], grid.shape[1], z1 - z0 + 2 * r):
            raise ValueError("vp_local must be the rank's ghosted slab")
        g = _lib.mm_grid()
        g.n[:] = list(grid.n)
        g.d[:] = list(grid.d)
        g.radius = r
        arr = (C.c_int * len(cuts))(*[int(c) for c in cuts])
        idb = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be 128 bytes")
            idb = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
        h = C.c_void_p()
        self._h = None
        check(lib().mm_cd_group_create(C.byref(g), arr, world, int(rank),
                                       C.cast(idb, C.c_void_p) if idb is not None else None,
                                       _fptr(vp_loc), C.byref(opts.to_c()), C.c_float(dt),
                                       float(vmax), int(device), _MODES[mode], C.byref(h)))
        self._h = h
        self.rank, self.world, self.cuts = rank, world, list(cuts)
        self.z0, self.nz = z0, z1 - z0
        eh = C.c_void_p()
        check(lib().mm_cd_group_engine(self._h, C.byref(eh)))
        lgrid = Grid3D((grid.n[0], grid.n[1], self.nz), grid.d, r)
        self.engine = AcousticCdEngine._view(eh, lgrid, (0, 0, z0), grid.n, opts, device, mode)

    def close(self):
        if self._h:
            self.engine._h = None
            lib().mm_cd_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, amp: float, src_global: Optional[Sequence[int]] = None):
        check(lib().mm_cd_group_step(self._h, C.c_float(amp),
                                     _i3(*src_global) if src_global is not None else None))

    def run(self, amps: np.ndarray, src_global: Optional[Sequence[int]] = None,
            record: bool = True, first_sample: int = 0) -> float:
        amps = np.ascontiguousarray(amps, dtype=np.float32)
        ms = C.c_float()
        check(lib().mm_cd_group_run(self._h, _fptr(amps), amps.size,
                                    _i3(*src_global) if src_global is not None else None,
                                    int(record), int(first_sample), C.byref(ms)))
        return ms.value


def step_local(groups, amp: float, src_global: Optional[Sequence[int]] = None):
    """One step of in-process ranks (ZSlabGroup made without an NCCL id) on one
    device: mm_cd_group_step_local (test hook; device-to-device halo copies)."""
    arr = (C.c_void_p * len(groups))(*[g._h for g in groups])
    check(lib().mm_cd_group_step_local(arr, len(groups), C.c_float(amp),
                                       _i3(*src_global) if src_global is not None else None))


class AcousticVdEngine:
    """Variable-density first-order acoustic propagator with CPML on the GPU.

    ref: propagator.hpp:147-176 (interface), propagator_impl.hpp:175-295;
    SURVEY.md §8(f) row 4.  ``model`` must carry a density volume (rho), as
    the reference requires (propagator_impl.hpp:186-187).  ``step`` takes the
    time-integrated wavelet sample (numerics.integrate_wavelet).
    """

    def __init__(self, grid: Grid3D, model, opts: Optional[EngineOptions] = None,
                 dt: float = 1e-3, *, device: int = 0):
        opts = opts or EngineOptions()
        self._h = None
        self._grid = grid
        vp = np.ascontiguousarray(model.vp, dtype=np.float32)
        rho = None if model.rho is None else np.ascontiguousarray(model.rho, dtype=np.float32)
        if vp.shape != grid.shape or (rho is not None and rho.shape != grid.shape):
            raise ValueError("model volumes must have the ghosted grid shape")
        vmax = model.vmax if model.vmax else float(grid.inner(vp).max())
        g = _lib.mm_grid()
        g.n[:] = list(grid.n)
        g.d[:] = list(grid.d)
        g.radius = grid.radius
        h = C.c_void_p()
        check(lib().mm_vd_create(C.byref(g), _fptr(vp), _fptr(rho) if rho is not None else None,
                                 C.byref(opts.to_c()), C.c_float(dt), float(vmax), int(device),
                                 C.byref(h)))
        self._h = h
        self.device = device
        self.options = opts
        self._nrec = 0
        self._cap = 0

    def close(self):
        if self._h:
            lib().mm_vd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    # -- reference interface ---------------------------------------------
    def step(self, source_amplitude: float, src: Optional[Sequence[int]] = None, runner=None):
        """ref: propagator.hpp:154-155."""
        check(lib().mm_vd_step(self._h, C.c_float(source_amplitude),
                               _i3(*src) if src is not None else None))

    def grid(self) -> Grid3D:
        return self._grid

    def dt(self) -> float:
        v = C.c_float()
        check(lib().mm_vd_get_dt(self._h, C.byref(v)))
        return v.value

    def pressure(self) -> np.ndarray:
        """ref: propagator.hpp:157 (a copy; see set_pressure)."""
        out = self._grid.field()
        check(lib().mm_vd_get_pressure(self._h, _fptr(out)))
        return out

    def velocity(self, axis: int) -> np.ndarray:
        """ref: propagator.hpp:158 (a copy; see set_velocity)."""
        out = self._grid.field()
        check(lib().mm_vd_get_velocity(self._h, int(axis), _fptr(out)))
        return out

    def set_pressure(self, p: np.ndarray):
        a = np.ascontiguousarray(p, dtype=np.float32)
        if a.shape != self._grid.shape:
            raise ValueError("pressure must have the ghosted grid shape")
        check(lib().mm_vd_set_pressure(self._h, _fptr(a)))

    def set_velocity(self, axis: int, v: np.ndarray):
        a = np.ascontiguousarray(v, dtype=np.float32)
        if a.shape != self._grid.shape:
            raise ValueError("velocity must have the ghosted grid shape")
        check(lib().mm_vd_set_velocity(self._h, int(axis), _fptr(a)))

    # -- sub-phases (ref: propagator_impl.hpp:275-295) --------------------
    def update_velocity(self):
        check(lib().mm_vd_update_velocity(self._h))

    def update_pressure(self):
        check(lib().mm_vd_update_pressure(self._h))

    def inject_source(self, amp: float, src: Sequence[int]):
        check(lib().mm_vd_inject_source(self._h, C.c_float(amp), _i3(*src)))

    def apply_free_surface(self):
        check(lib().mm_vd_apply_free_surface(self._h))

    def synchronize(self):
        check(lib().mm_vd_synchronize(self._h))

    def steps_taken(self) -> int:
        v = C.c_longlong()
        check(lib().mm_vd_steps_taken(self._h, C.byref(v)))
        return v.value

    # -- receivers / device loop -----------------------------------------
    def set_receivers(self, ijk: np.ndarray, capacity: int):
        ijk = np.ascontiguousarray(ijk, dtype=np.int32).reshape(-1, 3)
        check(lib().mm_vd_set_receivers(self._h, ijk.ctypes.data_as(C.POINTER(C.c_int)),
                                        ijk.shape[0], int(capacity)))
        self._nrec, self._cap = ijk.shape[0], int(capacity)

    def record(self, step: int):
        check(lib().mm_vd_record(self._h, int(step)))

    def traces(self, nsteps: Optional[int] = None) -> np.ndarray:
        nsteps = self._cap if nsteps is None else nsteps
        out = np.zeros((self._nrec, nsteps), np.float32)
        check(lib().mm_vd_get_traces(self._h, _fptr(out), int(nsteps)))
        return out

    def copy_trace_step(self, step: int, out: np.ndarray, asynchronous: bool = False):
        assert out.dtype == np.float32 and out.size >= self._nrec
        check(lib().mm_vd_copy_trace_step(self._h, int(step), _fptr(out), int(asynchronous)))

    def run(self, amps: np.ndarray, src: Optional[Sequence[int]] = None, record: bool = True,
            first_sample: int = 0) -> float:
        """Device-resident loop over len(amps) steps; returns device milliseconds."""
        amps = np.ascontiguousarray(amps, dtype=np.float32)
        ms = C.c_float()
        check(lib().mm_vd_run(self._h, _fptr(amps), amps.size,
                              _i3(*src) if src is not None else None, int(record),
                              int(first_sample), C.byref(ms)))
        return ms.value

    def stream_handle(self) -> int:
        s = C.c_void_p()
        check(lib().mm_vd_stream(self._h, C.byref(s)))
        return s.value or 0
