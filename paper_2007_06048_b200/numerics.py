"""Grid, stencil, CPML, model and source helpers (host side, through the C ABI).

Python mirror of the reference's setup layer; every number is computed by the
C++ library (``csrc/host_numerics.cpp``), bit-identical to the reference:

* ``Grid3D`` / ``make_grid`` / ``partition_regions``  -- ref: grid.hpp, grid.cpp
* ``second_derivative_coeffs`` / ``central_first_derivative_coeffs`` /
  ``staggered_first_derivative_coeffs``               -- ref: stencil.cpp
* ``build_profile``                                    -- ref: cpml.hpp:34-72
* ``taper_material`` / ``fill_ghosts_replicate``       -- ref: propagator.hpp:36-62, grid.hpp:96-108
* ``EarthModel`` / ``default_layered_model`` / ``constant_model`` / ``validate_model``
                                                       -- ref: model.hpp, model.cpp
* ``ricker`` / ``integrate_wavelet`` / ``default_receivers`` / ``ShotRecord``
                                                       -- ref: source.hpp, source.cpp

Fields are numpy float32 arrays in the reference layout: ghosted, z fastest,
shape ``(nx+2r, ny+2r, nz+2r)`` (ref: grid.hpp:61-65).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import ConfigError, ValidationError, check, lib

_i3 = C.c_int * 3
_d3 = C.c_double * 3


def _fptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_float))


# ---------------------------------------------------------------------- grid
@dataclass(frozen=True)
class IndexBox:
    """Half-open box [lo, hi) in interior coordinates (ref: grid.hpp:13-33)."""

    lo: tuple = (0, 0, 0)
    hi: tuple = (0, 0, 0)

    def empty(self) -> bool:
        return any(h <= l for l, h in zip(self.lo, self.hi))

    def volume(self) -> int:
        if self.empty():
            return 0
        return int(np.prod([h - l for l, h in zip(self.lo, self.hi)]))

    def contains(self, i, j, k) -> bool:
        p = (i, j, k)
        return all(l <= x < h for l, x, h in zip(self.lo, p, self.hi))


def intersect(a: IndexBox, b: IndexBox) -> IndexBox:  # ref: grid.hpp:35-43
    lo = tuple(max(x, y) for x, y in zip(a.lo, b.lo))
    hi = tuple(min(x, y) for x, y in zip(a.hi, b.hi))
    r = IndexBox(lo, hi)
    return IndexBox() if r.empty() else r


@dataclass(frozen=True)
class Grid3D:
    """ref: grid.hpp:49-73 (z fastest, ghost width = radius)."""

    n: tuple
    d: tuple
    radius: int = 4

    def ext(self, axis: int) -> int:
        return self.n[axis] + 2 * self.radius

    @property
    def shape(self) -> tuple:
        return tuple(self.ext(a) for a in range(3))

    def volume(self) -> int:
        return int(np.prod(self.shape))

    def interior(self) -> IndexBox:
        return IndexBox((0, 0, 0), tuple(self.n))

    def offset(self, i, j, k) -> int:
        r = self.radius
        return ((i + r) * self.ext(1) + (j + r)) * self.ext(2) + (k + r)

    def field(self, value: float = 0.0) -> np.ndarray:
        return np.full(self.shape, value, dtype=np.float32)

    def inner(self, f: np.ndarray) -> np.ndarray:
        """View of the interior of a ghosted field."""
        r = self.radius
        return f[r:r + self.n[0], r:r + self.n[1], r:r + self.n[2]]


_AXIS = ("x", "y", "z")


def make_grid(n, d, radius: int = 4) -> Grid3D:  # ref: grid.cpp:5-22
    n = tuple(int(x) for x in n)
    d = tuple(float(x) for x in d)
    for a in range(3):
        if n[a] < 1:
            raise ConfigError(f"grid size must be >= 1 along {_AXIS[a]}, got {n[a]}")
        if not d[a] > 0.0:
            raise ConfigError(f"grid spacing must be > 0 along {_AXIS[a]}")
    if radius < 1:
        raise ConfigError("stencil radius must be >= 1")
    return Grid3D(n, d, int(radius))


@dataclass
class RegionPartition:  # ref: grid.hpp:113-117
    inner: IndexBox
    slabs: list  # XLo, XHi, YLo, YHi, ZLo, ZHi


def partition_regions(grid: Grid3D, nd) -> RegionPartition:  # ref: grid.cpp:24-45
    nx, ny, nz = grid.n
    for a in range(3):
        if nd[a] < 0:
            raise ConfigError("ndamping must be >= 0")
        if 2 * nd[a] >= grid.n[a]:
            raise ConfigError(f"damping layers too thick along {_AXIS[a]}: "
                              f"2*{nd[a]} >= {grid.n[a]}")
    inner = IndexBox((nd[0], nd[1], nd[2]), (nx - nd[0], ny - nd[1], nz - nd[2]))
    slabs = [
        IndexBox((0, 0, 0), (nd[0], ny, nz)),
        IndexBox((nx - nd[0], 0, 0), (nx, ny, nz)),
        IndexBox((nd[0], 0, 0), (nx - nd[0], nd[1], nz)),
        IndexBox((nd[0], ny - nd[1], 0), (nx - nd[0], ny, nz)),
        IndexBox((nd[0], nd[1], 0), (nx - nd[0], ny - nd[1], nd[2])),
        IndexBox((nd[0], nd[1], nz - nd[2]), (nx - nd[0], ny - nd[1], nz)),
    ]
    slabs = [IndexBox() if s.empty() else s for s in slabs]
    return RegionPartition(inner, slabs)


def fill_ghosts_replicate(f: np.ndarray, grid: Grid3D) -> np.ndarray:
    """ref: grid.hpp:96-108 (in place; returns f)."""
    r = grid.radius
    nx, ny, nz = grid.n
    ix = np.clip(np.arange(-r, nx + r), 0, nx - 1) + r
    iy = np.clip(np.arange(-r, ny + r), 0, ny - 1) + r
    iz = np.clip(np.arange(-r, nz + r), 0, nz - 1) + r
    f[...] = f[np.ix_(ix, iy, iz)]
    return f


# ------------------------------------------------------------------- stencil
@dataclass
class StencilCoeffs:  # ref: stencil.hpp:17-23
    radius: int
    spacing: float
    c: np.ndarray
    center: float = 0.0


def second_derivative_coeffs(radius: int, h: float) -> StencilCoeffs:
    c = (C.c_double * 8)()
    center = C.c_double()
    check(lib().mm_second_derivative_coeffs(radius, h, c, C.byref(center)))
    return StencilCoeffs(radius, h, np.array(c[:radius]), center.value)


def central_first_derivative_coeffs(radius: int, h: float) -> StencilCoeffs:
    c = (C.c_double * 8)()
    check(lib().mm_central_first_derivative_coeffs(radius, h, c))
    return StencilCoeffs(radius, h, np.array(c[:radius]), 0.0)


def staggered_first_derivative_coeffs(radius: int, h: float) -> StencilCoeffs:
    """ref: stencil.cpp:76-97 (acoustic_iso's half-cell derivative)."""
    c = (C.c_double * 8)()
    check(lib().mm_staggered_first_derivative_coeffs(radius, h, c))
    return StencilCoeffs(radius, h, np.array(c[:radius]), 0.0)


# ---------------------------------------------------------------------- CPML
@dataclass
class AxisCpml:  # ref: cpml.hpp:13-18
    a: np.ndarray
    b: np.ndarray
    inv_kappa: np.ndarray


@dataclass
class CpmlProfile:  # ref: cpml.hpp:20-26
    axis: list
    ndamping: tuple = (0, 0, 0)
    d0: tuple = (0.0, 0.0, 0.0)


def build_profile(n, h, ndamping, fmax, vmax, dt, r_target=1e-3,
                  free_surface=False) -> CpmlProfile:
    n = tuple(int(x) for x in n)
    tot = sum(n)
    a = np.zeros(tot, np.float32)
    b = np.zeros(tot, np.float32)
    k = np.zeros(tot, np.float32)
    d0 = (C.c_double * 3)()
    check(lib().mm_build_profile(_i3(*n), _d3(*h), _i3(*ndamping), fmax, vmax, dt, r_target,
                                 int(free_surface), _fptr(a), _fptr(b), _fptr(k), d0))
    axes, o = [], 0
    for ax in range(3):
        axes.append(AxisCpml(a[o:o + n[ax]].copy(), b[o:o + n[ax]].copy(),
                             k[o:o + n[ax]].copy()))
        o += n[ax]
    return CpmlProfile(axes, tuple(ndamping), tuple(d0))


def taper_material(f: np.ndarray, ntaper, offset, global_n, grid: Grid3D) -> np.ndarray:
    """ref: propagator.hpp:36-62 (in place on a ghosted float32 field; returns f)."""
    assert f.shape == grid.shape and f.dtype == np.float32 and f.flags.c_contiguous
    check(lib().mm_taper_material(_fptr(f), _i3(*grid.n), grid.radius, _i3(*ntaper),
                                  _i3(*offset), _i3(*global_n)))
    return f


# --------------------------------------------------------------------- model
@dataclass
class EarthModel:  # ref: model.hpp:13-25 (vp, optional rho; vs is elastic-only)
    grid: Grid3D
    vp: np.ndarray
    vmin: float = 0.0
    vmax: float = 0.0
    rho: Optional[np.ndarray] = None  # acoustic_iso only

    def has_rho(self) -> bool:
        return self.rho is not None


def validate_model(m: EarthModel) -> EarthModel:  # ref: model.cpp:15-43
    vmin, vmax = C.c_float(), C.c_float()
    m.vp = np.ascontiguousarray(m.vp, dtype=np.float32)
    check(lib().mm_validate_model(_i3(*m.grid.n), m.grid.radius, _fptr(m.vp), C.byref(vmin),
                                  C.byref(vmax)))
    m.vmin, m.vmax = vmin.value, vmax.value
    if m.rho is not None:
        m.rho = np.ascontiguousarray(m.rho, dtype=np.float32)
        inner = m.grid.inner(m.rho)
        if not (np.isfinite(inner).all() and (inner > 0.0).all()):
            raise ValidationError("rho must be finite and > 0 everywhere")
        fill_ghosts_replicate(m.rho, m.grid)
    return m


def constant_model(grid: Grid3D, vp: float, rho: Optional[float] = None) -> EarthModel:
    """ref: model.cpp:45-61 (vs omitted: elastic only)."""
    return validate_model(EarthModel(grid, grid.field(vp), rho=None if rho is None
                                     else grid.field(rho)))


def default_layered_model(grid: Grid3D) -> EarthModel:  # ref: model.cpp:63-77
    vp = grid.field()
    vmin, vmax = C.c_float(), C.c_float()
    check(lib().mm_layered_model(_i3(*grid.n), grid.radius, _fptr(vp), C.byref(vmin),
                                 C.byref(vmax)))
    return EarthModel(grid, vp, vmin.value, vmax.value, rho=grid.field(1000.0))


def random_model(grid: Grid3D, lo: float = 1500.0, hi: float = 4500.0,
                 seed: int = 1) -> EarthModel:
    """Synthetic random-vp model U[lo, hi) (numpy PCG64 stream; the recipe of
    bench_stencil.cpp:11-16 with numpy's generator instead of mt19937)."""
    rng = np.random.default_rng(seed)
    vp = grid.field()
    grid.inner(vp)[...] = rng.uniform(lo, hi, size=grid.n).astype(np.float32)
    return validate_model(EarthModel(grid, vp))


# -------------------------------------------------------------------- source
@dataclass
class Wavelet:  # ref: source.hpp:13-19
    samples: np.ndarray
    dt: float
    fmax: float
    t0: float


def ricker(fmax: float, dt: float, nsteps: int) -> Wavelet:  # ref: source.cpp:11-28
    out = np.zeros(max(nsteps, 0), np.float32)
    check(lib().mm_ricker(fmax, dt, nsteps, _fptr(out) if nsteps > 0 else None))
    return Wavelet(out, dt, fmax, 1.5 / (fmax / 2.5))


def integrate_wavelet(w: Wavelet) -> Wavelet:  # ref: source.cpp:30-38
    """Running time integral (double accumulator): the source of the
    first-order acoustic_iso system."""
    src = np.ascontiguousarray(w.samples, dtype=np.float32)
    out = np.zeros_like(src)
    if src.size:
        check(lib().mm_integrate_wavelet(_fptr(src), src.size, float(w.dt), _fptr(out)))
    return Wavelet(out, w.dt, w.fmax, w.t0)


@dataclass
class AcquisitionGeometry:  # ref: source.hpp:27-36
    source_loc: tuple = (0, 0, 0)
    receivers: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int32))
    receiver_increment: tuple = (1, 1)
    source_increment: tuple = (1, 1, 0)
    nshots: int = 1
    time_rec: float = 0.0

    def nreceivers(self) -> int:
        return int(self.receivers.shape[0])


def default_receivers(grid: Grid3D, ndamping, increment=(1, 1)) -> AcquisitionGeometry:
    """ref: source.cpp:40-50 -- one receiver per (i, j) (strides `increment`) at
    k = ndamping[2]; source at the grid centre."""
    ii = np.arange(0, grid.n[0], increment[0])
    jj = np.arange(0, grid.n[1], increment[1])
    I, J = np.meshgrid(ii, jj, indexing="ij")
    rec = np.stack([I.ravel(), J.ravel(), np.full(I.size, ndamping[2])], axis=1).astype(np.int32)
    return AcquisitionGeometry(tuple(x // 2 for x in grid.n), rec, tuple(increment))


@dataclass
class ShotRecord:  # ref: source.hpp:44-52
    nsteps: int
    dt: float
    geometry: AcquisitionGeometry
    traces: np.ndarray  # [nreceivers, nsteps]

    def at(self, receiver: int, step: int) -> float:
        return float(self.traces[receiver, step])


def version() -> str:
    return lib().mm_version().decode()


__all__ = [n for n in dir() if not n.startswith("_")] + ["_lib"]
