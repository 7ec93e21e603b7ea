"""run() -- the reference's modeling driver on the GPU.

ref: driver.hpp:21-54 (SimConfig, RunReport), driver.cpp:19-29 (cfl_dt),
driver.cpp:37-47 (build_geometry), driver.cpp:83-144 (run).  Two propagators:
``acoustic_iso_cd`` (the hot path) and ``acoustic_iso`` (variable density,
SURVEY.md §8(f) row 4; integrated Ricker source, driver.cpp:122-128).  The
time loop itself runs in C++ (``mm_run`` in csrc/engine.cu, ``mm_run_vd`` in
csrc/vd_engine.cu): device-resident wavelet, device receiver recording, one
receiver-0 finiteness check per step.
``kernel_seconds`` is the device time of the step loop (CUDA events), the
analogue of the reference's "Time Kernel" (driver.cpp:102-107).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from . import _lib
from ._lib import ConfigError, ValidationError, check, lib
from .numerics import (AcquisitionGeometry, EarthModel, Grid3D, ShotRecord, default_receivers,
                       make_grid)


@dataclass
class SimConfig:  # ref: driver.hpp:21-47 (same defaults; no elastic_iso)
    propagator: str = "acoustic_iso_cd"
    ngrid: tuple = (100, 100, 100)
    dgrid: tuple = (20.0, 20.0, 20.0)
    nsteps: int = 1000
    fmax: float = 25.0
    cfl: float = 0.8
    ndamping: tuple = (27, 27, 27)
    ntaper: tuple = (3, 3, 3)
    taper: bool = True
    free_surface: bool = False
    r_target: float = 1e-3
    source_loc: Optional[tuple] = None
    receiver_increment: tuple = (1, 1)
    stencil_radius: int = 4

    def to_c(self) -> _lib.mm_sim_config:
        c = _lib.mm_sim_config()
        check(lib().mm_sim_config_default(C.byref(c)))
        c.ngrid[:] = [int(x) for x in self.ngrid]
        c.dgrid[:] = [float(x) for x in self.dgrid]
        c.nsteps = int(self.nsteps)
        c.fmax = float(self.fmax)
        c.cfl = float(self.cfl)
        c.ndamping[:] = [int(x) for x in self.ndamping]
        c.ntaper[:] = [int(x) for x in self.ntaper]
        c.taper = int(bool(self.taper))
        c.free_surface = int(bool(self.free_surface))
        c.r_target = float(self.r_target)
        c.has_source_loc = int(self.source_loc is not None)
        if self.source_loc is not None:
            c.source_loc[:] = [int(x) for x in self.source_loc]
        c.receiver_increment[:] = [int(x) for x in self.receiver_increment]
        c.stencil_radius = int(self.stencil_radius)
        return c


@dataclass
class RunReport:  # ref: driver.hpp:49-54
    dt: float = 0.0
    kernel_seconds: float = 0.0
    modeling_seconds: float = 0.0
    steps_run: int = 0


def cfl_dt(model: EarthModel, grid: Grid3D, cfl: float) -> float:  # ref: driver.cpp:19-29
    g = _lib.mm_grid()
    g.n[:] = list(grid.n)
    g.d[:] = list(grid.d)
    g.radius = grid.radius
    dt = C.c_double()
    check(lib().mm_cfl_dt(float(model.vmax), C.byref(g), float(cfl), C.byref(dt)))
    return dt.value


def build_geometry(config: SimConfig, grid: Grid3D) -> AcquisitionGeometry:
    """ref: driver.cpp:37-47."""
    g = default_receivers(grid, config.ndamping, config.receiver_increment)
    if config.source_loc is not None:
        g.source_loc = tuple(config.source_loc)
    if not grid.interior().contains(*g.source_loc):
        raise ConfigError("source location outside grid interior")
    return g


PROPAGATORS = ("acoustic_iso_cd", "acoustic_iso")


def run(config: SimConfig, model: EarthModel, *, device: int = 0,
        mode: str = "fast") -> Tuple[ShotRecord, RunReport]:
    """ref: driver.cpp:83-144.  ``mode`` selects the acoustic_iso_cd kernel
    family (acoustic_iso has one)."""
    if config.propagator not in PROPAGATORS:
        raise ConfigError(f"unknown propagator '{config.propagator}' (this build: "
                          f"{', '.join(PROPAGATORS)})")
    if config.nsteps < 1:
        raise ConfigError("nsteps must be >= 1")
    if tuple(model.grid.n) != tuple(config.ngrid):
        raise ConfigError("model grid does not match configured ngrid")
    grid = make_grid(config.ngrid, config.dgrid, config.stencil_radius)
    geom = build_geometry(config, grid)
    vp = np.ascontiguousarray(model.vp, dtype=np.float32)
    if vp.shape != grid.shape:
        raise ConfigError("model radius does not match the stencil radius")
    traces = np.zeros((geom.nreceivers(), config.nsteps), np.float32)
    rep = _lib.mm_run_report()
    if config.propagator == "acoustic_iso":
        if model.rho is None:
            raise ValidationError("acoustic_iso requires a density volume (rho)")
        rho = np.ascontiguousarray(model.rho, dtype=np.float32)
        check(lib().mm_run_vd(C.byref(config.to_c()), vp.ctypes.data_as(C.POINTER(C.c_float)),
                              rho.ctypes.data_as(C.POINTER(C.c_float)), int(device),
                              traces.ctypes.data_as(C.POINTER(C.c_float)), C.byref(rep)))
        record = ShotRecord(config.nsteps, rep.dt, geom, traces)
        return record, RunReport(rep.dt, rep.kernel_seconds, rep.modeling_seconds, rep.steps_run)
    from .propagator import _MODES
    check(lib().mm_run(C.byref(config.to_c()), vp.ctypes.data_as(C.POINTER(C.c_float)),
                       int(device), _MODES[mode],
                       traces.ctypes.data_as(C.POINTER(C.c_float)), C.byref(rep)))
    record = ShotRecord(config.nsteps, rep.dt, geom, traces)
    return record, RunReport(rep.dt, rep.kernel_seconds, rep.modeling_seconds, rep.steps_run)


# ------------------------------------------------------------------ report
# ref: driver.cpp:150-215 -- the Fortran-list-directed parameter block and the
# timing lines printed by `minimod model`.
def _f32_repr(v: float) -> str:
    return "%#.9g" % float(np.float32(v))


def _int_row(name: str, vals) -> str:
    return " %-18s =" % name + "".join("%13d" % int(v) for v in vals) + "\n"


def _float_row(name: str, vals) -> str:
    s = " %-18s =" % name
    for i, v in enumerate(vals):
        s += ("    " if i == 0 else "       ") + _f32_repr(v)
    return s + "    \n"


def render_parameter_block(config: SimConfig, model: EarthModel, nthreads: int = 1,
                           nshots: int = 1, time_rec: float = 0.0,
                           source_increment=(1, 1, 0)) -> str:
    """ref: driver.cpp:183-209 render_parameter_block."""
    grid = make_grid(config.ngrid, config.dgrid, config.stencil_radius)
    g = build_geometry(config, grid)
    r = config.stencil_radius
    return "".join([
        _int_row("nthreads", [nthreads]), " \n",
        _int_row("ngrid", config.ngrid), _float_row("dgrid", config.dgrid),
        _int_row("nsteps", [config.nsteps]), _float_row("fmax", [config.fmax]),
        _float_row("vmin", [model.vmin]), _float_row("vmax", [model.vmax]),
        _float_row("cfl", [config.cfl]), " \n",
        _int_row("stencil", [r, r, r]), _int_row("source_loc", g.source_loc),
        _int_row("ndamping", config.ndamping), _int_row("ntaper", config.ntaper), " \n",
        _int_row("nshots", [nshots]), _float_row("time_rec", [time_rec]),
        _int_row("nreceivers", [g.nreceivers()]),
        _int_row("receiver_increment", g.receiver_increment),
        _int_row("source_increment", source_increment), " \n",
    ])


def render_timing(report: RunReport) -> str:
    """ref: driver.cpp:211-215 render_timing."""
    return "Time Kernel    %10.2f\nTime Modeling  %10.2f\n" % (report.kernel_seconds,
                                                              report.modeling_seconds)

