"""minimod-b200: B200-native acoustic_iso_cd propagator (Minimod, arXiv 2007.06048).

Python front-end over the C-ABI CUDA library ``libminimod_b200.so``
(include/minimod_b200.h).  Mirrors the reference's engine/driver interface:
``AcousticCdEngine``, ``EngineOptions``, ``SimConfig``, ``run``, ``cfl_dt``,
``ricker``, ``default_layered_model`` ...; plus the next
propagator, ``AcousticVdEngine`` (acoustic_iso, variable density).
"""
import os as _os

# Each engine drives four CUDA streams (step, pass-1 side, interior side, trace
# copies).  With the driver's default of 8 hardware connections, a third engine
# in a process shares queues with the others and its interior kernel
# serialises behind pass 1 (168 vs 153 us/step at 240^3).  Only effective when
# set before the process creates its CUDA context.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from ._lib import (CollectiveError, ConfigError, CudaError, InstabilityError, MinimodError,
                   ValidationError, device_count, kernel_launch_count)
from .driver import (RunReport, SimConfig, build_geometry, cfl_dt, render_parameter_block,
                     render_timing, run)
from .numerics import (AcquisitionGeometry, AxisCpml, CpmlProfile, EarthModel, Grid3D, IndexBox,
                       RegionPartition, ShotRecord, StencilCoeffs, Wavelet, build_profile,
                       central_first_derivative_coeffs, constant_model, default_layered_model,
                       default_receivers, fill_ghosts_replicate, integrate_wavelet, intersect,
                       make_grid, staggered_first_derivative_coeffs,
                       partition_regions, random_model, ricker, second_derivative_coeffs,
                       taper_material, validate_model, version)
from .propagator import AcousticCdEngine, AcousticVdEngine, EngineOptions
from .shotio import load_model, load_record, save_model, save_record

__all__ = [
    "AcousticCdEngine", "AcousticVdEngine", "EngineOptions", "SimConfig", "RunReport", "run", "cfl_dt",
    "build_geometry", "Grid3D", "IndexBox", "RegionPartition", "make_grid", "partition_regions",
    "intersect", "fill_ghosts_replicate", "StencilCoeffs", "second_derivative_coeffs",
    "central_first_derivative_coeffs", "AxisCpml", "CpmlProfile", "build_profile",
    "taper_material", "EarthModel", "validate_model", "constant_model", "default_layered_model",
    "random_model", "Wavelet", "ricker", "AcquisitionGeometry", "default_receivers",
    "ShotRecord", "ConfigError", "ValidationError", "InstabilityError", "CudaError",
    "CollectiveError", "MinimodError", "device_count", "kernel_launch_count", "version",
    "render_parameter_block", "render_timing", "save_record", "load_record", "save_model",
    "load_model", "staggered_first_derivative_coeffs", "integrate_wavelet",
]
