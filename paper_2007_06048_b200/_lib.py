"""ctypes binding of libminimod_b200.so (the C ABI in include/minimod_b200.h).

The library is built in-tree (``python -m paper_2007_06048_b200.build``) and
loaded from this directory.  There is no fallback: if the library is missing
or cannot be loaded, importing the engine raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# MM_LIB_VARIANT=<name> loads an experiment build (build.py --variant <name>)
LIB_PATH = Path(__file__).resolve().parent / (
    f"libminimod_b200_{os.environ['MM_LIB_VARIANT']}.so" if os.environ.get("MM_LIB_VARIANT")
    else "libminimod_b200.so")

MM_OK, MM_ECONFIG, MM_EVALIDATION, MM_EINSTABILITY, MM_EINVAL, MM_ECUDA, MM_ENCCL = range(7)
MM_MODE_FAST, MM_MODE_STRICT, MM_MODE_FAST_FMA = 0, 1, 2


class MinimodError(RuntimeError):
    """Base class; ``code`` is the mm_status."""

    code = -1

    def __init__(self, msg: str, code: int | None = None):
        super().__init__(msg)
        if code is not None:
            self.code = code


class ConfigError(MinimodError):  # ref: errors.hpp:10-13
    code = MM_ECONFIG


class ValidationError(MinimodError):  # ref: errors.hpp:16-19
    code = MM_EVALIDATION


class InstabilityError(MinimodError):  # ref: errors.hpp:22-30
    code = MM_EINSTABILITY

    def __init__(self, msg: str, step: int):
        super().__init__(msg)
        self.step = step


class CudaError(MinimodError):
    code = MM_ECUDA


class CollectiveError(MinimodError):
    code = MM_ENCCL


class mm_grid(C.Structure):
    _fields_ = [("n", C.c_int * 3), ("d", C.c_double * 3), ("radius", C.c_int)]


class mm_engine_options(C.Structure):
    _fields_ = [("ndamping", C.c_int * 3), ("fmax", C.c_double), ("r_target", C.c_double),
                ("free_surface", C.c_int), ("taper", C.c_int), ("ntaper", C.c_int * 3)]


class mm_sim_config(C.Structure):
    _fields_ = [("ngrid", C.c_int * 3), ("dgrid", C.c_double * 3), ("nsteps", C.c_int),
                ("fmax", C.c_double), ("cfl", C.c_double), ("ndamping", C.c_int * 3),
                ("ntaper", C.c_int * 3), ("taper", C.c_int), ("free_surface", C.c_int),
                ("r_target", C.c_double), ("has_source_loc", C.c_int),
                ("source_loc", C.c_int * 3), ("receiver_increment", C.c_int * 2),
                ("stencil_radius", C.c_int)]


class mm_run_report(C.Structure):
    _fields_ = [("dt", C.c_double), ("kernel_seconds", C.c_double),
                ("modeling_seconds", C.c_double), ("steps_run", C.c_int),
                ("nreceivers", C.c_int)]


_P = C.c_void_p
_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "mm_last_error": [],
    "mm_last_instability_step": [],
    "mm_version": [],
    "mm_device_count": [_ip],
    "mm_kernel_launch_count": [],
    "mm_set_tuning": [C.c_char_p, C.c_longlong],
    "mm_get_tuning": [C.c_char_p, C.POINTER(C.c_longlong)],
    "mm_reset_tuning": [],
    "mm_second_derivative_coeffs": [C.c_int, C.c_double, _dp, _dp],
    "mm_central_first_derivative_coeffs": [C.c_int, C.c_double, _dp],
    "mm_cfl_dt": [C.c_double, C.POINTER(mm_grid), C.c_double, _dp],
    "mm_ricker": [C.c_double, C.c_double, C.c_int, _fp],
    "mm_build_profile": [_ip, _dp, _ip, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                         _fp, _fp, _fp, _dp],
    "mm_taper_material": [_fp, _ip, C.c_int, _ip, _ip, _ip],
    "mm_layered_model": [_ip, C.c_int, _fp, _fp, _fp],
    "mm_validate_model": [_ip, C.c_int, _fp, _fp, _fp],
    "mm_cd_create": [C.POINTER(mm_grid), _ip, _ip, _fp, C.POINTER(mm_engine_options), C.c_float,
                     C.c_double, C.c_int, C.c_int, C.POINTER(_P)],
    "mm_cd_destroy": [_P],
    "mm_cd_step": [_P, C.c_float, _ip],
    "mm_cd_update_boundary_psi": [_P],
    "mm_cd_update_inner": [_P],
    "mm_cd_update_boundary": [_P],
    "mm_cd_inject_source": [_P, C.c_float, _ip],
    "mm_cd_apply_free_surface": [_P],
    "mm_cd_rotate": [_P],
    "mm_cd_synchronize": [_P],
    "mm_cd_field_size": [_P, C.POINTER(C.c_size_t)],
    "mm_cd_get_dt": [_P, _fp],
    "mm_cd_get_mode": [_P, _ip],
    "mm_cd_steps_taken": [_P, C.POINTER(C.c_longlong)],
    "mm_cd_get_pressure": [_P, _fp],
    "mm_cd_get_pressure_prev": [_P, _fp],
    "mm_cd_get_velocity": [_P, _fp],
    "mm_cd_set_state": [_P, _fp, _fp],
    "mm_cd_get_profile": [_P, C.c_int, _fp, _fp, _fp],
    "mm_cd_set_profile": [_P, C.c_int, _fp, _fp, _fp],
    "mm_cd_get_d0": [_P, _dp],
    "mm_cd_set_receivers": [_P, _ip, C.c_int, C.c_int],
    "mm_cd_record": [_P, C.c_int],
    "mm_cd_get_traces": [_P, _fp, C.c_int],
    "mm_cd_copy_trace_step": [_P, C.c_int, _fp, C.c_int],
    "mm_cd_run": [_P, _fp, C.c_int, _ip, C.c_int, C.c_int, _fp],
    "mm_cd_stream": [_P, C.POINTER(_P)],
    "mm_cd_kernel_timing": [_P, C.c_int],
    "mm_cd_cpml_path": [_P, C.c_char_p, C.c_int],
    "mm_cd_kernel_times": [_P, C.c_int, C.c_void_p, _dp, C.POINTER(C.c_longlong), _ip],
    "mm_cd_halo_planes": [_P, C.c_int, C.c_int, C.POINTER(_P), C.POINTER(C.c_size_t)],
    "mm_cd_next_halo_planes": [_P, C.c_int, C.c_int, C.POINTER(_P), C.POINTER(C.c_size_t)],
    "mm_cd_update_planes": [_P, C.c_int, C.c_int],
    "mm_cd_update_plane_ranges": [_P, C.POINTER(C.c_int), C.c_int],
    "mm_nccl_get_unique_id": [C.c_void_p],
    "mm_zslab_validate_cuts": [_ip, C.c_int, C.c_int, C.c_int, C.c_int],
    "mm_cd_group_create": [C.POINTER(mm_grid), _ip, C.c_int, C.c_int, C.c_void_p, _fp,
                           C.POINTER(mm_engine_options), C.c_float, C.c_double, C.c_int, C.c_int,
                           C.POINTER(_P)],
    "mm_cd_group_destroy": [_P],
    "mm_cd_group_engine": [_P, C.POINTER(_P)],
    "mm_cd_group_slab": [_P, _ip, _ip],
    "mm_cd_group_step": [_P, C.c_float, _ip],
    "mm_cd_group_run": [_P, _fp, C.c_int, _ip, C.c_int, C.c_int, _fp],
    "mm_cd_group_step_local": [C.POINTER(_P), C.c_int, C.c_float, _ip],
    "mm_sim_config_default": [C.POINTER(mm_sim_config)],
    "mm_run": [C.POINTER(mm_sim_config), _fp, C.c_int, C.c_int, _fp, C.POINTER(mm_run_report)],
    # acoustic_iso (variable density)
    "mm_staggered_first_derivative_coeffs": [C.c_int, C.c_double, _dp],
    "mm_integrate_wavelet": [_fp, C.c_int, C.c_double, _fp],
    "mm_vd_create": [C.POINTER(mm_grid), _fp, _fp, C.POINTER(mm_engine_options), C.c_float,
                     C.c_double, C.c_int, C.POINTER(_P)],
    "mm_vd_destroy": [_P],
    "mm_vd_step": [_P, C.c_float, _ip],
    "mm_vd_update_velocity": [_P],
    "mm_vd_update_pressure": [_P],
    "mm_vd_inject_source": [_P, C.c_float, _ip],
    "mm_vd_apply_free_surface": [_P],
    "mm_vd_synchronize": [_P],
    "mm_vd_field_size": [_P, C.POINTER(C.c_size_t)],
    "mm_vd_get_dt": [_P, _fp],
    "mm_vd_steps_taken": [_P, C.POINTER(C.c_longlong)],
    "mm_vd_get_pressure": [_P, _fp],
    "mm_vd_get_velocity": [_P, C.c_int, _fp],
    "mm_vd_set_pressure": [_P, _fp],
    "mm_vd_set_velocity": [_P, C.c_int, _fp],
    "mm_vd_set_receivers": [_P, _ip, C.c_int, C.c_int],
    "mm_vd_record": [_P, C.c_int],
    "mm_vd_get_traces": [_P, _fp, C.c_int],
    "mm_vd_copy_trace_step": [_P, C.c_int, _fp, C.c_int],
    "mm_vd_run": [_P, _fp, C.c_int, _ip, C.c_int, C.c_int, _fp],
    "mm_vd_stream": [_P, C.POINTER(_P)],
    "mm_run_vd": [C.POINTER(mm_sim_config), _fp, _fp, C.c_int, _fp, C.POINTER(mm_run_report)],
}
_RESTYPES = {
    "mm_last_error": C.c_char_p,
    "mm_version": C.c_char_p,
    "mm_kernel_launch_count": C.c_longlong,
}

_lib = None


def lib() -> C.CDLL:
    """Load (once) and return the C-ABI library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2007_06048_b200.build` "
            "(there is no CPU fallback for the engines)")
    L = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
    for name, args in SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, C.c_int)
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == MM_OK:
        return
    L = lib()
    msg = L.mm_last_error().decode()
    if rc == MM_ECONFIG:
        raise ConfigError(msg)
    if rc == MM_EVALIDATION:
        raise ValidationError(msg)
    if rc == MM_EINSTABILITY:
        raise InstabilityError(msg, L.mm_last_instability_step())
    if rc == MM_EINVAL:
        raise ValueError(msg)
    if rc == MM_ECUDA:
        raise CudaError(msg)
    if rc == MM_ENCCL:
        raise CollectiveError(msg)
    raise MinimodError(msg, rc)


def device_count() -> int:
    n = C.c_int()
    check(lib().mm_device_count(C.byref(n)))
    return n.value


def set_tuning(name: str, value: int) -> None:
    """Process-wide tuning parameter (mm_set_tuning; csrc/engine.cu kTunables)."""
    check(lib().mm_set_tuning(name.encode(), int(value)))


def get_tuning(name: str) -> int:
    v = C.c_longlong()
    check(lib().mm_get_tuning(name.encode(), C.byref(v)))
    return v.value


def reset_tuning() -> None:
    check(lib().mm_reset_tuning())


class tuned:
    """Context manager: tuning parameters set for the block, then restored."""

    def __init__(self, **params):
        self.params = params
        self.saved = {}

    def __enter__(self):
        for k, v in self.params.items():
            self.saved[k] = get_tuning(k)
            set_tuning(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.saved.items():
            set_tuning(k, v)


def kernel_launch_count() -> int:
    return int(lib().mm_kernel_launch_count())


def loaded_path() -> str:
    return os.fspath(LIB_PATH)
