"""ctypes binding of the C-ABI in include/hwflow_c.h (+ hwflow_ext.h).

`Library(path)` binds any shared library that exports the interface — the
product (`lib/libhwflow_cuda.so`) or, in tests only, the CPU checkers under
oracle/. Arrays cross as numpy buffers (host memory).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HWF_OK, HWF_EINVAL, HWF_EDIVERGED, HWF_ECUDA = 0, 1, 2, 3
HWF_MAX_LEVELS = 8
HWF_MAX_GN = 32
DTYPE_U8, DTYPE_F64 = 0, 1

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class EnergyParamsC(C.Structure):  # energy.hpp:17-27
    _fields_ = [(n, C.c_double) for n in (
        "w_reg", "w_photo", "w_grad", "w_epi", "w_smooth", "w_mag",
        "w_s", "w_m", "w_d", "m_s", "m_m", "m_d", "eps_huber", "eps_color")]


class ScheduleC(C.Structure):  # solver.hpp:14-28
    _fields_ = [
        ("levels", C.c_int), ("n_gn_per_level", C.c_int), ("gn_per_level", C.c_int * HWF_MAX_LEVELS),
        ("pcg_iters", C.c_int), ("patch_iters", C.c_int), ("subdomain_px", C.c_int),
        ("boundary_px", C.c_int), ("grid_step", C.c_int), ("threads", C.c_int),
        ("lm_lambda", C.c_double), ("active_fields", C.c_uint32), ("coarse_s_offset", C.c_double * 2)]


class Frame4C(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("dtype", C.c_int), ("plane", C.c_void_p * 4)]


class ResultC(C.Structure):
    _fields_ = [("s", _dp), ("m", _dp), ("d", _dp), ("disparity", _dp), ("vis4", _u8p), ("grid_total", _dp)]


class StatsC(C.Structure):
    _fields_ = [("levels_used", C.c_int), ("gn_iters", C.c_int * HWF_MAX_LEVELS),
                ("energy_before", (C.c_double * HWF_MAX_GN) * HWF_MAX_LEVELS),
                ("energy_after", (C.c_double * HWF_MAX_GN) * HWF_MAX_LEVELS)]


class LevelC(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("grid_step", C.c_int),
                ("images", _dp * 4), ("illum", _dp * 4), ("total", _dp), ("delta", _dp),
                ("vis4", _u8p), ("outlier", _u8p), ("node_w", _dp), ("fundamental", _dp)]


class EnergyC(C.Structure):
    _fields_ = [("photo", C.c_double), ("grad", C.c_double), ("smooth", C.c_double), ("epi", C.c_double),
                ("mag", C.c_double), ("total", C.c_double), ("residual_count", C.c_int64)]


class RigC(C.Structure):  # geometry.hpp:14-23 StereoRig
    _fields_ = [("F", C.c_double * 9), ("has_projections", C.c_int), ("P0", C.c_double * 12),
                ("P1", C.c_double * 12)]


class HwflowError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class SolverDivergence(HwflowError):
    """core.hpp:19-21 — raised for HWF_EDIVERGED."""


class InvalidArgument(HwflowError, ValueError):
    pass


def ptr(a: np.ndarray | None, ctype=C.c_double):
    if a is None:
        return C.POINTER(ctype)()
    assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


def dptr(a):
    return ptr(a, C.c_double)


def u8ptr(a):
    return ptr(a, C.c_uint8)


_SIGS = {
    "hwf_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "hwf_destroy": (None, [C.c_void_p]),
    "hwf_last_error": (C.c_char_p, [C.c_void_p]),
    "hwf_backend": (C.c_char_p, []),
    "hwf_default_params": (None, [C.POINTER(EnergyParamsC)]),
    "hwf_preset_params": (C.c_int, [C.c_char_p, C.POINTER(EnergyParamsC)]),
    "hwf_validate_params": (C.c_int, [C.POINTER(EnergyParamsC)]),
    "hwf_default_schedule": (None, [C.POINTER(ScheduleC)]),
    "hwf_level_dims": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "hwf_solve_pair": (C.c_int, [C.c_void_p, C.POINTER(Frame4C), C.POINTER(EnergyParamsC), C.POINTER(ScheduleC),
                                 _dp, C.POINTER(ResultC), C.POINTER(StatsC)]),
    "hwf_solve_batch": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(Frame4C), C.POINTER(EnergyParamsC),
                                  C.POINTER(ScheduleC), _dp, C.POINTER(ResultC), C.POINTER(StatsC)]),
    "hwf_state_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "hwf_state_destroy": (None, [C.c_void_p]),
    "hwf_state_read": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, _dp, _dp]),
    "hwf_solve_batch_seq": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(Frame4C), C.POINTER(EnergyParamsC),
                                      C.POINTER(ScheduleC), _dp, C.c_void_p, C.c_void_p, C.POINTER(ResultC),
                                      C.POINTER(StatsC)]),
    "hwf_propagate_temporal": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]),
    "hwf_pyramid": (C.c_int, [C.c_void_p, C.POINTER(Frame4C), C.c_int, _dp]),
    "hwf_eval_energy": (C.c_int, [C.c_void_p, C.POINTER(LevelC), C.POINTER(EnergyParamsC), C.POINTER(EnergyC), _dp]),
    "hwf_refresh_weights": (C.c_int, [C.c_void_p, C.POINTER(LevelC), C.POINTER(EnergyParamsC), _u8p, _dp]),
    "hwf_linearize": (C.c_int, [C.c_void_p, C.POINTER(LevelC), C.POINTER(EnergyParamsC), C.c_uint32, C.c_double,
                                _dp, _dp, _dp]),
    "hwf_assemble_jacobian": (C.c_int, [C.c_void_p, C.POINTER(LevelC), C.POINTER(EnergyParamsC), C.c_uint32, C.c_int,
                                        _dp, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp, C.c_longlong,
                                        C.POINTER(C.c_longlong)]),
    "hwf_normal_dense": (C.c_int, [C.c_int, C.c_int, _dp, _dp]),
    "hwf_pcg": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _dp, _dp, C.c_int, _dp, _dp]),
    "hwf_schwarz": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_int,
                              _dp]),
    "hwf_gn_level": (C.c_int, [C.c_void_p, C.POINTER(LevelC), _dp, _dp, _u8p, _dp, C.POINTER(EnergyParamsC),
                               C.POINTER(ScheduleC), C.c_int, _dp, _dp]),
    "hwf_gn_level_trace": (C.c_int, [C.c_void_p, C.POINTER(LevelC), _dp, _dp, _u8p, _dp, C.POINTER(EnergyParamsC),
                                     C.POINTER(ScheduleC), C.c_int, _dp, _dp, _dp]),
    "hwf_occlusion": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, _u8p]),
    "hwf_illumination": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, _dp * 4, _dp, _u8p, _dp]),
    "hwf_prolongate": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _u8p, _dp, _dp,
                                 _u8p, _dp]),
    "hwf_validate_rig": (C.c_int, [C.c_void_p, C.POINTER(RigC)]),
    "hwf_triangulate": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp, _u8p]),
    "hwf_scene_points": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _dp, _dp, _dp, C.POINTER(RigC), _dp, _dp, _dp,
                                   _u8p]),
    "hwf_export_mesh_obj": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _dp, _u8p, _dp, _u8p, C.c_char_p]),
}

_EXT_SIGS = {
    "hwf_prepare_device": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(EnergyParamsC),
                                     C.POINTER(ScheduleC), _dp, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "hwf_run_device": (C.c_int, [C.c_void_p]),
    "hwf_sync": (C.c_int, [C.c_void_p, C.POINTER(StatsC)]),
    "hwf_stream": (C.c_void_p, [C.c_void_p]),
    "hwf_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "hwf_launch_count": (C.c_int, [C.c_void_p]),
    "hwf_pixel_kernel_times": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp]),
    "hwf_gn_iteration_times": (C.c_int, [C.c_void_p, C.c_int, _dp, C.POINTER(C.c_int)]),
    "hwf_submit_batch": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(Frame4C), C.POINTER(EnergyParamsC),
                                   C.POINTER(ScheduleC), _dp, C.POINTER(ResultC), C.POINTER(StatsC)]),
    "hwf_wait": (C.c_int, [C.c_void_p]),
}

_vpp = C.POINTER(C.c_void_p)
_SPLIT_SIGS = {  # include/hwflow_split.h (both the CUDA library and the oracle)
    "hwf_split_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(EnergyParamsC),
                                   C.POINTER(ScheduleC), _dp, C.c_int, C.c_int, _vpp]),
    "hwf_split_destroy": (None, [C.c_void_p]),
    "hwf_split_schedule": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "hwf_split_rows": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "hwf_split_buffer": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p, _vpp, C.POINTER(C.c_longlong)]),
    "hwf_split_swept": (C.c_char_p, [C.c_int]),
    "hwf_split_begin": (C.c_int, [C.c_void_p, C.POINTER(Frame4C)]),
    "hwf_split_upload": (C.c_int, [C.c_void_p, C.POINTER(Frame4C)]),
    "hwf_split_prologue": (C.c_int, [C.c_void_p]),
    "hwf_split_level_begin": (C.c_int, [C.c_void_p, C.c_int]),
    "hwf_split_linearize": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "hwf_split_sweep": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "hwf_split_row_elems": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.POINTER(C.c_longlong)]),
    "hwf_split_pcg": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int]),
    "hwf_split_pcg_scalars": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int]),
    "hwf_split_energy_after": (C.c_int, [C.c_void_p, C.c_int]),
    "hwf_split_level_end": (C.c_int, [C.c_void_p, C.c_int]),
    "hwf_split_finish": (C.c_int, [C.c_void_p, C.POINTER(ResultC), C.POINTER(StatsC)]),
}

EXPORTED = sorted(_SIGS)
EXPORTED_EXT = sorted(_EXT_SIGS)
EXPORTED_SPLIT = sorted(_SPLIT_SIGS)


class Library:
    """One loaded implementation of the C-ABI."""

    def __init__(self, path: str | Path):
        self.path = Path(path)
        self.lib = C.CDLL(str(self.path))
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.lib, name)
            fn.restype, fn.argtypes = res, args
        for name, (res, args) in _SPLIT_SIGS.items():
            fn = getattr(self.lib, name)
            fn.restype, fn.argtypes = res, args
        self.has_ext = all(hasattr(self.lib, n) for n in _EXT_SIGS)
        if self.has_ext:
            for name, (res, args) in _EXT_SIGS.items():
                fn = getattr(self.lib, name)
                fn.restype, fn.argtypes = res, args

    @property
    def backend(self) -> str:
        return self.lib.hwf_backend().decode()

    def __getattr__(self, name):
        return getattr(self.lib, name)


class Context:
    """hwf_ctx* with error translation (HWF_* codes -> exceptions)."""

    def __init__(self, lib: Library, device: int = 0):
        self.lib = lib
        h = C.c_void_p()
        rc = lib.hwf_create(device, C.byref(h))
        if rc != HWF_OK:
            raise HwflowError(rc, f"hwf_create failed for {lib.path.name} (device {device})")
        self.h = h

    def close(self):
        if self.h:
            self.lib.hwf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc == HWF_OK:
            return
        msg = (self.lib.hwf_last_error(self.h) or b"").decode()
        if rc == HWF_EDIVERGED:
            raise SolverDivergence(rc, msg)
        if rc == HWF_EINVAL:
            raise InvalidArgument(rc, msg)
        raise HwflowError(rc, msg)
