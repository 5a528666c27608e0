"""ctypes binding of the C-ABI in include/pcgpu.h (libpcgpu.so, sm_100a).

The library is built in-tree (``__graft_entry__.build()`` /
``make -C paper_1912_03744_b200/csrc``) into ``paper_1912_03744_b200/_lib/``.
There is no CPU fallback: if the shared library is missing this module raises,
and every stepper call goes to the CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# $PCGPU_LIB: another in-tree build of the library (A/B measurements)
LIB_PATH = os.environ.get("PCGPU_LIB") or os.path.join(_HERE, "_lib", "libpcgpu.so")

PCGPU_ABI_VERSION = 3
DIST_IPC_BYTES = 256

# pcgpu_status
OK, ERR_CONFIG, ERR_TAU_FLOOR, ERR_TABLE_RANGE, ERR_ZERO_PIVOT, ERR_CUDA, ERR_ARG = range(7)
# enums
MODE_EXACT = 0
SOURCE_NULL, SOURCE_JOULE, SOURCE_FIELD = 0, 1, 2
LAYOUT_CONTIGUOUS, LAYOUT_STRIDED = 0, 1
STOP_REACHED_TIME, STOP_PERIODIC, STOP_TAU_FLOOR = 0, 1, 2
SNAP_PRE_ON, SNAP_POST_OFF, SNAP_AT_TIME = 0, 1, 2

_dp = C.POINTER(C.c_double)

# pcgpu_evolve callbacks (include/pcgpu.h)
STEP_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_double, C.c_double,
                      C.POINTER(C.c_double))
SNAP_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_double, C.c_void_p)


class Table(C.Structure):
    _fields_ = [("n", C.c_int32), ("t", _dp), ("v", _dp)]


class Material(C.Structure):
    _fields_ = [("rho", C.c_double), ("cv", Table), ("lam", Table), ("chi", Table)]


class Desc(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32),
        ("nr", C.c_int32), ("nz", C.c_int32), ("nr_core", C.c_int32), ("nz_shared", C.c_int32),
        ("layer", C.POINTER(C.c_int32)),
        ("r_center", _dp), ("gap_r", _dp), ("width_z", _dp), ("gap_z", _dp),
        ("n_layers", C.c_int32),
        ("materials", C.POINTER(Material)),
        ("source_kind", C.c_int32), ("source_layer", C.c_int32), ("amplitude", C.c_double),
        ("t_per", C.c_double), ("t_src", C.c_double), ("t_trs", C.c_double),
        ("xi", C.c_double), ("zeta", C.c_double), ("waveform", C.c_int32),
        ("epsilon", C.c_double), ("max_iter", C.c_int32), ("tau_min", C.c_double),
        ("tau_transient_divisor", C.c_double), ("tau_source_divisor", C.c_double),
        ("halfpoint_rule", C.c_int32), ("range_policy", C.c_int32), ("all_neumann", C.c_int32),
        ("T0", C.c_double), ("t_ceiling", C.c_double),
        ("mode", C.c_int32), ("device", C.c_int32),
        ("row_extent", C.POINTER(C.c_int32)), ("col_extent", C.POINTER(C.c_int32)),
    ]


class Outcome(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32), ("last_delta", C.c_double)]


class StepResultC(C.Structure):
    _fields_ = [("tau_used", C.c_double), ("halvings", C.c_int32),
                ("radial", Outcome), ("axial", Outcome)]


class RunStats(C.Structure):
    _fields_ = [("t_end", C.c_double), ("steps", C.c_int64), ("halvings", C.c_int64),
                ("radial_iterations", C.c_int64), ("axial_iterations", C.c_int64),
                ("cell_updates", C.c_double), ("cell_updates_accepted", C.c_double),
                ("attempt_cells", C.c_double)]


# Every symbol include/pcgpu.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "pcgpu_abi_version", "pcgpu_device_count", "pcgpu_create", "pcgpu_destroy",
    "pcgpu_last_error", "pcgpu_error_line", "pcgpu_initial_tau", "pcgpu_pulse_value",
    "pcgpu_active_cells", "pcgpu_set_host_clock", "pcgpu_last_tau_floor",
    "pcgpu_resident_stats", "pcgpu_speculation_stats", "pcgpu_bind_power_field",
    "pcgpu_radial_half_step",
    "pcgpu_axial_half_step", "pcgpu_step", "pcgpu_step_host", "pcgpu_radial_half_step_host",
    "pcgpu_axial_half_step_host", "pcgpu_run", "pcgpu_clamp_events", "pcgpu_stream",
    "pcgpu_kernel_timing", "pcgpu_enable_kernel_timing", "pcgpu_launch_count",
    "pcgpu_tridiag_batch", "pcgpu_nccl_unique_id", "pcgpu_dist_create", "pcgpu_dist_destroy",
    "pcgpu_dist_last_error", "pcgpu_dist_plan", "pcgpu_dist_slabs", "pcgpu_dist_set_field",
    "pcgpu_dist_get_field", "pcgpu_dist_set_field_host", "pcgpu_dist_get_field_host",
    "pcgpu_pipeline_stats",
    "pcgpu_dist_run", "pcgpu_dist_stream", "pcgpu_dist_enable_timing",
    "pcgpu_dist_timing", "pcgpu_dist_launch_count", "pcgpu_run_growth", "pcgpu_describe", "pcgpu_dist_transport",
    "pcgpu_dist_ipc_export", "pcgpu_dist_ipc_import", "pcgpu_dist_peer_off", "pcgpu_evolve", "pcgpu_detector_periods",
    "pcgpu_evolve_host",
    "pcgpu_writer_create", "pcgpu_writer_destroy", "pcgpu_writer_submit", "pcgpu_writer_flush",
    "pcgpu_writer_last_error",
]

CLOCK_FN = C.CFUNCTYPE(C.c_double, C.c_void_p, C.c_double)

_lib = None


def load():
    """Load libpcgpu.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libpcgpu.so not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sig = {
        "pcgpu_abi_version": (C.c_int32, []),
        "pcgpu_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
        "pcgpu_create": (C.c_int, [C.POINTER(Desc), C.POINTER(vp)]),
        "pcgpu_destroy": (None, [vp]),
        "pcgpu_last_error": (C.c_char_p, [vp]),
        "pcgpu_error_line": (C.c_int64, [vp]),
        "pcgpu_initial_tau": (C.c_double, [vp, C.c_double]),
        "pcgpu_pulse_value": (C.c_double, [vp, C.c_double]),
        "pcgpu_active_cells": (C.c_int64, [vp]),
        "pcgpu_set_host_clock": (C.c_int, [vp, CLOCK_FN, CLOCK_FN, vp]),
        "pcgpu_last_tau_floor": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                           C.POINTER(C.c_double)]),
        "pcgpu_resident_stats": (C.c_int, [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "pcgpu_speculation_stats": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                              C.POINTER(C.c_int64)]),
        "pcgpu_bind_power_field": (C.c_int, [vp, vp]),
        "pcgpu_radial_half_step": (C.c_int, [vp, vp, C.c_double, C.c_double, vp,
                                             C.POINTER(Outcome)]),
        "pcgpu_axial_half_step": (C.c_int, [vp, vp, C.c_double, C.c_double, vp,
                                            C.POINTER(Outcome)]),
        "pcgpu_step": (C.c_int, [vp, vp, C.c_double, C.POINTER(StepResultC)]),
        "pcgpu_step_host": (C.c_int, [vp, vp, C.c_double, C.POINTER(StepResultC)]),
        "pcgpu_radial_half_step_host": (C.c_int, [vp, vp, C.c_double, C.c_double, vp,
                                                  C.POINTER(Outcome)]),
        "pcgpu_axial_half_step_host": (C.c_int, [vp, vp, C.c_double, C.c_double, vp,
                                                 C.POINTER(Outcome)]),
        "pcgpu_run": (C.c_int, [vp, vp, C.c_double, C.c_int32, C.POINTER(StepResultC),
                                C.POINTER(RunStats)]),
        "pcgpu_clamp_events": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
        "pcgpu_run_growth": (C.c_int, [vp, vp, C.c_double, C.c_double, C.c_int32, C.c_double,
                                       C.c_double, C.c_int32, C.c_double,
                                       C.POINTER(StepResultC), C.POINTER(RunStats)]),
        "pcgpu_stream": (vp, [vp]),
        "pcgpu_kernel_timing": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
        "pcgpu_enable_kernel_timing": (C.c_int, [vp, C.c_int32]),
        "pcgpu_launch_count": (C.c_int64, [vp]),
        "pcgpu_describe": (C.c_int32, [vp, C.c_char_p, C.c_int32]),
        "pcgpu_evolve": (C.c_int, [vp, vp, vp, STEP_CB, SNAP_CB, vp, vp]),
        "pcgpu_detector_periods": (C.c_int, [vp, vp, C.c_int32]),
        "pcgpu_evolve_host": (C.c_int, [vp, vp, vp, STEP_CB, SNAP_CB, vp, vp]),
        "pcgpu_writer_create": (C.c_int, [C.POINTER(Desc), vp, C.c_int32, C.POINTER(vp)]),
        "pcgpu_writer_destroy": (None, [vp]),
        "pcgpu_writer_submit": (C.c_int, [vp, vp, vp, C.c_char_p, C.c_int32, C.c_char_p]),
        "pcgpu_writer_flush": (C.c_int, [vp, C.POINTER(C.c_int64)]),
        "pcgpu_writer_last_error": (C.c_char_p, [vp]),
        "pcgpu_tridiag_batch": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, C.c_int64, C.c_int32,
                                          C.c_int32, vp, C.POINTER(C.c_int64)]),
        "pcgpu_nccl_unique_id": (C.c_int, [vp]),
        "pcgpu_dist_create": (C.c_int, [C.POINTER(Desc), C.c_int32, C.c_int32, vp,
                                        C.POINTER(vp)]),
        "pcgpu_dist_destroy": (None, [vp]),
        "pcgpu_dist_last_error": (C.c_char_p, [vp]),
        "pcgpu_dist_plan": (C.c_int, [C.POINTER(Desc), C.c_int32, C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32)]),
        "pcgpu_dist_slabs": (C.c_int, [vp] + [C.POINTER(C.c_int32)] * 4),
        "pcgpu_dist_set_field": (C.c_int, [vp, vp]),
        "pcgpu_dist_get_field": (C.c_int, [vp, vp]),
        "pcgpu_dist_set_field_host": (C.c_int, [vp, vp]),
        "pcgpu_pipeline_stats": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "pcgpu_dist_get_field_host": (C.c_int, [vp, vp]),
        "pcgpu_dist_run": (C.c_int, [vp, C.c_double, C.c_int32, C.POINTER(StepResultC),
                                     C.POINTER(RunStats)]),
        "pcgpu_dist_stream": (vp, [vp]),
        "pcgpu_dist_launch_count": (C.c_int64, [vp]),
        "pcgpu_dist_transport": (C.c_int32, [vp]),
        "pcgpu_dist_ipc_export": (C.c_int, [vp, vp]),
        "pcgpu_dist_ipc_import": (C.c_int, [vp, vp]),
        "pcgpu_dist_peer_off": (C.c_int, [vp]),
        "pcgpu_dist_enable_timing": (C.c_int, [vp, C.c_int32]),
        "pcgpu_dist_timing": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    if lib.pcgpu_abi_version() != PCGPU_ABI_VERSION:
        raise RuntimeError("libpcgpu.so ABI version mismatch")
    _lib = lib
    return lib
