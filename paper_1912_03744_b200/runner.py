"""Host mirror of pulsecell's runner (proj/include/pulsecell/runner.hpp) over
the device-resident runner pcgpu_evolve.

Same names and semantics as the reference: RegimeDetectorConfig, ProbeSpec,
TraceEntry, StopReason, RunnerConfig, Snapshot, EvolutionResult,
probe_cell / probe_value (runner.cpp:20-33) and evolve (runner.cpp:97-190).
The field stays on the device; each step returns only the probe values, and
snapshots are copied to host arrays when they occur.
"""
from __future__ import annotations

import bisect
import ctypes as C
import enum
from dataclasses import dataclass, field as dc_field
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N
from .errors import ConfigError
from .geometry import Grid


@dataclass
class RegimeDetectorConfig:  # runner.hpp:12-23
    samples_per_period: int = 64
    tolerance: float = 1e-3
    min_periods: int = 2

    def validate(self) -> None:
        if self.samples_per_period < 1:
            raise ConfigError("detector.samples_per_period: must be >= 1")
        if not self.tolerance > 0:
            raise ConfigError("detector.tolerance: must be > 0")
        if self.min_periods < 1:
            raise ConfigError("detector.min_periods: must be >= 1")


@dataclass
class ProbeSpec:  # runner.hpp:25-27
    r: float = 0.0
    z: float = 0.0


@dataclass
class TraceEntry:  # runner.hpp:29-33
    t: float
    tau: float
    values: List[float]


class StopReason(enum.IntEnum):  # runner.hpp:35
    ReachedTime = 0
    PeriodicRegime = 1
    TauFloor = 2


@dataclass
class RunnerConfig:  # runner.hpp:93-103
    t_end: float = 1.0
    detector: RegimeDetectorConfig = dc_field(default_factory=RegimeDetectorConfig)
    probes: List[ProbeSpec] = dc_field(default_factory=list)
    snapshot_times: List[float] = dc_field(default_factory=list)
    snapshot_pre_on: bool = True
    snapshot_post_off: bool = True

    def validate(self) -> None:
        if not self.t_end > 0:
            raise ConfigError("runner.t_end: must be > 0")
        self.detector.validate()
        for ts in self.snapshot_times:
            if ts < 0:
                raise ConfigError("runner.snapshot_times: must be >= 0")


@dataclass
class Snapshot:  # runner.hpp:106-109
    t: float
    field: Optional[np.ndarray]
    path: Optional[str] = None  # set when the snapshot went to a SnapshotWriter instead


@dataclass
class EvolutionResult:  # runner.hpp:111-122
    field: object = None
    t: float = 0.0
    steps: int = 0
    reason: StopReason = StopReason.ReachedTime
    trace: List[TraceEntry] = dc_field(default_factory=list)
    pre_on: Optional[Snapshot] = None
    post_off: Optional[Snapshot] = None
    at_times: List[Snapshot] = dc_field(default_factory=list)
    detector_periods: List[np.ndarray] = dc_field(default_factory=list)
    fire_t: float = -1.0
    error: str = ""


def _nearest_index(centers: List[float], x: float) -> int:  # runner.cpp:10-16
    hi = bisect.bisect_left(centers, x)
    if hi == 0:
        return 0
    if hi == len(centers):
        return len(centers) - 1
    return hi - 1 if (x - centers[hi - 1] <= centers[hi] - x) else hi


def probe_cell(grid: Grid, r: float, z: float) -> Tuple[int, int]:  # runner.cpp:20-28
    rc = [grid.r_center(i) for i in range(grid.nr())]
    zc = [grid.z_center(j) for j in range(grid.nz())]
    i, j = _nearest_index(rc, r), _nearest_index(zc, z)
    if not grid.in_mask(i, j):
        raise ConfigError(f"probe location ({r}, {z}) falls outside the domain")
    return i, j


def probe_value(grid: Grid, fld: np.ndarray, r: float, z: float) -> float:
    i, j = probe_cell(grid, r, z)
    return float(fld[i, j])


class RunnerCfgC(C.Structure):
    _fields_ = [("t_end", C.c_double), ("n_probes", C.c_int32),
                ("probe_i", C.POINTER(C.c_int32)), ("probe_j", C.POINTER(C.c_int32)),
                ("n_snapshot_times", C.c_int32), ("snapshot_times", C.POINTER(C.c_double)),
                ("snapshot_pre_on", C.c_int32), ("snapshot_post_off", C.c_int32),
                ("detector_samples_per_period", C.c_int32), ("detector_min_periods", C.c_int32),
                ("detector_tolerance", C.c_double), ("source_on", C.c_int32),
                # NULL: the library's restatement of RegimeDetector (runner.cpp:35-95)
                ("detect", C.c_void_p), ("detect_user", C.c_void_p)]


class EvolveResultC(C.Structure):
    _fields_ = [("t", C.c_double), ("steps", C.c_int64), ("reason", C.c_int32),
                ("fire_t", C.c_double), ("detector_periods", C.c_int32)]




def evolve(stepper, timing, initial, t_end: float, cfg: RunnerConfig, writer=None,
           snapshot_file=None) -> EvolutionResult:
    """pulsecell::evolve (runner.cpp:97-190) on an AdiStepper of this package.
    `initial` is a torch CUDA field (column-major (nr, nz)); it is advanced in
    place and returned as result.field.

    With a snapshot_io.SnapshotWriter and snapshot_file(kind, t, index) ->
    (path, SnapshotFormat, header) or None, snapshots are written to files off
    the critical path (the device field goes to the writer; no host copy on
    the stepping thread) and the result's Snapshots carry the path."""
    import torch
    cfg.validate()
    grid = stepper.grid()
    cells = [probe_cell(grid, p.r, p.z) for p in cfg.probes]
    pi = (C.c_int32 * max(1, len(cells)))(*[c[0] for c in cells])
    pj = (C.c_int32 * max(1, len(cells)))(*[c[1] for c in cells])
    times = (C.c_double * max(1, len(cfg.snapshot_times)))(*cfg.snapshot_times)
    c = RunnerCfgC(t_end, len(cells), pi, pj, len(cfg.snapshot_times), times,
                   1 if cfg.snapshot_pre_on else 0, 1 if cfg.snapshot_post_off else 0,
                   cfg.detector.samples_per_period, cfg.detector.min_periods,
                   cfg.detector.tolerance, 1 if timing.I0 > 0 else 0)
    res = EvolutionResult(field=initial)
    nr, nz = grid.nr(), grid.nz()
    dev = initial.device

    def host_copy(ptr: int) -> np.ndarray:
        # the library synchronised its stream before the callback
        flat = _view(ptr, nr * nz, dev).cpu().numpy()
        return flat.reshape(nz, nr).T.copy(order="F")

    errors: List[BaseException] = []  # exceptions cannot cross the C callback

    def on_step(_u, step, t, tau, vals):
        try:
            res.trace.append(TraceEntry(t, tau, [vals[k] for k in range(len(cells))]))
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    counts = [0, 0, 0]

    def on_snap(_u, kind, t, ptr):
        try:
            target = snapshot_file(kind, t, counts[kind]) if (writer and snapshot_file) else None
            counts[kind] += 1
            if target is not None:
                path, fmt, header = target
                writer.submit(ptr, path, fmt, header)
                snap = Snapshot(t, None, path)
            else:
                snap = Snapshot(t, host_copy(ptr))
            if kind == N.SNAP_PRE_ON:
                res.pre_on = snap
            elif kind == N.SNAP_POST_OFF:
                res.post_off = snap
            else:
                res.at_times.append(snap)
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    step_cb, snap_cb = N.STEP_CB(on_step), N.SNAP_CB(on_snap)
    out = EvolveResultC()
    rc = stepper._lib.pcgpu_evolve(stepper._h, C.c_void_p(stepper._field(initial, True)[0]),
                                   C.byref(c), step_cb, snap_cb, None, C.byref(out))
    stepper._check(rc)
    if errors:
        raise errors[0]
    res.t, res.steps, res.fire_t = out.t, int(out.steps), out.fire_t
    res.reason = StopReason(out.reason)
    if res.reason == StopReason.TauFloor:
        res.error = stepper._lib.pcgpu_last_error(stepper._h).decode()
    if out.detector_periods > 0:
        s = cfg.detector.samples_per_period
        buf = (C.c_double * (out.detector_periods * s))()
        stepper._lib.pcgpu_detector_periods(stepper._h, buf, out.detector_periods)
        arr = np.frombuffer(buf, dtype=np.float64).reshape(out.detector_periods, s)
        res.detector_periods = [arr[k].copy() for k in range(out.detector_periods)]
    return res


def _view(ptr: int, n: int, dev):
    """A torch tensor over n float64 at a raw device pointer (no copy)."""
    import torch

    class _Holder:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_Holder(), device=dev)
