"""B200 AdiStepper -- the drop-in for pulsecell::AdiStepper (solver.hpp:66-106).

Same constructor arguments, method names, argument meaning and error
behaviour as the reference; the work happens in libpcgpu.so (hand-written
sm_100a FP64 kernels) through the C-ABI of include/pcgpu.h. The reference's
LinePool argument becomes a DevicePlan (which GPU).

Fields are float64 (nr, nz) arrays in the reference's column-major Array2
layout: numpy arrays with order='F' (host; copied through the *_host entry
points) or torch CUDA tensors whose memory is column-major, e.g.
``torch.empty(nz, nr, dtype=torch.float64, device='cuda').t()`` (device; zero copy).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N
from .desc import build_desc
from .errors import ConfigError, DeviceError, LineError, TableRangeError, TauFloorError
from .geometry import Grid
from .materials import HalfPointRule, LayerMaterials, RangePolicy
from .source import FieldSource, SourceModel, SourceSpec


@dataclass
class SolverConfig:
    """solver.hpp:12-31 (same defaults)."""
    epsilon: float = 1e-6
    max_iter: int = 10
    tau_min: float = -1.0
    tau_transient_divisor: float = 1000.0
    tau_source_divisor: float = 100.0
    halfpoint_rule: HalfPointRule = HalfPointRule.MeanTemperature
    range_policy: RangePolicy = RangePolicy.Clamp
    all_neumann: bool = False
    T0: float = 4.2
    t_ceiling: float = 300.0

    def validate(self) -> None:  # solver.cpp:33-42
        if not self.epsilon > 0:
            raise ConfigError("solver.epsilon: must be > 0")
        if self.max_iter < 1:
            raise ConfigError("solver.max_iter: must be >= 1")
        if not self.tau_transient_divisor > 0:
            raise ConfigError("solver.tau_transient_divisor: must be > 0")
        if not self.tau_source_divisor > 0:
            raise ConfigError("solver.tau_source_divisor: must be > 0")
        if not self.T0 > 0:
            raise ConfigError("solver.T0: must be > 0")
        if not self.t_ceiling > self.T0:
            raise ConfigError("solver.t_ceiling: must exceed T0")

    def effective_tau_min(self, t_per: float) -> float:
        return self.tau_min if self.tau_min > 0 else 1e-12 * t_per


def initial_tau(t: float, source: SourceSpec, cfg: SolverConfig) -> float:
    """solver.cpp:44-51."""
    import math
    phase = math.fmod(t, source.t_per)
    in_transient = phase <= source.t_trs or (source.t_src <= phase <= source.t_src + source.t_trs)
    return (source.t_trs / cfg.tau_transient_divisor if in_transient
            else source.t_src / cfg.tau_source_divisor)


def make_field(grid: Grid, value: float) -> np.ndarray:
    """solver.cpp:121-123: constant nr x nz field, column-major."""
    return np.full((grid.nr(), grid.nz()), value, dtype=np.float64, order="F")


@dataclass
class GrowthPolicy:
    """BASELINE.json adaptive dt (configs[2], configs[4]): start at 1e-5 s, halve
    when Picard does not converge within max_iter (the reference's own halving,
    solver.cpp:369-371), grow x1.2 after 5 easy steps (accepted without
    halving), cap at 1e-3 s. Not in the reference; the same
    policy runs in the CPU oracle (oracle_run_growth)."""
    tau_start: float = 1e-5
    grow: float = 1.2
    easy_steps: int = 5
    tau_max: float = 1e-3


@dataclass
class HalfStepOutcome:  # solver.hpp:50-54
    converged: bool = False
    iterations: int = 0
    last_delta: float = 0.0


@dataclass
class StepResult:  # solver.hpp:56-60
    tau_used: float = 0.0
    halvings: int = 0
    radial: HalfStepOutcome = field(default_factory=HalfStepOutcome)
    axial: HalfStepOutcome = field(default_factory=HalfStepOutcome)


@dataclass
class DevicePlan:
    """Replaces the reference's ExecPlan/LinePool: which GPU. The kernels are
    bit-identical to the reference ("exact", the only mode)."""
    device: int = 0
    mode: str = "exact"

    def mode_id(self) -> int:
        if self.mode != "exact":
            raise ConfigError(f"exec.mode: unknown mode {self.mode!r} (only 'exact' exists)")
        return N.MODE_EXACT


def _outcome(o: N.Outcome) -> HalfStepOutcome:
    return HalfStepOutcome(bool(o.converged), int(o.iterations), float(o.last_delta))


def _step_result(r: N.StepResultC) -> StepResult:
    return StepResult(float(r.tau_used), int(r.halvings), _outcome(r.radial), _outcome(r.axial))


class AdiStepper:
    """ADI stepper with Picard iteration and tau halving on the GPU."""

    def __init__(self, grid: Grid, mats: LayerMaterials, source: SourceModel,
                 timing: SourceSpec, cfg: SolverConfig, plan: Optional[DevicePlan] = None):
        self._lib = N.load()
        self._grid, self._mats, self._source = grid, list(mats), source
        self._timing, self._cfg = timing, cfg
        self._plan = plan or DevicePlan()
        cfg.validate()  # solver.cpp:133
        timing.validate()  # solver.cpp:134
        if len(self._mats) != grid.domain().layer_count():
            raise ConfigError("stepper: one material required per layer")
        if any(m is None for m in self._mats):
            raise ConfigError("stepper: null material")
        desc, self._keep = build_desc(grid, self._mats, source, timing, cfg,
                                      self._plan.mode_id(), self._plan.device)
        h = C.c_void_p()
        rc = self._lib.pcgpu_create(C.byref(desc), C.byref(h))
        if rc != N.OK:
            msg = self._lib.pcgpu_last_error(None).decode()
            if rc == N.ERR_CONFIG:
                raise ConfigError(msg)
            raise DeviceError(f"pcgpu_create failed ({rc}): {msg}")
        self._h = h
        self._nr, self._nz = grid.nr(), grid.nz()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.pcgpu_destroy(h)
            self._h = None

    # -- accessors (solver.hpp:84-85) --
    def config(self) -> SolverConfig:
        return self._cfg

    def grid(self) -> Grid:
        return self._grid

    def handle(self) -> C.c_void_p:
        return self._h

    def mode(self) -> str:
        return self._plan.mode

    # -- error mapping (errors.hpp) --
    def _check(self, rc: int) -> None:
        if rc == N.OK:
            return
        msg = self._lib.pcgpu_last_error(self._h).decode()
        line = int(self._lib.pcgpu_error_line(self._h))
        if rc == N.ERR_TAU_FLOOR:
            tau, floor, t = C.c_double(), C.c_double(), C.c_double()
            self._lib.pcgpu_last_tau_floor(self._h, C.byref(tau), C.byref(floor), C.byref(t))
            raise TauFloorError(msg, tau.value, floor.value, t.value)
        if rc == N.ERR_TABLE_RANGE:
            raise LineError(line, msg, TableRangeError)
        if rc == N.ERR_ZERO_PIVOT:
            raise LineError(line, msg)
        if rc == N.ERR_CONFIG:
            raise ConfigError(msg)
        raise DeviceError(f"pcgpu error {rc}: {msg}")

    def _field(self, a, writable: bool) -> Tuple[int, bool]:
        """(pointer, is_device) for a column-major nr x nz float64 field."""
        nr, nz = self._nr, self._nz
        if isinstance(a, np.ndarray):
            if a.dtype != np.float64 or a.shape != (nr, nz) or not a.flags.f_contiguous:
                raise ValueError("field must be a float64 (nr, nz) Fortran-ordered array")
            if writable and not a.flags.writeable:
                raise ValueError("output field is read-only")
            return a.ctypes.data, False
        try:
            import torch
        except ImportError:  # pragma: no cover
            raise TypeError("field must be a numpy array or a torch CUDA tensor")
        if isinstance(a, torch.Tensor):
            if not a.is_cuda or a.dtype != torch.float64 or tuple(a.shape) != (nr, nz) \
                    or a.stride() != (1, nr):
                raise ValueError("device field must be a CUDA float64 (nr, nz) tensor with "
                                 "column-major strides (1, nr)")
            return a.data_ptr(), True
        raise TypeError("field must be a numpy array or a torch CUDA tensor")

    def _bind_source(self, t: float, tau: float) -> None:
        if isinstance(self._source, FieldSource):
            self._source.bind_time(t + 0.5 * tau)
            p = np.asfortranarray(self._source.power_field(self._grid, t + 0.5 * tau),
                                  dtype=np.float64)
            import torch
            dev = torch.from_numpy(p.T.copy()).to(f"cuda:{self._plan.device}")
            torch.cuda.synchronize()
            self._check(self._lib.pcgpu_bind_power_field(self._h, C.c_void_p(dev.data_ptr())))
            self._pow_keep = dev
        else:
            self._source.bind_time(t + 0.5 * tau)

    def _half(self, radial: bool, src, t: float, tau: float, out) -> HalfStepOutcome:
        ps, ds = self._field(src, False)
        po, do = self._field(out, True)
        if ds != do:
            raise ValueError("input and output fields must both be host or both be device")
        if ps == po:
            raise ValueError("out must not alias the input field")  # solver.cpp:237, :336
        self._bind_source(t, tau)
        o = N.Outcome()
        if ds:
            f = self._lib.pcgpu_radial_half_step if radial else self._lib.pcgpu_axial_half_step
        else:
            f = (self._lib.pcgpu_radial_half_step_host if radial
                 else self._lib.pcgpu_axial_half_step_host)
        self._check(f(self._h, C.c_void_p(ps), t, tau, C.c_void_p(po), C.byref(o)))
        return _outcome(o)

    def radial_half_step(self, T_cur, t: float, tau: float, out) -> HalfStepOutcome:
        """Implicit-in-r half-step (solver.hpp:70-74)."""
        return self._half(True, T_cur, t, tau, out)

    def axial_half_step(self, T_half, t: float, tau: float, out) -> HalfStepOutcome:
        """Implicit-in-z half-step (solver.hpp:76-78)."""
        return self._half(False, T_half, t, tau, out)

    def step(self, fld, t: float) -> StepResult:
        """One accepted step with tau halving (solver.hpp:80-82); fld updated in place."""
        p, dev = self._field(fld, True)
        r = N.StepResultC()
        f = self._lib.pcgpu_step if dev else self._lib.pcgpu_step_host
        self._check(f(self._h, C.c_void_p(p), t, C.byref(r)))
        return _step_result(r)

    def run(self, fld, t0: float, nsteps: int, keep_results: bool = False):
        """nsteps x step() with t += tau_used, field resident on the device
        (bench.cpp:20-22 loop). Returns (t_end, stats dict, [StepResult])."""
        p, dev = self._field(fld, True)
        if not dev:
            raise ValueError("run() takes a device field (torch CUDA tensor)")
        res = (N.StepResultC * nsteps)() if keep_results and nsteps > 0 else None
        st = N.RunStats()
        rc = self._lib.pcgpu_run(self._h, C.c_void_p(p), t0, int(nsteps), res, C.byref(st))
        stats = {k: getattr(st, k) for k, _ in N.RunStats._fields_}
        self._check(rc)
        results = [_step_result(r) for r in res] if res is not None else []
        return float(st.t_end), stats, results

    def run_growth(self, fld, t0: float, t_end: float, max_steps: int,
                   policy: Optional["GrowthPolicy"] = None, keep_results: bool = False):
        """Run under the BASELINE growth policy (device field); returns
        (t_end, stats, [StepResult])."""
        pol = policy or GrowthPolicy()
        p, dev = self._field(fld, True)
        if not dev:
            raise ValueError("run_growth() takes a device field (torch CUDA tensor)")
        res = (N.StepResultC * max_steps)() if keep_results and max_steps > 0 else None
        st = N.RunStats()
        rc = self._lib.pcgpu_run_growth(self._h, C.c_void_p(p), t0, t_end, int(max_steps),
                                        pol.tau_start, pol.grow, int(pol.easy_steps),
                                        pol.tau_max, res, C.byref(st))
        stats = {k: getattr(st, k) for k, _ in N.RunStats._fields_}
        self._check(rc)
        n = int(st.steps)
        results = [_step_result(res[k]) for k in range(n)] if res is not None else []
        return float(st.t_end), stats, results

    def clamp_events(self) -> List[int]:
        """MaterialTable::clamp_events() per layer (materials.hpp:85)."""
        n = len(self._mats)
        arr = (C.c_uint64 * n)()
        self._check(self._lib.pcgpu_clamp_events(self._h, arr))
        return [int(v) for v in arr]

    def initial_tau(self, t: float) -> float:
        return float(self._lib.pcgpu_initial_tau(self._h, t))

    def pulse_value(self, t: float) -> float:
        return float(self._lib.pcgpu_pulse_value(self._h, t))

    def stream(self) -> int:
        return int(self._lib.pcgpu_stream(self._h) or 0)

    def enable_kernel_timing(self, on: bool = True) -> None:
        self._lib.pcgpu_enable_kernel_timing(self._h, 1 if on else 0)

    def kernel_timing(self) -> dict:
        rm, am = C.c_double(), C.c_double()
        rl, al = C.c_int64(), C.c_int64()
        self._lib.pcgpu_kernel_timing(self._h, C.byref(rm), C.byref(rl), C.byref(am),
                                      C.byref(al))
        return {"radial_ms": rm.value, "radial_launches": rl.value, "axial_ms": am.value,
                "axial_launches": al.value}

    def pipeline_stats(self) -> dict:
        """Host-field steps that overlapped the copy-in with the radial sweep,
        and how many of them redid the radial half-step (pcgpu_pipeline_stats)."""
        a, b = C.c_int64(), C.c_int64()
        self._check(self._lib.pcgpu_pipeline_stats(self._h, C.byref(a), C.byref(b)))
        return {"steps": a.value, "fallbacks": b.value}

    def launch_count(self) -> int:
        return int(self._lib.pcgpu_launch_count(self._h))

    def speculation_stats(self) -> dict:
        """Host-driven runs (pcgpu_speculation_stats): speculative batches,
        the steps they accepted, batches undone and replayed."""
        b, s, r = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self._lib.pcgpu_speculation_stats(self._h, C.byref(b), C.byref(s), C.byref(r)))
        return {"batches": b.value, "steps": s.value, "rollbacks": r.value}

    def resident_stats(self) -> dict:
        """The resident stepper (whole steps in one cooperative launch per
        batch; pcgpu_resident_stats): grid size (0: not used on this grid),
        batches, steps, steps redone host-driven."""
        g = C.c_int32()
        b, s, hs = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self._lib.pcgpu_resident_stats(self._h, C.byref(g), C.byref(b), C.byref(s),
                                                   C.byref(hs)))
        return {"grid": g.value, "batches": b.value, "steps": s.value, "host_steps": hs.value}

    def evolve(self, timing, initial, t_end: float, cfg, writer=None, snapshot_file=None):
        """pulsecell::evolve (runner.cpp:97-190) with the field resident on the
        device; see paper_1912_03744_b200.runner.evolve."""
        from .runner import evolve
        return evolve(self, timing, initial, t_end, cfg, writer, snapshot_file)

    def describe(self) -> str:
        """The kernel variants the library selected for this problem."""
        buf = C.create_string_buffer(256)
        self._lib.pcgpu_describe(self._h, buf, 256)
        return buf.value.decode()
