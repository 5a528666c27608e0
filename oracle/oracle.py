"""TEST INFRASTRUCTURE ONLY -- ctypes access to the two CPU checkers.

* ``PortStepper``: the plain-C restatement (oracle/adi_oracle.c ->
  oracle/_build/liboracle.so), same pcgpu_desc input as the GPU library.
* ``RefStepper``: the reference's own AdiStepper, compiled unchanged from
  /root/reference/proj/src into oracle/_ref/libpcref.so (ref_bridge.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module; the product path (paper_1912_03744_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List

import numpy as np

from paper_1912_03744_b200 import _native as N
from paper_1912_03744_b200.desc import build_desc
from paper_1912_03744_b200.solver import HalfStepOutcome, StepResult

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libpcref.so")

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class RefSpec(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32), ("layer_radii", _dp), ("radial_divisions", C.POINTER(C.c_int32)),
        ("core_length", C.c_double), ("outer_length", C.c_double),
        ("axial_divisions_core", C.c_int32), ("axial_divisions_outer", C.c_int32),
        ("source_layer", C.c_int32), ("materials", C.POINTER(N.Material)),
        ("source_kind", C.c_int32),
        ("t_per", C.c_double), ("t_src", C.c_double), ("t_trs", C.c_double),
        ("xi", C.c_double), ("zeta", C.c_double), ("I0", C.c_double), ("S_C", C.c_double),
        ("waveform", C.c_int32), ("joule_dimensional", C.c_int32),
        ("epsilon", C.c_double), ("max_iter", C.c_int32), ("tau_min", C.c_double),
        ("tau_transient_divisor", C.c_double), ("tau_source_divisor", C.c_double),
        ("halfpoint_rule", C.c_int32), ("range_policy", C.c_int32), ("all_neumann", C.c_int32),
        ("T0", C.c_double), ("t_ceiling", C.c_double),
        ("workers", C.c_int32), ("chunking", C.c_int32),
    ]


class RefEvolveIO(C.Structure):
    """pcref_evolve_io (oracle/ref_bridge.h)."""
    _fields_ = [
        ("t_end", C.c_double), ("n_probes", C.c_int32), ("probe_r", _dp), ("probe_z", _dp),
        ("n_snapshot_times", C.c_int32), ("snapshot_times", _dp),
        ("snapshot_pre_on", C.c_int32), ("snapshot_post_off", C.c_int32),
        ("detector_samples_per_period", C.c_int32), ("detector_min_periods", C.c_int32),
        ("detector_tolerance", C.c_double), ("I0", C.c_double),
        ("t", C.c_double), ("fire_t", C.c_double), ("steps", C.c_int64), ("reason", C.c_int32),
        ("trace_cap", C.c_int64), ("trace_t", _dp), ("trace_tau", _dp), ("trace_values", _dp),
        ("has_pre_on", C.c_int32), ("has_post_off", C.c_int32),
        ("pre_on_t", C.c_double), ("post_off_t", C.c_double),
        ("pre_on_field", _dp), ("post_off_field", _dp),
        ("at_cap", C.c_int32), ("at_count", C.c_int32), ("at_t", _dp), ("at_fields", _dp),
        ("det_cap", C.c_int32), ("det_rows", C.c_int32), ("det_values", _dp),
        ("probe_i", C.c_int32 * 16), ("probe_j", C.c_int32 * 16),
    ]


_port = None
_ref = None


def port_available() -> bool:
    return os.path.exists(PORT_LIB)


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def _load_port():
    global _port
    if _port is None:
        lib = C.CDLL(PORT_LIB)
        O, S, R = C.POINTER(N.Outcome), C.POINTER(N.StepResultC), C.POINTER(N.RunStats)
        for name, res, args in [
            ("oracle_create", C.c_int, [C.POINTER(N.Desc), C.POINTER(_vp)]),
            ("oracle_destroy", None, [_vp]),
            ("oracle_last_error", C.c_char_p, [_vp]),
            ("oracle_error_line", C.c_int64, [_vp]),
            ("oracle_initial_tau", C.c_double, [_vp, C.c_double]),
            ("oracle_pulse_value", C.c_double, [_vp, C.c_double]),
            ("oracle_bind_power_field", C.c_int, [_vp, _vp]),
            ("oracle_radial_half_step", C.c_int, [_vp, _vp, C.c_double, C.c_double, _vp, O]),
            ("oracle_axial_half_step", C.c_int, [_vp, _vp, C.c_double, C.c_double, _vp, O]),
            ("oracle_step", C.c_int, [_vp, _vp, C.c_double, S]),
            ("oracle_run", C.c_int, [_vp, _vp, C.c_double, C.c_int32, S, R]),
            ("oracle_clamp_events", C.c_int, [_vp, C.POINTER(C.c_uint64)]),
            ("oracle_run_growth", C.c_int, [_vp, _vp, C.c_double, C.c_double, C.c_int32,
                                            C.c_double, C.c_double, C.c_int32, C.c_double, S,
                                            R]),
            ("oracle_thomas", C.c_int, [_vp] * 6 + [C.c_int64]),
            ("oracle_thomas_batch", C.c_int, [_vp] * 5 + [C.c_int64, C.c_int64, C.c_int32,
                                                          C.POINTER(C.c_int64)]),
        ]:
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _port = lib
    return _port


def _load_ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_LIB)
        O, S, R = C.POINTER(N.Outcome), C.POINTER(N.StepResultC), C.POINTER(N.RunStats)
        i64 = C.POINTER(C.c_int64)
        for name, res, args in [
            ("pcref_create", C.c_int, [C.POINTER(RefSpec), C.POINTER(_vp)]),
            ("pcref_destroy", None, [_vp]),
            ("pcref_last_error", C.c_char_p, [_vp]),
            ("pcref_error_line", C.c_int64, [_vp]),
            ("pcref_grid_dims", None, [_vp, i64, i64, i64, i64, i64]),
            ("pcref_grid_arrays", None, [_vp] * 8),
            ("pcref_source_amplitude", C.c_double, [_vp]),
            ("pcref_tau_floor", C.c_double, [_vp]),
            ("pcref_initial_tau", C.c_double, [_vp, C.c_double]),
            ("pcref_pulse_value", C.c_double, [_vp, C.c_double]),
            ("pcref_bind_power_field", C.c_int, [_vp, _vp]),
            ("pcref_radial_half_step", C.c_int, [_vp, _vp, C.c_double, C.c_double, _vp, O]),
            ("pcref_axial_half_step", C.c_int, [_vp, _vp, C.c_double, C.c_double, _vp, O]),
            ("pcref_step", C.c_int, [_vp, _vp, C.c_double, S]),
            ("pcref_run", C.c_int, [_vp, _vp, C.c_double, C.c_int32, S, R]),
            ("pcref_run_growth", C.c_int, [_vp, _vp, C.c_double, C.c_double, C.c_int32,
                                           C.c_double, C.c_double, C.c_int32, C.c_double, S, R]),
            ("pcref_evolve", C.c_int, [_vp, _vp, C.POINTER(RefEvolveIO)]),
            ("pcref_write_snapshot", C.c_int, [_vp, _vp, C.c_char_p, C.c_int32, C.c_char_p]),
            ("pcref_write_trace", C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, C.c_char_p,
                                            C.c_char_p]),
            ("pcref_write_phase_trace", C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_double,
                                                  C.c_char_p, C.c_char_p]),
            ("pcref_clamp_events", C.c_int, [_vp, C.POINTER(C.c_uint64)]),
            ("pcref_apply_lambda_r", C.c_double, [_vp, _vp, C.c_int64, C.c_int64]),
            ("pcref_apply_lambda_z", C.c_double, [_vp, _vp, C.c_int64, C.c_int64]),
            ("pcref_weighted_heat_sum", C.c_double, [_vp, _vp]),
            ("pcref_eval", C.c_int, [_vp, C.c_int32, C.c_int32, C.c_double, _dp]),
            ("pcref_thomas_batch", C.c_int, [_vp] * 5 + [C.c_int64, C.c_int64, C.c_int32,
                                                         C.c_int32, i64]),
        ]:
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _ref = lib
    return _ref


def _outcome(o) -> HalfStepOutcome:
    return HalfStepOutcome(bool(o.converged), int(o.iterations), float(o.last_delta))


def _result(r) -> StepResult:
    return StepResult(float(r.tau_used), int(r.halvings), _outcome(r.radial), _outcome(r.axial))


def _ptr(a: np.ndarray) -> _vp:
    assert a.dtype == np.float64 and a.flags.f_contiguous
    return _vp(a.ctypes.data)


class _Base:
    prefix = ""

    def _call(self, name, *args):
        return getattr(self.lib, self.prefix + name)(self.h, *args)

    def _check(self, rc):
        if rc != N.OK:
            msg = self._call("last_error").decode()
            raise OracleError(rc, msg, int(self._call("error_line")))

    def radial_half_step(self, T_cur, t, tau, out) -> HalfStepOutcome:
        o = N.Outcome()
        self._check(self._call("radial_half_step", _ptr(T_cur), t, tau, _ptr(out), C.byref(o)))
        return _outcome(o)

    def axial_half_step(self, T_half, t, tau, out) -> HalfStepOutcome:
        o = N.Outcome()
        self._check(self._call("axial_half_step", _ptr(T_half), t, tau, _ptr(out), C.byref(o)))
        return _outcome(o)

    def step(self, field, t) -> StepResult:
        r = N.StepResultC()
        self._check(self._call("step", _ptr(field), t, C.byref(r)))
        return _result(r)

    def run(self, field, t0, nsteps):
        res = (N.StepResultC * max(1, nsteps))()
        st = N.RunStats()
        rc = self._call("run", _ptr(field), t0, int(nsteps), res, C.byref(st))
        stats = {k: getattr(st, k) for k, _ in N.RunStats._fields_}
        self._check(rc)
        return float(st.t_end), stats, [_result(res[k]) for k in range(nsteps)]

    def run_growth(self, field, t0, t_end, max_steps, policy=None):
        """The BASELINE growth policy (pcgpu_run_growth's controller): the
        port's oracle_run_growth, or for RefStepper the reference's own
        half-steps under the same controller (pcref_run_growth)."""
        from paper_1912_03744_b200.solver import GrowthPolicy
        pol = policy or GrowthPolicy()
        res = (N.StepResultC * max(1, max_steps))()
        st = N.RunStats()
        rc = self._call("run_growth", _ptr(field), t0, t_end, int(max_steps), pol.tau_start,
                        pol.grow, int(pol.easy_steps), pol.tau_max, res, C.byref(st))
        stats = {k: getattr(st, k) for k, _ in N.RunStats._fields_}
        self._check(rc)
        return float(st.t_end), stats, [_result(res[k]) for k in range(int(st.steps))]

    def clamp_events(self) -> List[int]:
        arr = (C.c_uint64 * self.n_layers)()
        self._check(self._call("clamp_events", arr))
        return [int(v) for v in arr]

    def bind_power_field(self, p: np.ndarray):
        p = np.asfortranarray(p, dtype=np.float64)
        self._check(self._call("bind_power_field", _ptr(p)))

    def initial_tau(self, t):
        return float(self._call("initial_tau", t))

    def pulse_value(self, t):
        return float(self._call("pulse_value", t))


def ref_evolve(ref: "RefStepper", field: np.ndarray, t_end: float, cfg, I0: float,
               trace_cap: int = 200000, at_cap: int = 16, det_cap: int = 4096):
    """pulsecell::evolve of the reference itself (runner.cpp:97-190). Returns a
    dict: field (in place), t, steps, reason, fire_t, trace (t, tau, values),
    pre_on / post_off (t, field) or None, at_times [(t, field)], detector rows,
    and the probe cells the reference chose."""
    nr, nz = field.shape
    cells = nr * nz
    npr = len(cfg.probes)
    pr = np.array([p.r for p in cfg.probes] or [0.0])
    pz = np.array([p.z for p in cfg.probes] or [0.0])
    st = np.array(cfg.snapshot_times or [0.0])
    tt, ttau = np.zeros(trace_cap), np.zeros(trace_cap)
    tv = np.zeros(trace_cap * max(1, npr))
    pre, post = np.zeros(cells), np.zeros(cells)
    at_t, at_f = np.zeros(at_cap), np.zeros(at_cap * cells)
    s = cfg.detector.samples_per_period
    dv = np.zeros(det_cap * s)
    io = RefEvolveIO()
    io.t_end, io.n_probes = t_end, npr
    io.probe_r, io.probe_z = pr.ctypes.data_as(_dp), pz.ctypes.data_as(_dp)
    io.n_snapshot_times, io.snapshot_times = len(cfg.snapshot_times), st.ctypes.data_as(_dp)
    io.snapshot_pre_on, io.snapshot_post_off = int(cfg.snapshot_pre_on), int(cfg.snapshot_post_off)
    io.detector_samples_per_period, io.detector_min_periods = s, cfg.detector.min_periods
    io.detector_tolerance, io.I0 = cfg.detector.tolerance, I0
    io.trace_cap = trace_cap
    io.trace_t, io.trace_tau, io.trace_values = (a.ctypes.data_as(_dp) for a in (tt, ttau, tv))
    io.pre_on_field, io.post_off_field = pre.ctypes.data_as(_dp), post.ctypes.data_as(_dp)
    io.at_cap, io.at_t, io.at_fields = at_cap, at_t.ctypes.data_as(_dp), at_f.ctypes.data_as(_dp)
    io.det_cap, io.det_values = det_cap, dv.ctypes.data_as(_dp)
    ref._check(ref.lib.pcref_evolve(ref.h, _ptr(field), C.byref(io)))
    n = int(io.steps)
    assert n <= trace_cap
    shape = (nr, nz)
    return {
        "t": io.t, "steps": n, "reason": int(io.reason), "fire_t": io.fire_t,
        "trace": [(tt[k], ttau[k], list(tv[k * npr:(k + 1) * npr])) for k in range(n)],
        "pre_on": (io.pre_on_t, pre.reshape(shape, order="F")) if io.has_pre_on else None,
        "post_off": (io.post_off_t, post.reshape(shape, order="F")) if io.has_post_off else None,
        "at_times": [(at_t[k], at_f[k * cells:(k + 1) * cells].reshape(shape, order="F"))
                     for k in range(min(io.at_count, at_cap))],
        "detector": [dv[k * s:(k + 1) * s].copy() for k in range(min(io.det_rows, det_cap))],
        "probe_cells": [(io.probe_i[k], io.probe_j[k]) for k in range(min(npr, 16))],
        "error": ref.lib.pcref_last_error(ref.h).decode() if io.reason == 2 else "",
    }


class OracleError(RuntimeError):
    def __init__(self, code, msg, line=-1):
        super().__init__(f"[{code}] {msg}")
        self.code, self.line = code, line


class PortStepper(_Base):
    """The C restatement, driven by the same descriptor as the GPU library."""
    prefix = "oracle_"

    def __init__(self, case, source_kind=None, explicit_extents=False):
        from paper_1912_03744_b200.source import FieldSource, JouleSource, NullSource
        self.lib = _load_port()
        grid = case.grid()
        kind = case.source_kind if source_kind is None else source_kind
        src = _source_for(case, grid, kind)
        desc, self._keep = build_desc(grid, case.materials, src, case.timing, case.solver,
                                      explicit_extents=explicit_extents)
        h = _vp()
        rc = self.lib.oracle_create(C.byref(desc), C.byref(h))
        if rc != N.OK:
            raise OracleError(rc, "oracle_create failed")
        self.h = h
        self.n_layers = len(case.materials)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.oracle_destroy(self.h)
            self.h = None


def _source_for(case, grid, kind):
    from paper_1912_03744_b200.source import FieldSource, JouleSource, NullSource
    if kind == N.SOURCE_JOULE:
        d = case.domain
        return JouleSource(case.timing, d.source_layer, case.materials[d.source_layer],
                           case.solver.range_policy)
    if kind == N.SOURCE_FIELD:
        return FieldSource(grid)
    return NullSource()


class RefStepper(_Base):
    """The reference's own AdiStepper (compiled from /root/reference sources)."""
    prefix = "pcref_"

    def __init__(self, case, workers: int = 1, chunking: int = 0, source_kind=None):
        self.lib = _load_ref()
        d, g, ts, cfg = case.domain, case.gridspec, case.timing, case.solver
        keep = []
        radii = np.asarray(d.layer_radii, dtype=np.float64)
        divs = np.asarray(g.radial_divisions, dtype=np.int32)
        keep += [radii, divs]
        m_arr = (N.Material * len(case.materials))()
        from paper_1912_03744_b200.desc import _table
        for k, m in enumerate(case.materials):
            m_arr[k] = N.Material(m.rho(), _table(m.cv, keep), _table(m.lam, keep),
                                  _table(m.chi, keep))
        keep.append(m_arr)
        s = RefSpec()
        s.n_layers = len(d.layer_radii)
        s.layer_radii = radii.ctypes.data_as(_dp)
        s.radial_divisions = divs.ctypes.data_as(C.POINTER(C.c_int32))
        s.core_length, s.outer_length = d.core_length, d.outer_length
        s.axial_divisions_core, s.axial_divisions_outer = g.axial_divisions_core, g.axial_divisions_outer
        s.source_layer = d.source_layer
        s.materials = C.cast(m_arr, C.POINTER(N.Material))
        s.source_kind = case.source_kind if source_kind is None else source_kind
        s.t_per, s.t_src, s.t_trs, s.xi, s.zeta = ts.t_per, ts.t_src, ts.t_trs, ts.xi, ts.zeta
        s.I0, s.S_C, s.waveform = ts.I0, ts.S_C, int(ts.waveform)
        s.joule_dimensional = 1 if ts.joule_dimensional else 0
        s.epsilon, s.max_iter, s.tau_min = cfg.epsilon, cfg.max_iter, cfg.tau_min
        s.tau_transient_divisor, s.tau_source_divisor = cfg.tau_transient_divisor, cfg.tau_source_divisor
        s.halfpoint_rule, s.range_policy = int(cfg.halfpoint_rule), int(cfg.range_policy)
        s.all_neumann = 1 if cfg.all_neumann else 0
        s.T0, s.t_ceiling = cfg.T0, cfg.t_ceiling
        s.workers, s.chunking = workers, chunking
        self._keep = keep
        h = _vp()
        rc = self.lib.pcref_create(C.byref(s), C.byref(h))
        if rc != N.OK:
            raise OracleError(rc, self.lib.pcref_last_error(None).decode())
        self.h = h
        self.n_layers = len(case.materials)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.pcref_destroy(self.h)
            self.h = None

    def grid_arrays(self):
        nr, nz, nrc, nzs, act = (C.c_int64() for _ in range(5))
        self.lib.pcref_grid_dims(self.h, *(C.byref(v) for v in (nr, nz, nrc, nzs, act)))
        nr, nz = nr.value, nz.value
        out = dict(r_center=np.zeros(nr), width_r=np.zeros(nr), gap_r=np.zeros(nr + 1),
                   z_center=np.zeros(nz), width_z=np.zeros(nz), gap_z=np.zeros(nz + 1),
                   layer=np.zeros(nr, dtype=np.int32))
        self.lib.pcref_grid_arrays(self.h, *(_vp(out[k].ctypes.data) for k in
                                             ("r_center", "width_r", "gap_r", "z_center",
                                              "width_z", "gap_z", "layer")))
        out.update(nr=nr, nz=nz, nr_core=nrc.value, nz_shared=nzs.value, active=act.value)
        return out

    def source_amplitude(self):
        return float(self.lib.pcref_source_amplitude(self.h))

    def weighted_heat_sum(self, field):
        return float(self.lib.pcref_weighted_heat_sum(self.h, _ptr(field)))

    def apply_lambda_r(self, field, i, j):
        return float(self.lib.pcref_apply_lambda_r(self.h, _ptr(field), i, j))

    def apply_lambda_z(self, field, i, j):
        return float(self.lib.pcref_apply_lambda_z(self.h, _ptr(field), i, j))


def port_thomas_batch(a, b, c, d, n, batch, layout):
    lib = _load_port()
    x = np.zeros_like(d)
    failed = C.c_int64(-1)
    rc = lib.oracle_thomas_batch(*(_vp(v.ctypes.data) for v in (a, b, c, d, x)), n, batch, layout,
                                 C.byref(failed))
    return rc, x, failed.value


def ref_thomas_batch(a, b, c, d, n, batch, layout, workers=1):
    lib = _load_ref()
    x = np.zeros_like(d)
    failed = C.c_int64(-1)
    rc = lib.pcref_thomas_batch(*(_vp(v.ctypes.data) for v in (a, b, c, d, x)), n, batch, layout,
                                workers, C.byref(failed))
    return rc, x, failed.value
