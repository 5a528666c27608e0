"""Device-resident runner: pcgpu_evolve against the
reference's own pulsecell::evolve (runner.cpp:97-190, compiled unchanged into
oracle/_ref/libpcref.so), bit for bit: the step trace (t, tau, probe values),
stop reason and time, the regime detector's resampled periods and firing
time, and every snapshot (pre turn-on, post turn-off, at requested times)."""
import numpy as np
import pytest

from oracle.oracle import RefStepper, ref_evolve
from paper_1912_03744_b200 import configs
from paper_1912_03744_b200.runner import (ProbeSpec, RegimeDetectorConfig, RunnerConfig,
                                          StopReason, probe_cell)
from paper_1912_03744_b200.solver import make_field

from helpers import gpu_stepper, to_dev, to_host

pytestmark = pytest.mark.gpu


def _cell(I0=0.8, **solver_kw):
    kw = dict(tau_transient_divisor=10.0, tau_source_divisor=20.0)
    kw.update(solver_kw)
    case = configs.step_cell(True, **kw)
    case.timing.I0 = I0
    return case


def _cfg(case, periods, **kw):
    d = case.domain
    cfg = RunnerConfig(
        t_end=periods * case.timing.t_per,
        detector=RegimeDetectorConfig(samples_per_period=16, tolerance=kw.pop("tol", 1e-3),
                                      min_periods=kw.pop("min_periods", 2)),
        probes=[ProbeSpec(0.2, 0.3), ProbeSpec(0.9 * d.layer_radii[-1], 1.0),
                ProbeSpec(0.3, 1.8)],
        snapshot_times=kw.pop("times", [0.0, 0.0105, 0.25]),
        snapshot_pre_on=True, snapshot_post_off=True)
    return cfg


def _run_both(case, cfg, init=None):
    g = case.grid()
    f0 = make_field(g, case.solver.T0) if init is None else init
    ref = RefStepper(case)
    fr = f0.copy(order="F")
    want = ref_evolve(ref, fr, cfg.t_end, cfg, case.timing.I0)
    gpu = gpu_stepper(case, "exact")
    fg = to_dev(f0)
    got = gpu.evolve(case.timing, fg, cfg.t_end, cfg)
    return g, fr, want, to_host(fg), got


def _assert_same(g, fr, want, fg, got):
    m = g.mask()
    assert got.steps == want["steps"] and got.t == want["t"]
    assert int(got.reason) == want["reason"] and got.fire_t == want["fire_t"]
    assert len(got.trace) == want["steps"]
    for e, (t, tau, vals) in zip(got.trace, want["trace"]):
        assert (e.t, e.tau, e.values) == (t, tau, vals)
    for name in ("pre_on", "post_off"):
        a, b = getattr(got, name), want[name]
        assert (a is None) == (b is None)
        if a is not None:
            assert a.t == b[0] and np.array_equal(a.field[m], b[1][m])
    assert len(got.at_times) == len(want["at_times"])
    for a, (t, f) in zip(got.at_times, want["at_times"]):
        assert a.t == t and np.array_equal(a.field[m], f[m])
    assert len(got.detector_periods) == len(want["detector"])
    for a, b in zip(got.detector_periods, want["detector"]):
        assert np.array_equal(a, b)
    assert np.array_equal(fg[m], fr[m])


def test_probe_cells_match_reference(cuda):
    case = _cell()
    cfg = _cfg(case, 0.05)
    g = case.grid()
    want = ref_evolve(RefStepper(case), make_field(g, case.solver.T0), cfg.t_end, cfg,
                      case.timing.I0)
    assert [probe_cell(g, p.r, p.z) for p in cfg.probes] == [tuple(c) for c in want["probe_cells"]]


def test_probe_outside_domain_raises_like_reference(cuda):
    from oracle.oracle import OracleError
    from paper_1912_03744_b200.errors import ConfigError
    case = _cell()
    cfg = _cfg(case, 0.05)
    cfg.probes.append(ProbeSpec(0.65, 1.7))  # layer 1 ends at z = 1.5
    g = case.grid()
    with pytest.raises(OracleError, match="outside the domain"):
        ref_evolve(RefStepper(case), make_field(g, case.solver.T0), cfg.t_end, cfg,
                   case.timing.I0)
    with pytest.raises(ConfigError, match="outside the domain"):
        gpu_stepper(case, "exact").evolve(case.timing, to_dev(make_field(g, case.solver.T0)),
                                          cfg.t_end, cfg)


def test_evolve_powered_detector_and_snapshots_bitwise(cuda):
    """Several pulse periods: pre-on / post-off captures at every period, the
    regime detector over probe 0 (fires or not exactly like the reference)."""
    case = _cell()
    cfg = _cfg(case, 6, tol=5e-2, min_periods=1)
    g, fr, want, fg, got = _run_both(case, cfg)
    assert want["steps"] > 100 and len(want["detector"]) >= 2
    assert want["pre_on"] is not None and want["post_off"] is not None
    _assert_same(g, fr, want, fg, got)


def test_evolve_unpowered_reaches_time_bitwise(cuda):
    """I0 = 0: no regime detection; runs to t_end from a non-uniform field."""
    case = _cell(I0=0.0)
    cfg = _cfg(case, 1.5)
    init = configs.smooth_field(case.grid(), 20.0)
    g, fr, want, fg, got = _run_both(case, cfg, init)
    assert want["reason"] == int(StopReason.ReachedTime) and want["fire_t"] == -1
    _assert_same(g, fr, want, fg, got)


def test_evolve_tau_floor_stop_bitwise(cuda):
    """max_iter = 1 and a high tau floor: the first step that needs halving
    ends the run with TauFloor and the last accepted field."""
    case = _cell(max_iter=1, tau_min=5e-4)
    cfg = _cfg(case, 1)
    init = configs.smooth_field(case.grid(), 20.0)
    g, fr, want, fg, got = _run_both(case, cfg, init)
    assert want["reason"] == int(StopReason.TauFloor)
    assert got.error and want["error"]
    _assert_same(g, fr, want, fg, got)
