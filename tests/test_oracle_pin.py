"""Pin the C restatement (oracle/adi_oracle.c) to the reference itself.

The reference library (oracle/_ref/libpcref.so) is compiled from the
reference's own sources; both run the same cases and must agree bit-for-bit:
fields, per-step (tau, halvings, iteration counts, last_delta), clamp counts
and error behaviour. Skipped only where the reference build is absent (the
GPU box carries the prebuilt .so, so it runs there too).
"""
import numpy as np
import pytest

from oracle.oracle import OracleError, PortStepper, RefStepper, port_thomas_batch, ref_available, \
    ref_thomas_batch
from paper_1912_03744_b200 import configs
from paper_1912_03744_b200.materials import HalfPointRule, RangePolicy
from paper_1912_03744_b200.solver import make_field

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _init(case, kind):
    g = case.grid()
    if kind == "T0":
        return make_field(g, case.solver.T0)
    return configs.smooth_field(g, {"smooth": 6.0, "smooth20": 20.0}[kind])


CASES = [
    ("stepcell-nl", lambda: configs.step_cell(True), "smooth", 30, 0.0),
    ("stepcell-lin", lambda: configs.step_cell(False), "smooth", 30, 0.0),
    ("stepcell-meanlambda", lambda: configs.step_cell(True, halfpoint_rule=HalfPointRule.MeanLambda,
                                                      tau_source_divisor=1.0), "smooth20", 10, 0.05),
    ("stepcell-harmonic", lambda: configs.step_cell(
        True, halfpoint_rule=HalfPointRule.TwoSidedHarmonic, tau_source_divisor=1.0), "smooth20", 10,
     0.05),
    ("stepcell-neumann", lambda: configs.step_cell(True, all_neumann=True, tau_source_divisor=2.0),
     "smooth20", 10, 0.05),
    ("stepcell-maxiter1", lambda: configs.step_cell(True, max_iter=1), "smooth20", 2, 0.001),
    ("stepcell-null", lambda: configs.step_cell(True, source=configs.SOURCE_NULL,
                                                tau_source_divisor=1.0), "smooth20", 10, 0.05),
    ("paper-small", configs.paper_like_small, "T0", 40, 0.0),
    ("paper-small-late", configs.paper_like_small, "T0", 40, 0.0099),
    ("cfg0-150", lambda: configs.cfg0(150), "T0", 150, 0.0),
    ("cfg4-small", lambda: configs.scaled(configs.cfg4(), [44, 5, 13, 3], 128, 87), "T0", 40, 0.0),
]


@pytest.mark.parametrize("name,build,init,steps,t0", CASES, ids=[c[0] for c in CASES])
def test_port_matches_reference_bitwise(name, build, init, steps, t0):
    case = build()
    ref, port = RefStepper(case), PortStepper(case)
    f_ref = _init(case, init)
    f_port = f_ref.copy(order="F")
    te_r, st_r, res_r = ref.run(f_ref, t0, steps)
    te_p, st_p, res_p = port.run(f_port, t0, steps)
    assert te_r == te_p
    assert res_r == res_p  # tau_used, halvings, iterations and last_delta, every step
    m = case.grid().mask()
    assert np.array_equal(f_ref[m], f_port[m])
    assert ref.clamp_events() == port.clamp_events()


def test_half_steps_bitwise_and_clamp_counts():
    case = configs.step_cell(True)
    g = case.grid()
    ref, port = RefStepper(case), PortStepper(case)
    f = configs.smooth_field(g, 250.0)  # above the 0..400 K table? no: inside; push one cell out
    f[0, 0] = 450.0  # out of table range -> clamp events on both paths
    for half in ("radial_half_step", "axial_half_step"):
        o1, o2 = make_field(g, 0.0), make_field(g, 0.0)
        r1 = getattr(ref, half)(f, 0.0, 2e-3, o1)
        r2 = getattr(port, half)(f, 0.0, 2e-3, o2)
        assert r1 == r2
        assert np.array_equal(o1[g.mask()], o2[g.mask()])
    assert ref.clamp_events() == port.clamp_events()
    assert sum(ref.clamp_events()) > 0


def test_strict_range_error_line():
    case = configs.step_cell(True, range_policy=RangePolicy.Strict)
    g = case.grid()
    ref, port = RefStepper(case), PortStepper(case)
    f = configs.smooth_field(g)
    f[3, 5] = 500.0
    for stepper in (ref, port):
        out = make_field(g, 0.0)
        with pytest.raises(OracleError) as e:
            stepper.radial_half_step(f, 0.0, 1e-3, out)
        assert e.value.code == 3
    with pytest.raises(OracleError) as e1:
        ref.radial_half_step(f, 0.0, 1e-3, make_field(g, 0.0))
    with pytest.raises(OracleError) as e2:
        port.radial_half_step(f, 0.0, 1e-3, make_field(g, 0.0))
    assert e1.value.line == e2.value.line


def test_tau_floor_error():
    case = configs.step_cell(True, max_iter=1)
    case.solver.tau_min = 0.9 * 1e-7  # first halving trips the floor (test_solver.cpp:340-352)
    g = case.grid()
    for stepper in (RefStepper(case), PortStepper(case)):
        with pytest.raises(OracleError) as e:
            stepper.step(configs.smooth_field(g, 20.0), 0.001)
        assert e.value.code == 2


def test_pulse_and_initial_tau_match():
    case = configs.paper_like_small()
    ref, port = RefStepper(case), PortStepper(case)
    for t in np.linspace(0.0, 0.35, 701):
        assert ref.pulse_value(t) == port.pulse_value(t)
        assert ref.initial_tau(t) == port.initial_tau(t)


@pytest.mark.parametrize("layout", [0, 1])
def test_thomas_batch_port_matches_reference(layout):
    rng = np.random.default_rng(7)
    n, batch = 100, 64
    lo = rng.uniform(-1, 0, n * batch)
    up = rng.uniform(-1, 0, n * batch)
    dg = 2.05 + np.abs(lo) + np.abs(up)
    rhs = rng.uniform(-1, 1, n * batch)
    rc1, x1, _ = ref_thomas_batch(lo, dg, up, rhs, n, batch, layout, workers=3)
    rc2, x2, _ = port_thomas_batch(lo, dg, up, rhs, n, batch, layout)
    assert rc1 == rc2 == 0
    assert np.array_equal(x1, x2)


def test_thomas_zero_pivot_reports_lowest_system():
    n, batch = 5, 8
    a = np.zeros(n * batch); c = np.zeros(n * batch); d = np.ones(n * batch)
    b = np.ones(n * batch)
    b[3 * n + 2] = 0.0
    b[6 * n + 0] = 0.0
    rc1, _, f1 = ref_thomas_batch(a, b, c, d, n, batch, 0)
    rc2, _, f2 = port_thomas_batch(a, b, c, d, n, batch, 0)
    assert rc1 == rc2 == 4 and f1 == f2 == 3
