"""Flow sweeps (every Picard iteration of a sweep in one persistent launch,
Picard items taken from a ready queue; adi_kernels.h) against the oracle:
bit-identical fields and tau / halving / iteration / delta sequences, clamp
events counted only for the iterations the reference runs (a speculative
iteration after convergence counts nothing), and the reference's lowest
failing line under the strict range policy. The flow is the default for
grids of more line blocks than SMs (configs[3]); here it is forced on small
grids (PCGPU_FLOW=1). The other stepper tests run on it too through the
`stepper_path` fixture's "flow" parameter."""
import numpy as np
import pytest

from oracle.oracle import OracleError, PortStepper
from paper_1912_03744_b200 import configs
from paper_1912_03744_b200.errors import LineError, TableRangeError
from paper_1912_03744_b200.materials import RangePolicy
from paper_1912_03744_b200.solver import make_field

from helpers import gpu_stepper, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def flow_on(monkeypatch):
    monkeypatch.setenv("PCGPU_RESIDENT", "0")
    monkeypatch.setenv("PCGPU_FLOW", "1")


@pytest.fixture(params=["exact-lean", "exact-x"])
def lookup_kind(request, monkeypatch):
    if request.param == "exact-x":
        monkeypatch.setenv("PCGPU_NO_EXACTLEAN", "1")
    return request.param


def _seq(results):
    return np.array([[r.tau_used, r.halvings, r.radial.iterations, r.axial.iterations,
                      r.radial.last_delta, r.axial.last_delta] for r in results])


def _cfg4e():
    """configs[4]'s materials on a 64 x 128 staircase (even line counts: both
    sweeps can flow)."""
    return configs.scaled(configs.cfg4(), [44, 5, 13, 2], 128, 87)


def _cold_spots(case):
    f = make_field(case.grid(), case.solver.T0)
    f[10:12, 20:23] = 3.9
    f[46, 30:32] = 3.95
    f[50:52, 5:7] = 3.95
    f[63, 40] = 3.97
    return f


def test_flow_selected(cuda):
    gpu = gpu_stepper(_cfg4e(), "exact")
    assert "steps=host-driven flow=radial+axial" in gpu.describe()


@pytest.mark.parametrize("driver", ["run", "step"])
def test_flow_clamp_events_bitwise(cuda, lookup_kind, driver):
    """Cells below the tables in several layers: fields, sequences and the
    per-layer clamp counts equal the oracle's, through speculative batches
    (run) and step by step (step)."""
    case = _cfg4e()
    g = case.grid()
    f = _cold_spots(case)
    port, gpu = PortStepper(case), gpu_stepper(case, "exact")
    assert "flow=radial+axial" in gpu.describe()
    fo = f.copy(order="F")
    te_o, _, res_o = port.run(fo, 0.0, 8)
    fg = to_dev(f)
    if driver == "run":
        te_g, _, res_g = gpu.run(fg, 0.0, 8, keep_results=True)
    else:
        res_g, te_g = [], 0.0
        for _ in range(8):
            r = gpu.step(fg, te_g)
            res_g.append(r)
            te_g += r.tau_used
    assert te_g == te_o
    assert np.array_equal(_seq(res_g), _seq(res_o))
    m = g.mask()
    assert np.array_equal(to_host(fg)[m], fo[m])
    assert gpu.clamp_events() == port.clamp_events()
    assert sum(1 for c in port.clamp_events() if c) >= 2


def test_flow_strict_range_lowest_line(cuda, lookup_kind):
    case = _cfg4e()
    case.solver.range_policy = RangePolicy.Strict
    g = case.grid()
    f = make_field(g, case.solver.T0)
    f[40, 70] = 500.0
    f[20, 12] = 1.0
    port, gpu = PortStepper(case), gpu_stepper(case, "exact")
    for half in ("radial_half_step", "axial_half_step"):
        with pytest.raises(OracleError) as eo:
            getattr(port, half)(f, 0.0, 1e-4, make_field(g, 0.0))
        with pytest.raises(LineError) as eg:
            getattr(gpu, half)(f, 0.0, 1e-4, make_field(g, 0.0))
        assert eg.value.cause is TableRangeError
        assert eg.value.line == eo.value.line
    with pytest.raises(OracleError) as eo:
        port.step(f.copy(order="F"), 0.0)
    with pytest.raises(LineError) as eg:
        gpu.step(to_dev(f), 0.0)
    assert eg.value.line == eo.value.line


def test_flow_half_steps_bitwise(cuda):
    """Both half-steps alone (the per-sweep status merge: iterations, last
    delta, converged flag) on a smooth field that needs several iterations."""
    case = _cfg4e()
    g = case.grid()
    f = configs.smooth_field(g, 20.0)
    port, gpu = PortStepper(case), gpu_stepper(case, "exact")
    for half in ("radial_half_step", "axial_half_step"):
        oo, og = make_field(g, 0.0), make_field(g, 0.0)
        ro = getattr(port, half)(f, 0.0, 2e-4, oo)
        rg = getattr(gpu, half)(f, 0.0, 2e-4, og)
        assert (rg.converged, rg.iterations, rg.last_delta) == \
            (ro.converged, ro.iterations, ro.last_delta)
        assert ro.iterations >= 3
        assert np.array_equal(og[g.mask()], oo[g.mask()])


def test_flow_halvings_and_iteration_changes(cuda):
    """A coarse cell whose Picard counts change from step to step and whose
    steps halve (max_iter 6): the speculation (iterations started before the
    previous one is known) never changes a result."""
    case = configs.scaled(configs.cfg0(), [23, 3, 5, 1], 64)
    case.solver.tau_source_divisor = 10.0
    case.solver.max_iter = 6
    g = case.grid()
    port, gpu = PortStepper(case), gpu_stepper(case, "exact")
    assert "flow=radial+axial" in gpu.describe()
    fo = make_field(g, case.solver.T0)
    te_o, _, res_o = port.run(fo, 0.02, 30)
    fg = to_dev(make_field(g, case.solver.T0))
    te_g, _, res_g = gpu.run(fg, 0.02, 30, keep_results=True)
    assert te_g == te_o
    assert np.array_equal(_seq(res_g), _seq(res_o))
    assert np.array_equal(to_host(fg)[g.mask()], fo[g.mask()])
    assert sum(r.halvings for r in res_o) > 0
    assert len({r.radial.iterations for r in res_o}) >= 2
