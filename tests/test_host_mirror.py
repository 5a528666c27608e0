"""Host-side mirror of the reference interface: Grid metrics, pulse, tau and
validation must be bit-identical to the reference's own (oracle/_ref)."""
import math

import numpy as np
import pytest

from oracle.oracle import RefStepper, ref_available
from paper_1912_03744_b200 import configs
from paper_1912_03744_b200.errors import ConfigError
from paper_1912_03744_b200.geometry import DomainSpec, Grid, GridSpec, cell_metrics
from paper_1912_03744_b200.solver import SolverConfig, initial_tau
from paper_1912_03744_b200.source import JouleSource, pulse_value

ALL = [configs.step_cell(True), configs.paper_like_small(), configs.cfg0(),
       configs.scaled(configs.cfg4(), [44, 5, 13, 3], 128, 87), configs.cfg4(), configs.cfg2()]


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("case", ALL, ids=lambda c: c.name)
def test_grid_metrics_bitwise(case):
    g = case.grid()
    ga = RefStepper(case).grid_arrays()
    assert (ga["nr"], ga["nz"], ga["nr_core"], ga["nz_shared"], ga["active"]) == \
        (g.nr(), g.nz(), g.nr_core(), g.nz_shared(), g.active_cells())
    for k, v in (("r_center", g.r_centers), ("width_r", g.width_r_arr), ("gap_r", g.gap_r_arr),
                 ("z_center", g.z_centers), ("width_z", g.width_z_arr), ("gap_z", g.gap_z_arr),
                 ("layer", g.layer_arr)):
        assert np.array_equal(ga[k], v), k


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_pulse_tau_amplitude_bitwise():
    case = configs.paper_like_small()
    ref = RefStepper(case)
    src = JouleSource(case.timing, 2, case.materials[2])
    assert src.amplitude == ref.source_amplitude()
    for t in np.linspace(0, 0.3, 301):
        assert pulse_value(t, case.timing) == ref.pulse_value(t)
        assert initial_tau(t, case.timing, case.solver) == ref.initial_tau(t)


def test_cfg_shapes_match_survey():
    # grid sizes and fixed-dt choices
    assert (configs.cfg0().grid().nr(), configs.cfg0().grid().nz()) == (100, 200)
    g4 = configs.cfg4().grid()
    assert (g4.nr(), g4.nz(), g4.nr_core(), g4.nz_shared()) == (2048, 4096, 1412, 2793)
    assert g4.active_cells() == 7559900
    c0 = configs.cfg0()
    for t in (0.0, 0.005, 0.05, 0.105, 0.5):
        assert initial_tau(t, c0.timing, c0.solver) == 1e-4
    c3 = configs.cfg3()
    for t in (0.0, 0.05, 0.5):
        assert initial_tau(t, c3.timing, c3.solver) == 1e-5
    assert GridSpec([5650, 565, 1695, 282]).radial_divisions and sum([5650, 565, 1695, 282]) == 8192


def test_validation_errors():
    with pytest.raises(ConfigError):
        DomainSpec([1.0, 0.5], 1, 1, ["a", "b"], 0).validate()
    with pytest.raises(ConfigError):
        Grid(DomainSpec([1.0], 1.0, 2.0, ["a"], 0), GridSpec([3], 2, 2))
    with pytest.raises(ConfigError):
        SolverConfig(epsilon=0).validate()
    with pytest.raises(ConfigError):
        SolverConfig(t_ceiling=1.0).validate()


def test_cell_metrics_at_interface():
    # interface gap jump (test_geometry.cpp:113-132 pattern)
    g = Grid(DomainSpec([1.0, 1.1], 1.0, 1.0, ["a", "b"], 0), GridSpec([10, 2], 2, 2))
    m = cell_metrics(g, 9, 0)
    assert math.isclose(m.hbar, 0.5 * (0.1 + 0.075), rel_tol=1e-14)
    assert math.isclose(m.r_lo, 0.5 * (g.r_center(8) + g.r_center(9)), rel_tol=0)
