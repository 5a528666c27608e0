"""Host parts of the device-resident runner (no GPU): the probe_cell mirror
against the reference's own probe_cell (runner.cpp:20-28, through the
reference library's evolve), and RunnerConfig validation like
runner.hpp:96-102."""
import pytest

from oracle.oracle import RefStepper, ref_evolve
from paper_1912_03744_b200 import configs
from paper_1912_03744_b200.errors import ConfigError
from paper_1912_03744_b200.runner import (ProbeSpec, RegimeDetectorConfig, RunnerConfig,
                                          probe_cell)
from paper_1912_03744_b200.solver import make_field


def test_probe_cell_matches_reference():
    case = configs.step_cell(True, tau_transient_divisor=10.0, tau_source_divisor=20.0)
    g = case.grid()
    d = case.domain
    rs = [0.0, 0.05, 0.25, 0.5, 0.55, 0.8, 0.99, d.layer_radii[-1]]
    zs = [0.0, 0.1, 0.75, 1.3]
    probes = [ProbeSpec(r, z) for r in rs for z in zs][:16]
    cfg = RunnerConfig(t_end=1e-5, probes=probes, snapshot_pre_on=False,
                       snapshot_post_off=False)
    want = ref_evolve(RefStepper(case), make_field(g, case.solver.T0), cfg.t_end, cfg,
                      case.timing.I0)
    got = [probe_cell(g, p.r, p.z) for p in probes]
    assert got == [tuple(c) for c in want["probe_cells"]]


@pytest.mark.parametrize("bad", [
    dict(t_end=0.0), dict(snapshot_times=[-1.0]),
    dict(detector=RegimeDetectorConfig(samples_per_period=0)),
    dict(detector=RegimeDetectorConfig(tolerance=0.0)),
    dict(detector=RegimeDetectorConfig(min_periods=0)),
])
def test_runner_config_validation(bad):
    with pytest.raises(ConfigError):
        RunnerConfig(**bad).validate()
