"""Generalised stepped domain (beyond the reference's two-level
Grid). The reference cannot express it, so the checker is the C restatement
(oracle/adi_oracle.c) with explicit per-line extents; that path is first
pinned to the reference itself on a two-level grid (same extents passed
explicitly), then the CUDA path is compared with it bit for bit on two- and
three-level staircases."""
import numpy as np
import pytest

from oracle.oracle import PortStepper, RefStepper
from paper_1912_03744_b200 import configs
from paper_1912_03744_b200.solver import make_field


def _small(case):
    return configs.scaled(case, [44, 5, 13, 3], 128, 87)


def test_grid_extents_are_prefix_masks():
    for ins in (0.022, 0.0185, 0.015):
        g = _small(configs.cfg4_staircase(insulator_length=ins)).grid()
        ce, re = g.col_extents(), g.row_extents()
        assert np.all(np.diff(ce) <= 0) and np.all(np.diff(re) <= 0)
        for i in range(g.nr()):
            for j in (0, ce[i] - 1, min(ce[i], g.nz() - 1)):
                assert (j < ce[i]) == (i < re[j])
        assert g.active_cells() == int(ce.sum()) == int(g.mask().sum())
    # insulator_length == outer_length: the reference's own two levels
    two = _small(configs.cfg4_staircase(insulator_length=0.015))
    assert two.domain.is_two_level()
    ref = _small(configs.cfg4()).grid()
    g = two.grid()
    assert np.array_equal(g.z_centers, ref.z_centers)
    assert np.array_equal(g.col_extents(), ref.col_extents())


def test_explicit_extents_oracle_pinned_to_reference():
    """The oracle's explicit-extent path on a two-level grid == the reference."""
    case = _small(configs.cfg4())
    g = case.grid()
    ref, port = RefStepper(case), PortStepper(case, explicit_extents=True)
    fr, fp = make_field(g, case.solver.T0), make_field(g, case.solver.T0)
    _, _, rr = ref.run(fr, 0.0, 8)
    _, _, rp = port.run(fp, 0.0, 8)
    assert [(a.tau_used, a.halvings, a.radial, a.axial) for a in rr] == \
        [(b.tau_used, b.halvings, b.radial, b.axial) for b in rp]
    assert np.array_equal(fr[g.mask()], fp[g.mask()])


@pytest.mark.gpu
@pytest.mark.parametrize("ins", [0.022, 0.0185])
def test_staircase_exact_bitwise_vs_oracle(cuda, ins):
    from helpers import gpu_stepper, to_dev, to_host
    case = _small(configs.cfg4_staircase(insulator_length=ins))
    g = case.grid()
    port = PortStepper(case)
    fo = make_field(g, case.solver.T0)
    _, _, ro = port.run(fo, 0.0, 12)
    gpu = gpu_stepper(case, "exact")
    fg = to_dev(make_field(g, case.solver.T0))
    _, _, rg = gpu.run(fg, 0.0, 12, keep_results=True)
    assert [(a.tau_used, a.halvings, a.radial, a.axial) for a in rg] == \
        [(b.tau_used, b.halvings, b.radial, b.axial) for b in ro]
    m = g.mask()
    assert np.array_equal(to_host(fg)[m], fo[m])
    assert gpu.clamp_events() == port.clamp_events()


@pytest.mark.gpu
def test_staircase_partitioned_exact_bitwise(cuda):
    from paper_1912_03744_b200.dist import PartitionedAdi
    from helpers import gpu_stepper, to_dev, to_host
    case = _small(configs.cfg4_staircase(insulator_length=0.0185))
    g = case.grid()
    single = gpu_stepper(case, "exact")
    f1 = to_dev(make_field(g, case.solver.T0))
    _, _, r1 = single.run(f1, 0.0, 6, keep_results=True)
    part = PartitionedAdi(g, case.materials, configs.make_source(case, g), case.timing,
                          case.solver, device=0, emulate=3, mode="exact")
    part.set_field(to_dev(make_field(g, case.solver.T0)))
    _, _, r2 = part.run(0.0, 6, keep_results=True)
    out = to_dev(make_field(g, 0.0))
    part.get_field(out)
    assert [(a.tau_used, a.radial, a.axial) for a in r1] == \
        [(b.tau_used, b.radial, b.axial) for b in r2]
    m = g.mask()
    assert np.array_equal(to_host(out)[m], to_host(f1)[m])
