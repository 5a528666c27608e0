"""BASELINE.json configurations and the reference test fixtures.

Each builder returns a ``Case``: the reference-level inputs (DomainSpec,
GridSpec, per-layer MaterialTables, SourceSpec, SolverConfig, source kind)
from which both the GPU stepper and the CPU oracles are constructed. The
power-law materials of BASELINE are expressed as the reference's piecewise-
linear tables on uniform 1 K knots starting below T0; the tables
are the input, so parity is to the reference's interpolation.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

from .geometry import DomainSpec, Grid, GridSpec
from .materials import HalfPointRule, MaterialTable, PropertyTable, RangePolicy
from .solver import SolverConfig
from .source import SourceSpec, Waveform

SOURCE_NULL, SOURCE_JOULE, SOURCE_FIELD = 0, 1, 2


@dataclass
class Case:
    name: str
    domain: DomainSpec
    gridspec: GridSpec
    materials: List[MaterialTable]
    timing: SourceSpec
    solver: SolverConfig
    source_kind: int = SOURCE_JOULE
    steps: int = 1          # fixed-dt step count (configs 0/3) or a parity-test budget
    t_end: Optional[float] = None  # adaptive configs: simulated time
    notes: str = ""

    def grid(self) -> Grid:
        return Grid(self.domain, self.gridspec)


# ---- BASELINE material model (configs[0]) ----------------------------------
LAMBDA0 = [400.0, 0.1, 5.0, 1.0]
ALPHA = [0.8, 1.0, 1.2, 1.0]
C0 = [1e3, 5e2, 8e2, 6e2]
KNOTS = np.arange(4.0, 301.0, 1.0)  # uniform 1 K knots over [4, 300]


def power_law_materials(alpha=ALPHA, chi_slope=0.01, source_layer=2) -> List[MaterialTable]:
    mats = []
    for m in range(4):
        cv = PropertyTable(KNOTS, C0[m] * (KNOTS / 4.2) ** 3)        # rho*c_V, rho = 1
        lam = PropertyTable(KNOTS, LAMBDA0[m] * (KNOTS / 4.2) ** alpha[m])
        chi = None
        if m == source_layer:  # chi = 1e-5 (1 + slope T): exactly linear, 2 knots
            chi = PropertyTable([4.0, 300.0], [1e-5 * (1 + chi_slope * 4.0),
                                               1e-5 * (1 + chi_slope * 300.0)])
        mats.append(MaterialTable(f"layer{m}", 1.0, cv, lam, chi))
    return mats


RADII = [1.0e-3, 1.1e-3, 1.4e-3, 1.45e-3]


def _domain(core=0.02, outer=0.02) -> DomainSpec:
    return DomainSpec(list(RADII), core, outer, [f"layer{m}" for m in range(4)], 2)


def _joule(domain: DomainSpec, t_per=1.0, t_src=0.1, t_trs=0.01, I0=1.0) -> SourceSpec:
    return SourceSpec(t_per=t_per, t_src=t_src, t_trs=t_trs, I0=I0,
                      S_C=domain.source_cross_section(), waveform=Waveform.Rectangular,
                      joule_dimensional=True)


def cfg0(steps: int = 2000) -> Case:
    """configs[0]: 100 x 200, tau = 1e-4 for 2000 steps, eps 1e-8, max_iter 20."""
    d = _domain()
    return Case("cfg0", d, GridSpec([69, 7, 21, 3], 200, 200), power_law_materials(),
                _joule(d), SolverConfig(epsilon=1e-8, max_iter=20, tau_transient_divisor=100.0,
                                        tau_source_divisor=1000.0),
                steps=steps, notes="tau = 0.01/100 = 0.1/1000 = 1e-4 in every window")


def cfg2(periods: float = 5.0) -> Case:
    """configs[2]: 1024 x 2048, adaptive (native controller), max_iter 10."""
    d = _domain()
    return Case("cfg2", d, GridSpec([706, 71, 212, 35], 2048, 2048), power_law_materials(),
                _joule(d), SolverConfig(epsilon=1e-8, max_iter=10, tau_transient_divisor=1000.0,
                                        tau_source_divisor=100.0),
                t_end=periods * 1.0, notes="1e-5 in transient windows, 1e-3 elsewhere")


def cfg3(steps: int = 200, nr_div=(5650, 565, 1695, 282), nz: int = 16384) -> Case:
    """configs[3]: 8192 x 16384, tau = 1e-5 for 200 steps."""
    d = _domain()
    return Case("cfg3", d, GridSpec(list(nr_div), nz, nz), power_law_materials(),
                _joule(d), SolverConfig(epsilon=1e-8, max_iter=20, tau_transient_divisor=1000.0,
                                        tau_source_divisor=10000.0),
                steps=steps, notes="tau = 0.01/1000 = 0.1/10000 = 1e-5 in every window")


def cfg4(periods: float = 10.0) -> Case:
    """configs[4]: stepped 2048 x 4096 (2-level reference approximation), stiffer
    nonlinearity, I0 = 3 A, t_src/t_per = 0.3, adaptive."""
    d = _domain(core=0.022, outer=0.015)
    return Case("cfg4", d, GridSpec([1412, 141, 424, 71], 4096, 2793),
                power_law_materials(alpha=[1.5, 1.0, 2.0, 1.0], chi_slope=0.05),
                _joule(d, t_src=0.3, I0=3.0),
                SolverConfig(epsilon=1e-8, max_iter=10, tau_transient_divisor=1000.0,
                             tau_source_divisor=300.0),
                t_end=periods * 1.0, notes="2-level staircase: core to 22 mm, shell to 15 mm")


def cfg4_staircase(periods: float = 10.0, insulator_length: float = 0.022) -> Case:
    """configs[4] on the generalised stepped domain (beyond the
    reference's two-level Grid): r_max(z) = 1.45 mm below 15 mm and 1.1 mm
    above (core and insulator to `insulator_length` ... 22 mm), the copper
    core to 22 mm. insulator_length < 22 mm gives three axial levels. No
    reference oracle exists for it; the C restatement (oracle/) is the checker."""
    c = cfg4(periods)
    d = replace(c.domain, layer_lengths=[0.022, insulator_length, 0.015, 0.015])
    return replace(c, name="cfg4-staircase", domain=d,
                   notes=f"staircase: core 22 mm, insulator {insulator_length * 1e3:g} mm, "
                         "heater and coating 15 mm")


def scaled(case: Case, nr_div, nz_core: int, nz_outer: Optional[int] = None,
           name: Optional[str] = None) -> Case:
    """Same physics on a smaller grid (parity tests at oracle-friendly sizes)."""
    return replace(case, name=name or case.name + "-small",
                   gridspec=GridSpec(list(nr_div), nz_core, nz_outer or nz_core))


# ---- reference test fixtures -------------------------------------------------
def step_cell(nonlinear: bool = True, source: int = SOURCE_JOULE, **solver_kw) -> Case:
    """StepCell fixture of the reference solver tests (test_solver.cpp:15-77)."""
    d = DomainSpec([0.5, 0.8, 1.0], 2.0, 1.5, ["core", "mid", "skin"], 1)
    g = GridSpec([6, 5, 4], 8, 6)

    def lin(a, b):
        return PropertyTable([0.0, 400.0], [a, b])

    if nonlinear:
        mats = [MaterialTable("core", 2.0, lin(1.0, 3.0), lin(1.0, 41.0)),
                MaterialTable("mid", 1.0, lin(1.0, 3.0), lin(1.0, 41.0), lin(2.0, 2.0)),
                MaterialTable("skin", 1.5, lin(1.0, 3.0), lin(1.0, 41.0))]
    else:
        mats = [MaterialTable("core", 2.0, lin(0.8, 0.8), lin(2.0, 2.0)),
                MaterialTable("mid", 1.0, lin(1.1, 1.1), lin(0.5, 0.5), lin(2.0, 2.0)),
                MaterialTable("skin", 1.5, lin(0.9, 0.9), lin(1.0, 1.0))]
    timing = SourceSpec(t_per=0.1, t_src=0.01, t_trs=1e-4, I0=0.8,
                        S_C=d.source_cross_section(), waveform=Waveform.Rectangular)
    return Case("stepcell", d, g, mats, timing, SolverConfig(**solver_kw), source_kind=source)


def smooth_field(grid: Grid, base: float = 6.0) -> np.ndarray:
    """StepCell::smooth_field (test_solver.cpp:69-76)."""
    f = np.full((grid.nr(), grid.nz()), 4.2, dtype=np.float64, order="F")
    for i in range(grid.nr()):
        for j in range(grid.col_extent(i)):
            f[i, j] = base + 2.0 * math.sin(3.0 * grid.r_center(i)) * math.cos(1.7 * grid.z_center(j))
    return f


def paper_like_small(source: int = SOURCE_JOULE) -> Case:
    """A 64 x 32 stepped coarsening in the spirit of the acceptance suite's
    small paper cell (acceptance_main.cpp:64-90), with the BASELINE materials
    and a transient (erf) pulse."""
    d = DomainSpec(list(RADII), 0.02, 0.015, [f"layer{m}" for m in range(4)], 2)
    t = SourceSpec(t_per=0.1, t_src=0.01, t_trs=1e-4, I0=1.0, S_C=d.source_cross_section(),
                   waveform=Waveform.Transient, joule_dimensional=True)
    return Case("paper_small", d, GridSpec([40, 6, 14, 4], 32, 24), power_law_materials(), t,
                SolverConfig(epsilon=1e-8, max_iter=10), source_kind=source)


# ---- the reference's own input configuration --------------------------------
def synthetic_materials(names=("copper_like", "insulator_like", "graphite_like",
                               "coating_like")) -> List[MaterialTable]:
    """proj/configs/materials_synthetic.json: the reference's synthetic
    two-knot tables (the paper's cryogenic data is not available)."""
    def t(a, b):
        return PropertyTable([2.0, 400.0], [a, b])
    table = {
        "copper_like": MaterialTable("copper_like", 10.0, t(1.8, 2.2), t(800.0, 800.0)),
        "insulator_like": MaterialTable("insulator_like", 1.0, t(0.05, 0.08), t(0.0008, 0.0012)),
        "graphite_like": MaterialTable("graphite_like", 1.0, t(0.95, 1.1), t(0.05, 0.09),
                                       t(100.0, 110.0)),
        "coating_like": MaterialTable("coating_like", 1.0, t(0.5, 0.6), t(0.5, 0.55)),
    }
    return [table[n] for n in names]


def paper_cell(steps: int = 2000) -> Case:
    """proj/configs/paper_cell.json:1-38 -- the paper's 1210 x 100 cell (the grid
    of PAPER.md's only performance figure): layer radii 0.24/0.245/0.25/0.2501,
    core 5.0 and shell 4.0 long, radial divisions [800, 200, 200, 10], axial
    100 (core) / 80 (shell), materials_synthetic.json, transient (erf) pulse
    t_per 0.1, t_src 0.01, t_trs 1e-4, xi 4, zeta 2, I0 0.5742, S_C derived
    from the domain (config.cpp:207), epsilon 1e-6, max_iter 10, the other
    solver settings at their defaults (tau 1e-7 in the transient windows,
    1e-4 elsewhere). Units as the reference's config (dimensionless Joule
    factor I0^2 / S_C)."""
    d = DomainSpec([0.24, 0.245, 0.25, 0.2501], 5.0, 4.0,
                   ["copper_like", "insulator_like", "graphite_like", "coating_like"], 2)
    timing = SourceSpec(t_per=0.1, t_src=0.01, t_trs=1e-4, xi=4.0, zeta=2.0, I0=0.5742,
                        S_C=d.source_cross_section(), waveform=Waveform.Transient)
    return Case("paper_cell", d, GridSpec([800, 200, 200, 10], 100, 80), synthetic_materials(),
                timing, SolverConfig(epsilon=1e-6, max_iter=10), steps=steps,
                notes="the reference's paper_cell.json")


def small_paper(materials: str = "synthetic", I0: float = 0.0) -> Case:
    """The acceptance suite's paper cell coarsened to 64 x 32
    (acceptance_main.cpp:64-103): small_paper_domain, small_paper_gridspec,
    paper_timing(I0); materials_synthetic.json or constant_materials()."""
    d = DomainSpec([0.24, 0.245, 0.25, 0.2501], 5.0, 4.0, ["core", "ins", "heat", "coat"], 2)
    if materials == "synthetic":
        mats = synthetic_materials()
    else:
        def lin(v):
            return PropertyTable([0.0, 400.0], [v, v])
        mats = [MaterialTable("core", 2.0, lin(1.0), lin(2.0)),
                MaterialTable("ins", 1.0, lin(0.8), lin(0.5), lin(2.0)),
                MaterialTable("heat", 1.0, lin(1.2), lin(1.0), lin(2.0)),
                MaterialTable("coat", 1.5, lin(0.9), lin(0.8))]
    timing = SourceSpec(t_per=0.1, t_src=0.01, t_trs=1e-4, xi=4.0, zeta=2.0, I0=I0,
                        S_C=math.pi * (0.25 * 0.25 - 0.245 * 0.245), waveform=Waveform.Transient)
    return Case("small_paper", d, GridSpec([40, 8, 8, 8], 40, 24), mats, timing,
                SolverConfig(), source_kind=SOURCE_NULL if I0 == 0.0 else SOURCE_JOULE)


def make_source(case: Case, grid: Optional[Grid] = None):
    """The SourceModel a Case describes (JouleSource / NullSource / FieldSource)."""
    from .source import FieldSource, JouleSource, NullSource
    d = case.domain
    if case.source_kind == SOURCE_JOULE:
        return JouleSource(case.timing, d.source_layer, case.materials[d.source_layer],
                           case.solver.range_policy)
    if case.source_kind == SOURCE_FIELD:
        return FieldSource(grid or case.grid())
    return NullSource()


CONFIGS = {"cfg0": cfg0, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "paper_cell": paper_cell}
