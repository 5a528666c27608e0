"""The reference's acceptance criteria and its own input configuration, run on
the GPU stepper (through the C-ABI), with the reference's tolerances:

  paper_cell.json        proj/configs/paper_cell.json:1-38 (the paper's 1210 x 100 cell)
  equilibrium            acceptance_main.cpp:122-144 (1000 steps, drift <= 1e-12)
  maximum principle      acceptance_main.cpp:173-236, test_solver.cpp:371-431
  MMS convergence order  acceptance_main.cpp:239-371 (FIELD source, order >= 1.8)
  dense fixed-point      test_solver.cpp:268-303, acceptance_main.cpp:373-416
                         (oracles.hpp:61-176; error <= epsilon)

Exact mode is bit-identical to the reference, so these hold wherever the
reference's own criteria hold; here they are checked on the GPU results
themselves (and bit for bit against the reference / the C restatement where
it applies).
"""
import math
import os

import numpy as np
import pytest

from oracle.oracle import PortStepper, RefStepper, ref_available
from paper_1912_03744_b200 import configs
from paper_1912_03744_b200.geometry import DomainSpec, GridSpec
from paper_1912_03744_b200.materials import MaterialTable, Property, PropertyTable
from paper_1912_03744_b200.solver import SolverConfig, make_field
from paper_1912_03744_b200.source import FieldSource, JouleSource, SourceSpec, Waveform

from acceptance_oracles import Manufactured, dense_axial_half_step, dense_radial_half_step
from helpers import gpu_stepper, to_dev, to_host

pytestmark = pytest.mark.gpu


def _seq(results):
    return np.array([[r.tau_used, r.halvings, r.radial.iterations, r.axial.iterations,
                      r.radial.last_delta, r.axial.last_delta] for r in results])


def test_paper_cell_bitwise_vs_reference(cuda):
    """The reference's own input configuration (paper_cell.json: 1210 x 100,
    materials_synthetic.json, transient erf pulse): 1200 step() calls -- the
    first transient window at tau = 1e-7, the pulse plateau at 1e-4 and the
    turn-off window -- bit for bit against the reference's AdiStepper (the C
    restatement if the reference library is absent)."""
    case = configs.paper_cell(1200)
    g = case.grid()
    assert (g.nr(), g.nz(), g.active_cells()) == (1210, 100, 112800)
    cpu = (RefStepper(case, workers=os.cpu_count() or 1) if ref_available()
           else PortStepper(case))
    fo = make_field(g, case.solver.T0)
    te_o, _, res_o = cpu.run(fo, 0.0, case.steps)
    gpu = gpu_stepper(case)
    fg = to_dev(make_field(g, case.solver.T0))
    te_g, _, res_g = gpu.run(fg, 0.0, case.steps, keep_results=True)
    assert te_g == te_o
    assert np.array_equal(_seq(res_g), _seq(res_o))
    tau_trs = case.timing.t_trs / case.solver.tau_transient_divisor  # 1e-7
    tau_src = case.timing.t_src / case.solver.tau_source_divisor    # 1e-4
    assert {tau_trs, tau_src} <= {r.tau_used for r in res_o}
    m = g.mask()
    assert np.array_equal(to_host(fg)[m], fo[m])
    assert np.max(fo[m]) > case.solver.T0  # the heater heated
    assert gpu.clamp_events() == cpu.clamp_events()


def test_equilibrium_1000_steps(cuda, stepper_path):
    """acceptance_main.cpp:122-144: the 64 x 32 paper cell with the synthetic
    materials and no source stays at T0 over 1000 steps (max drift <= 1e-12);
    bit for bit against the C restatement."""
    case = configs.small_paper("synthetic", I0=0.0)
    g = case.grid()
    assert (g.nr(), g.nz()) == (64, 32)
    gpu = gpu_stepper(case)
    fg = to_dev(make_field(g, case.solver.T0))
    _, _, res = gpu.run(fg, 0.0, 1000, keep_results=True)
    f = to_host(fg)
    m = g.mask()
    assert np.max(np.abs(f[m] - case.solver.T0)) <= 1e-12
    port = PortStepper(case)
    fo = make_field(g, case.solver.T0)
    _, _, res_o = port.run(fo, 0.0, 1000)
    assert np.array_equal(_seq(res), _seq(res_o)) and np.array_equal(f[m], fo[m])


def test_maximum_principle(cuda):
    """acceptance_main.cpp:173-236: with tau at half the bound that keeps the
    explicit transverse halves convex combinations, a random field in
    [4.5, 60] stays inside its initial bracket, cell by cell, for 200 steps."""
    case = configs.small_paper("constant", I0=0.0)
    g = case.grid()
    mats, cfg = case.materials, case.solver
    lam_max = max(m.eval(Property.Conductivity, 10.0) for m in mats)
    tau_bound = 1e30
    for i in range(g.nr()):
        mat = mats[g.layer(i)]
        rc = mat.rho() * mat.eval(Property.HeatCapacity, 10.0)
        for j in range(g.col_extent(i)):
            n, m = g.row_extent(j), g.col_extent(i)
            dz = dr = 0.0
            inv_eta = 1.0 / g.control_z(j)
            if j > 0:
                dz += lam_max / g.gap_z(j) * inv_eta
            if j < m - 1:
                dz += lam_max / g.gap_z(j + 1) * inv_eta
            elif g.layer(i) == 0:
                dz += lam_max / (0.5 * g.width_z(j)) * inv_eta
            inv_vol = 1.0 / (g.r_center(i) * g.control_r(i))
            if i > 0:
                dr += g.face_r_lo(i) * lam_max / g.gap_r(i) * inv_vol
            if i < n - 1:
                dr += g.face_r_lo(i + 1) * lam_max / g.gap_r(i + 1) * inv_vol
            tau_bound = min(tau_bound, 2.0 * rc / max(dz, dr))
    tau = 0.5 * tau_bound
    t = case.timing
    t.t_src = 100.0 * tau
    t.t_per = 10.0 * t.t_src
    t.t_trs = 1e-4 * t.t_src
    rng = np.random.default_rng(77)
    f0 = make_field(g, cfg.T0)
    msk = g.mask()
    f0[msk] = rng.uniform(4.5, 60.0, size=int(msk.sum()))
    lo, hi = min(cfg.T0, f0[msk].min()), max(cfg.T0, f0[msk].max())
    gpu = gpu_stepper(case)
    fg = to_dev(f0)
    tt = 0.05 * t.t_per
    for k in range(200):
        tt += gpu.step(fg, tt).tau_used
        f = to_host(fg)[msk]
        assert f.min() >= lo and f.max() <= hi, f"bracket violated at step {k}"


class _ManufacturedSource(FieldSource):
    """acceptance_main.cpp:262-274: power = the manufactured source at the
    bound half-step time, T-independent."""

    def __init__(self, grid, m):
        super().__init__(grid)
        self.m = m
        r = np.array([grid.r_center(i) for i in range(grid.nr())])
        z = np.array([grid.z_center(j) for j in range(grid.nz())])
        self.R, self.Zc = np.meshgrid(r, z, indexing="ij")

    def power_field(self, grid, t):
        return np.asfortranarray(self.m.source(self.R, self.Zc, t))


def _mms_march(m, n, tau, t_end):
    """MmsRun::march (acceptance_main.cpp:276-334) on the GPU stepper: the
    half-steps driven directly with the manufactured source bound per
    half-step."""
    import torch
    d = DomainSpec([m.R], m.Z, m.Z, ["uni"], 0)
    gs = GridSpec([n], n, n)
    uni = MaterialTable("uni", m.rho, PropertyTable([0.0, 400.0], [m.cv, m.cv]),
                        PropertyTable([0.0, 400.0], [m.lam, m.lam]))
    timing = SourceSpec(t_per=1.0, t_src=0.1, t_trs=1e-3, S_C=1.0, waveform=Waveform.Transient)
    cfg = SolverConfig(epsilon=1e-11, max_iter=60, T0=m.T0)
    case = configs.Case("mms", d, gs, [uni], timing, cfg, source_kind=configs.SOURCE_FIELD)
    g = case.grid()
    gpu = gpu_stepper(case, source=_ManufacturedSource(g, m))
    r = np.array([g.r_center(i) for i in range(g.nr())])
    z = np.array([g.z_center(j) for j in range(g.nz())])
    R, Zc = np.meshgrid(r, z, indexing="ij")
    f = to_dev(np.asfortranarray(m.exact(R, Zc, 0.0)))
    half, nxt = torch.empty_like(f), torch.empty_like(f)
    t = 0.0
    for _ in range(int(round(t_end / tau))):
        assert gpu.radial_half_step(f, t, tau, half).converged, "radial diverged"
        assert gpu.axial_half_step(half, t, tau, nxt).converged, "axial diverged"
        f, nxt = nxt, f
        t += tau
    return to_host(f), R, Zc


def test_mms_convergence_order(cuda):
    """acceptance_main.cpp:335-371: spatial order (24 -> 48 cells at tau 2e-4)
    and temporal order (tau 1e-3 -> 5e-4 against tau 1e-5 on 24 cells) of the
    scheme on the manufactured solution, both >= 1.8."""
    m = Manufactured()
    t_end = 0.02
    err = []
    for n in (24, 48):
        f, R, Zc = _mms_march(m, n, 2e-4, t_end)
        err.append(float(np.max(np.abs(f - m.exact(R, Zc, t_end)))))
    p_space = math.log2(err[0] / err[1])
    ref, _, _ = _mms_march(m, 24, 1e-5, t_end)
    terr = [float(np.max(np.abs(_mms_march(m, 24, tau, t_end)[0] - ref))) for tau in (1e-3, 5e-4)]
    p_time = math.log2(terr[0] / terr[1])
    print(f"MMS spatial order {p_space:.3f} (errors {err}), temporal order {p_time:.3f} ({terr})")
    assert p_space >= 1.8 and p_time >= 1.8


def test_half_steps_match_dense_fixed_point_oracle(cuda):
    """test_solver.cpp:268-303: on the nonlinear StepCell, each GPU half-step
    agrees with the dense fixed-point oracle (oracles.hpp:61-176: the whole
    system over all masked cells, frozen coefficients, re-solved until the
    iterate settles) to within epsilon."""
    case = configs.step_cell(True)
    g = case.grid()
    cfg = case.solver
    src = configs.make_source(case, g)
    tau, t = 2e-3, 0.0
    src.bind_time(t + 0.5 * tau)
    f = configs.smooth_field(g)
    gpu = gpu_stepper(case)
    half = make_field(g, 0.0)
    assert gpu.radial_half_step(f, t, tau, half).converged
    half_ref = dense_radial_half_step(case, src, f, tau, cfg.epsilon * 1e-3)
    msk = g.mask()
    assert np.max(np.abs(half[msk] - half_ref[msk])) <= cfg.epsilon
    nxt = make_field(g, 0.0)
    assert gpu.axial_half_step(half, t, tau, nxt).converged
    next_ref = dense_axial_half_step(case, src, half, tau, cfg.epsilon * 1e-3)
    assert np.max(np.abs(nxt[msk] - next_ref[msk])) <= cfg.epsilon


def test_nonlinear_oracle_half_steps(cuda):
    """acceptance_main.cpp:373-416 (a): 6 x 4 single-layer cylinder with
    lambda(T) = 1 + 0.1 T; both half-steps within epsilon of the dense
    fixed-point oracle."""
    d = DomainSpec([1.0], 1.0, 1.0, ["nl"], 0)
    gs = GridSpec([6], 4, 4)
    mat = MaterialTable("nl", 1.0, PropertyTable([0.0, 400.0], [1.0, 1.0]),
                        PropertyTable([0.0, 400.0], [1.0, 41.0]),
                        PropertyTable([0.0, 400.0], [2.0, 2.0]))
    timing = SourceSpec(t_per=1.0, t_src=0.5, t_trs=1e-3, I0=1.0, S_C=1.0,
                        waveform=Waveform.Rectangular)
    case = configs.Case("nl", d, gs, [mat], timing, SolverConfig())
    g = case.grid()
    src = JouleSource(timing, 0, mat)
    tau = 1e-3
    src.bind_time(0.5 * tau)
    f0 = make_field(g, case.solver.T0)
    for i in range(g.nr()):
        for j in range(g.nz()):
            f0[i, j] = 5.0 + 2.0 * math.cos(3.0 * g.r_center(i)) * math.cos(2.0 * g.z_center(j))
    gpu = gpu_stepper(case)
    half, nxt = f0.copy(order="F"), f0.copy(order="F")
    assert gpu.radial_half_step(f0, 0.0, tau, half).converged
    ref_h = dense_radial_half_step(case, src, f0, tau, 1e-9)
    assert np.max(np.abs(half - ref_h)) <= case.solver.epsilon
    assert gpu.axial_half_step(half, 0.0, tau, nxt).converged
    ref_n = dense_axial_half_step(case, src, half, tau, 1e-9)
    assert np.max(np.abs(nxt - ref_n)) <= case.solver.epsilon
