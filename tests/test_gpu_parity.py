"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Exact mode must be BIT-IDENTICAL to the reference (fields, tau sequence,
Picard iteration counts, last_delta, clamp counts, error lines). The oracle is
the C restatement (pinned to the reference itself by test_oracle_pin.py and to
the committed fixtures by test_golden.py).
"""
import math
import os

import numpy as np
import pytest

from oracle.oracle import OracleError, PortStepper, port_thomas_batch
from paper_1912_03744_b200 import configs
from paper_1912_03744_b200.errors import LineError, TableRangeError, TauFloorError
from paper_1912_03744_b200.materials import HalfPointRule, RangePolicy
from paper_1912_03744_b200.solver import make_field
from paper_1912_03744_b200.source import FieldSource, NullSource

from helpers import gpu_stepper, to_dev, to_host

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden_cases():
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(GOLD, "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    return mg.CASES


def _seq(results):
    return np.array([[r.tau_used, r.halvings, r.radial.iterations, r.axial.iterations,
                      r.radial.last_delta, r.axial.last_delta] for r in results])


@pytest.mark.parametrize("case_def", _golden_cases(), ids=lambda c: c[0])
def test_exact_matches_golden_bitwise(cuda, case_def, stepper_path):
    name, build, init, steps, t0 = case_def
    z = np.load(os.path.join(GOLD, f"{name}.npz"))
    case = build()
    gpu = gpu_stepper(case, "exact")
    f = to_dev(np.asfortranarray(z["initial"]))
    t_end, stats, res = gpu.run(f, float(z["t0"]), int(z["steps"]), keep_results=True)
    assert np.array_equal(_seq(res), z["seq"])
    assert t_end == float(z["t_end"])
    m = case.grid().mask()
    assert np.array_equal(to_host(f)[m], z["final"][m])
    assert gpu.clamp_events() == [int(v) for v in z["clamp"]]
    assert (gpu.resident_stats()["grid"] > 0) == (stepper_path == "resident")


def test_exact_cfg0_2000_steps_bitwise(cuda, stepper_path):
    """configs[0] in full: 100 x 200, tau = 1e-4, 2000 steps."""
    case = configs.cfg0(2000)
    g = case.grid()
    port = PortStepper(case)
    fo = make_field(g, case.solver.T0)
    te_o, st_o, res_o = port.run(fo, 0.0, case.steps)
    gpu = gpu_stepper(case, "exact")
    fg = to_dev(make_field(g, case.solver.T0))
    te_g, st_g, res_g = gpu.run(fg, 0.0, case.steps, keep_results=True)
    assert te_g == te_o
    assert np.array_equal(_seq(res_g), _seq(res_o))
    m = g.mask()
    assert np.array_equal(to_host(fg)[m], fo[m])
    assert max(r.radial.iterations for r in res_o) >= 2  # nonlinear Picard work happened


@pytest.mark.parametrize("nr_div,nz", [
    ([1, 1, 1, 1], 1),     # 4 x 1: a single row / single-cell lines
    ([1, 1, 1, 1], 2),
    ([2, 1, 1, 1], 3),     # odd line counts: no TMA (16-B row alignment)
    ([9, 1, 4, 2], 33),    # one past a 32-line CTA, one past a 16-row tile
    ([13, 1, 1, 1], 32),   # exactly one CTA of lines, exactly one radial tile
    ([25, 2, 3, 2], 64),   # two axial tiles of 32 rows, 32 radial rows (two tiles)
    ([40, 3, 9, 3], 97),
])
def test_exact_edge_grids_bitwise(cuda, nr_div, nz, stepper_path):
    """Grids at and around the kernels' tile and CTA boundaries (and below
    them) against the oracle: fields, tau / iteration / delta sequences."""
    case = configs.scaled(configs.cfg0(12), nr_div, nz)
    g = case.grid()
    port = PortStepper(case)
    f0 = configs.smooth_field(g, 30.0)
    fo = f0.copy(order="F")
    gpu = gpu_stepper(case, "exact")
    fg = to_dev(f0.copy(order="F"))
    try:
        te_o, _, res_o = port.run(fo, 0.0, case.steps)
    except OracleError as e:  # the reference gives up (tau floor): so must the GPU
        with pytest.raises(TauFloorError):
            gpu.run(fg, 0.0, case.steps)
        assert "fell below floor" in str(e)
        return
    te_g, _, res_g = gpu.run(fg, 0.0, case.steps, keep_results=True)
    assert te_g == te_o
    assert np.array_equal(_seq(res_g), _seq(res_o))
    m = g.mask()
    assert np.array_equal(to_host(fg)[m], fo[m])


def test_exact_rcp_redo_path_bitwise(cuda, monkeypatch):
    """The line solvers' fallback for a flagged pivot (the tile redone with
    __drcp_rn from the saved recurrence state), forced on every full tile."""
    monkeypatch.setenv("PCGPU_RCP_REDO", "1")
    case = configs.cfg0(200)
    g = case.grid()
    port = PortStepper(case)
    fo = make_field(g, case.solver.T0)
    te_o, _, res_o = port.run(fo, 0.0, case.steps)
    gpu = gpu_stepper(case, "exact")
    fg = to_dev(make_field(g, case.solver.T0))
    te_g, _, res_g = gpu.run(fg, 0.0, case.steps, keep_results=True)
    assert te_g == te_o
    assert np.array_equal(_seq(res_g), _seq(res_o))
    m = g.mask()
    assert np.array_equal(to_host(fg)[m], fo[m])


@pytest.mark.parametrize("rule", list(HalfPointRule))
@pytest.mark.parametrize("api", ["device", "host"])
def test_exact_half_steps_bitwise(cuda, rule, api):
    case = configs.step_cell(True, halfpoint_rule=rule)
    g = case.grid()
    port, gpu = PortStepper(case), gpu_stepper(case, "exact")
    f = configs.smooth_field(g, 30.0)
    for tau in (2e-3, 5e-2):
        ho = make_field(g, 0.0)
        r_o = port.radial_half_step(f, 0.0, tau, ho)
        if api == "host":
            hg = make_field(g, 0.0)
            r_g = gpu.radial_half_step(f, 0.0, tau, hg)
        else:
            hgd = to_dev(make_field(g, 0.0))
            r_g = gpu.radial_half_step(to_dev(f), 0.0, tau, hgd)
            hg = to_host(hgd)
        assert r_g == r_o
        m = g.mask()
        assert np.array_equal(hg[m], ho[m])
        no = make_field(g, 0.0)
        a_o = port.axial_half_step(ho, 0.0, tau, no)
        if api == "host":
            ng = make_field(g, 0.0)
            a_g = gpu.axial_half_step(ho, 0.0, tau, ng)
        else:
            ngd = to_dev(make_field(g, 0.0))
            a_g = gpu.axial_half_step(to_dev(ho), 0.0, tau, ngd)
            ng = to_host(ngd)
        assert a_g == a_o
        assert np.array_equal(ng[m], no[m])


def test_equilibrium_one_iteration(cuda):
    """test_solver.cpp:217-244."""
    case = configs.step_cell(True, source=configs.SOURCE_NULL)
    g = case.grid()
    gpu = gpu_stepper(case, "exact", NullSource())
    f = make_field(g, case.solver.T0)
    out = make_field(g, 0.0)
    r = gpu.radial_half_step(f, 0.0, 1e-3, out)
    assert r.converged and r.iterations == 1
    assert np.abs(out[g.mask()] - 4.2).max() <= 1e-13
    out2 = make_field(g, 0.0)
    r2 = gpu.axial_half_step(out, 0.0, 1e-3, out2)
    assert r2.converged and r2.iterations == 1
    assert np.abs(out2[g.mask()] - 4.2).max() <= 1e-13


def test_constant_coefficients_two_iterations_exact_zero(cuda):
    """test_solver.cpp:246-266: identical rebuilt system, identical solve."""
    case = configs.step_cell(False, source=configs.SOURCE_NULL)
    g = case.grid()
    gpu = gpu_stepper(case, "exact", NullSource())
    f = configs.smooth_field(g)
    out = make_field(g, 0.0)
    r = gpu.radial_half_step(f, 0.0, 2e-3, out)
    assert r.converged and r.iterations == 2 and r.last_delta == 0.0
    out2 = make_field(g, 0.0)
    r2 = gpu.axial_half_step(out, 0.0, 2e-3, out2)
    assert r2.converged and r2.iterations == 2 and r2.last_delta == 0.0


def test_max_iter_one_forces_halving(cuda):
    """test_solver.cpp:319-338."""
    case = configs.step_cell(True, max_iter=1)
    g = case.grid()
    gpu = gpu_stepper(case, "exact")
    f = to_dev(configs.smooth_field(g, 20.0))
    t = 0.001
    tau0 = gpu.initial_tau(t)
    r = gpu.step(f, t)
    assert r.halvings >= 1
    assert r.tau_used == tau0 / 2 ** r.halvings
    assert r.radial.converged and r.axial.converged


def test_tau_floor_raises(cuda, stepper_path):
    """test_solver.cpp:340-352; TauFloorError carries the reference's tau,
    floor and time (solver.cpp:371)."""
    case = configs.step_cell(True, max_iter=1)
    case.solver.tau_min = 0.9 * 1e-7
    f0 = configs.smooth_field(case.grid(), 20.0)
    port = PortStepper(case)
    with pytest.raises(OracleError) as eo:
        port.step(f0.copy(order="F"), 0.001)
    gpu = gpu_stepper(case, "exact")
    fg = to_dev(f0)
    with pytest.raises(TauFloorError) as eg:
        gpu.step(fg, 0.001)
    assert "fell below floor" in str(eo.value) and "fell below floor" in str(eg.value)
    tau = gpu.initial_tau(0.001)
    while tau >= case.solver.tau_min:  # step()'s halving sequence (solver.cpp:368-371)
        tau *= 0.5
    assert (eg.value.tau, eg.value.floor, eg.value.time) == (tau, case.solver.tau_min, 0.001)
    m = case.grid().mask()
    assert np.array_equal(to_host(fg)[m], f0[m])  # the field is left untouched


def test_resident_batches_and_host_redo_bitwise(cuda, monkeypatch):
    """The resident stepper runs a whole fixed-dt run in one batch (one
    cooperative launch, one host sync); a step with more halvings than the
    batch precomputed (forced with PCGPU_RES_MAX_HALV=0) is redone
    host-driven from the intact field, with its clamp events counted once."""
    case = configs.cfg0(300)
    gpu = gpu_stepper(case, "exact")
    g = case.grid()
    fg = to_dev(make_field(g, case.solver.T0))
    l0 = gpu.launch_count()
    gpu.run(fg, 0.0, case.steps)
    st = gpu.resident_stats()
    assert st["grid"] > 0 and st["batches"] == 1 and st["steps"] == case.steps
    assert gpu.launch_count() - l0 == 1  # the whole run is one kernel launch
    z = np.load(os.path.join(GOLD, "cfg0_coarse_halving.npz"))
    name, build, init, steps, t0 = [c for c in _golden_cases() if c[0] == "cfg0_coarse_halving"][0]
    monkeypatch.setenv("PCGPU_RES_MAX_HALV", "0")
    case2 = build()
    gpu2 = gpu_stepper(case2, "exact")
    f = to_dev(np.asfortranarray(z["initial"]))
    t_end, stats, res = gpu2.run(f, float(z["t0"]), int(z["steps"]), keep_results=True)
    assert np.array_equal(_seq(res), z["seq"]) and t_end == float(z["t_end"])
    assert np.array_equal(to_host(f)[case2.grid().mask()], z["final"][case2.grid().mask()])
    assert gpu2.clamp_events() == [int(v) for v in z["clamp"]]
    st2 = gpu2.resident_stats()
    assert st2["host_steps"] == sum(1 for r in res if r.halvings > 0) > 0


def test_speculative_batches_bitwise(cuda, monkeypatch):
    """Host-driven runs (the configs[3] path) enqueue batches of steps with the
    predicted Picard counts and read once per batch: configs[0]'s 2000 steps
    mostly in batches, and a run whose counts change and that halves, where
    batches are undone and replayed -- both bit for bit against the C
    restatement, with the clamp counts; and the step-by-step path
    (PCGPU_NO_SPECULATE) for comparison."""
    monkeypatch.setenv("PCGPU_RESIDENT", "0")
    case = configs.cfg0(2000)
    g = case.grid()
    port = PortStepper(case)
    fo = make_field(g, case.solver.T0)
    te_o, _, res_o = port.run(fo, 0.0, case.steps)
    gpu = gpu_stepper(case, "exact")
    fg = to_dev(make_field(g, case.solver.T0))
    te_g, _, res_g = gpu.run(fg, 0.0, case.steps, keep_results=True)
    assert te_g == te_o and np.array_equal(_seq(res_g), _seq(res_o))
    assert np.array_equal(to_host(fg)[g.mask()], fo[g.mask()])
    sp = gpu.speculation_stats()
    assert sp["steps"] > case.steps // 2, sp
    z = np.load(os.path.join(GOLD, "cfg0_coarse_halving.npz"))
    name, build, init, steps, t0 = [c for c in _golden_cases() if c[0] == "cfg0_coarse_halving"][0]
    for spec in (True, False):
        if not spec:
            monkeypatch.setenv("PCGPU_NO_SPECULATE", "1")
        case2 = build()
        gpu2 = gpu_stepper(case2, "exact")
        f = to_dev(np.asfortranarray(z["initial"]))
        t_end, _, res = gpu2.run(f, float(z["t0"]), int(z["steps"]), keep_results=True)
        assert np.array_equal(_seq(res), z["seq"]) and t_end == float(z["t_end"])
        assert np.array_equal(to_host(f)[case2.grid().mask()], z["final"][case2.grid().mask()])
        assert gpu2.clamp_events() == [int(v) for v in z["clamp"]]
        sp2 = gpu2.speculation_stats()
        if spec:
            assert sp2["batches"] > 0 and sp2["rollbacks"] > 0, sp2
        else:
            assert sp2["batches"] == 0


def test_field_source_rejected_by_whole_steps(cuda):
    """A FIELD source's power is bound per half-step (the caller binds it
    before each half-step): step / run / evolve refuse it (ConfigError)
    instead of stepping with an unbound or stale power field."""
    from paper_1912_03744_b200.errors import ConfigError
    case = configs.step_cell(True)
    g = case.grid()
    gpu = gpu_stepper(case, "exact", source=FieldSource(g))
    with pytest.raises(ConfigError):
        gpu.step(to_dev(configs.smooth_field(g)), 0.0)
    with pytest.raises(ConfigError):
        gpu.run(to_dev(configs.smooth_field(g)), 0.0, 2)


def test_strict_range_lowest_line(cuda):
    case = configs.step_cell(True, range_policy=RangePolicy.Strict)
    g = case.grid()
    f = configs.smooth_field(g)
    f[3, 5] = 500.0
    f[9, 2] = 600.0
    port, gpu = PortStepper(case), gpu_stepper(case, "exact")
    with pytest.raises(OracleError) as eo:
        port.radial_half_step(f, 0.0, 1e-3, make_field(g, 0.0))
    with pytest.raises(LineError) as eg:
        gpu.radial_half_step(f, 0.0, 1e-3, make_field(g, 0.0))
    assert eg.value.cause is TableRangeError
    assert eg.value.line == eo.value.line


def _heat_sum(case, f):
    """weighted_heat_sum (solver.cpp:103-119), Kahan-summed."""
    g = case.grid()
    s = comp = 0.0
    for i in range(g.nr()):
        mat = case.materials[g.layer(i)]
        for j in range(g.col_extent(i)):
            cv = mat.cv(f[i, j])
            term = g.r_center(i) * g.control_r(i) * g.control_z(j) * mat.rho() * cv * f[i, j]
            y = term - comp
            t = s + y
            comp = (t - s) - y
            s = t
    return s


def test_conservation_all_neumann(cuda):
    """test_solver.cpp:354-369: source-free heat is conserved."""
    case = configs.step_cell(False, source=configs.SOURCE_NULL, all_neumann=True)
    gpu = gpu_stepper(case, "exact", NullSource())
    f = configs.smooth_field(case.grid(), 12.0)
    before = _heat_sum(case, f)
    fd = to_dev(f)
    t = 0.0
    for _ in range(30):
        t += gpu.step(fd, t).tau_used
    after = _heat_sum(case, to_host(fd))
    assert abs(after - before) / abs(before) <= 1e-11


def test_z_independence(cuda):
    """test_solver.cpp:433-468."""
    case = configs.step_cell(True, source=configs.SOURCE_NULL, all_neumann=True)
    case.domain.outer_length = case.domain.core_length
    g = case.grid()
    gpu = gpu_stepper(case, "exact", NullSource())
    f = make_field(g, 4.2)
    for i in range(g.nr()):
        f[i, :] = 5.0 + math.cos(2.0 * g.r_center(i))
    fd = to_dev(f)
    t = 0.0
    for _ in range(20):
        t += gpu.step(fd, t).tau_used
    h = to_host(fd)
    assert np.abs(h - h[:, :1]).max() <= 1e-12


class _Manufactured(FieldSource):
    """T-independent per-cell power (the acceptance suite's MMS pattern)."""

    def power_field(self, grid, t):
        r = grid.r_centers[:, None]
        z = grid.z_centers[None, :]
        return np.asfortranarray(1e3 * np.exp(-5 * t) * np.cos(np.pi * r * r) * np.cos(0.5 * np.pi * z)
                                 + 0 * r * z)


def test_field_source_half_steps_bitwise(cuda):
    case = configs.step_cell(True, source=configs.SOURCE_FIELD)
    g = case.grid()
    src = _Manufactured(g)
    gpu = gpu_stepper(case, "exact", src)
    port = PortStepper(case)
    f = configs.smooth_field(g, 10.0)
    t, tau = 0.01, 1e-3
    port.bind_power_field(src.power_field(g, t + 0.5 * tau))
    ho, hg = make_field(g, 0.0), make_field(g, 0.0)
    assert gpu.radial_half_step(f, t, tau, hg) == port.radial_half_step(f, t, tau, ho)
    assert np.array_equal(hg[g.mask()], ho[g.mask()])
    no, ng = make_field(g, 0.0), make_field(g, 0.0)
    assert gpu.axial_half_step(ho, t, tau, ng) == port.axial_half_step(ho, t, tau, no)
    assert np.array_equal(ng[g.mask()], no[g.mask()])


@pytest.mark.parametrize("kind", ["exact-lean", "exact-x"])
def test_field_source_exact_lookups_half_steps_bitwise(cuda, kind, monkeypatch):
    """A bound per-cell source on the power-law tables: the ws kernels' aux
    staging with both exact lookup variants, odd and even slab widths."""
    if kind == "exact-x":
        monkeypatch.setenv("PCGPU_NO_EXACTLEAN", "1")
    case = configs.scaled(configs.cfg4(), [44, 5, 13, 3], 128, 87)
    case.source_kind = configs.SOURCE_FIELD
    g = case.grid()
    src = _Manufactured(g)
    gpu = gpu_stepper(case, "exact", src)
    assert f"lookups={kind} " in gpu.describe()
    port = PortStepper(case)
    f = configs.smooth_field(g, 10.0)
    t, tau = 0.01, 1e-5
    port.bind_power_field(src.power_field(g, t + 0.5 * tau))
    ho, hg = make_field(g, 0.0), make_field(g, 0.0)
    assert gpu.radial_half_step(f, t, tau, hg) == port.radial_half_step(f, t, tau, ho)
    assert np.array_equal(hg[g.mask()], ho[g.mask()])
    no, ng = make_field(g, 0.0), make_field(g, 0.0)
    assert gpu.axial_half_step(ho, t, tau, ng) == port.axial_half_step(ho, t, tau, no)
    assert np.array_equal(ng[g.mask()], no[g.mask()])


@pytest.mark.parametrize("layout", [0, 1])
def test_tridiag_batch_exact_bitwise(cuda, layout):
    import torch
    from paper_1912_03744_b200.tridiagonal import thomas_solve_batch
    z = np.load(os.path.join(GOLD, "thomas_batch.npz"))
    batch, n = z["x"].shape
    if layout == 0:
        host = [np.ascontiguousarray(z[k].reshape(-1)) for k in ("lower", "diag", "upper", "rhs")]
    else:
        host = [np.ascontiguousarray(z[k].T.reshape(-1)) for k in ("lower", "diag", "upper", "rhs")]
    dev = [torch.from_numpy(h).cuda() for h in host]
    x = torch.empty_like(dev[3])
    thomas_solve_batch(*dev, x, n, batch, layout, exact=True)
    got = x.cpu().numpy()
    want = z["x"].reshape(-1) if layout == 0 else np.ascontiguousarray(z["x"].T).reshape(-1)
    assert np.array_equal(got, want)


def test_tridiag_cfg1_full_size_vs_reference(cuda):
    """configs[1] in full -- 131072 systems of length 1024 drawn from
    std::mt19937_64(2024) as SURVEY 8(d) specifies -- in both layouts, every
    system bit for bit against the reference's own thomas_solve_inplace over a
    LinePool of all host cores (the C restatement without the reference)."""
    import torch
    from oracle.oracle import port_thomas_batch, ref_available, ref_thomas_batch
    from paper_1912_03744_b200.tridiagonal import CONTIGUOUS, STRIDED, thomas_solve_batch
    from tools.bench_tridiag import generate
    batch, n = 131072, 1024
    a, b, c, d = generate(batch, n)
    bands = [v.ravel() for v in (a, b, c, d)]
    if ref_available():
        rc, want, _ = ref_thomas_batch(*bands, n, batch, 0, workers=os.cpu_count() or 1)
    else:
        rc, want, _ = port_thomas_batch(*bands, n, batch, 0)
    assert rc == 0
    want = want.reshape(batch, n)
    for layout in (CONTIGUOUS, STRIDED):
        host = (a, b, c, d) if layout == CONTIGUOUS else tuple(v.T for v in (a, b, c, d))
        dev = [torch.from_numpy(np.ascontiguousarray(v)).cuda().view(-1) for v in host]
        x = torch.empty_like(dev[3])
        thomas_solve_batch(*dev, x, n, batch, layout)
        got = x.view(batch, n) if layout == CONTIGUOUS else x.view(n, batch).t()
        assert np.array_equal(got.cpu().numpy(), want), layout
        del dev, x
        torch.cuda.empty_cache()


def test_tridiag_batch_rejects_bad_tensors(cuda):
    """The binding validates dtype, contiguity, size and device before any
    pointer reaches the kernels (an out-of-bounds write otherwise)."""
    import torch
    from paper_1912_03744_b200.tridiagonal import thomas_solve_batch
    n, batch = 8, 4
    ok = [torch.ones(n * batch, dtype=torch.float64, device="cuda") for _ in range(5)]
    bad_dtype = ok[:3] + [ok[3].float(), ok[4]]
    with pytest.raises(ValueError):
        thomas_solve_batch(*bad_dtype, n, batch)
    strided = torch.ones(2 * n * batch, dtype=torch.float64, device="cuda")[::2]
    with pytest.raises(ValueError):
        thomas_solve_batch(*ok[:4], strided, n, batch)
    with pytest.raises(ValueError):
        thomas_solve_batch(*ok[:4], ok[4][:-1], n, batch)
    with pytest.raises(ValueError):
        thomas_solve_batch(*ok[:4], ok[4].cpu(), n, batch)


@pytest.mark.parametrize("n,batch", [(2, 1), (16, 32), (30, 33), (1024, 200), (1000, 97),
                                     (7, 40)])
def test_tridiag_batch_contiguous_fused_ragged(cuda, n, batch):
    """The fused contiguous kernel (TMA tiles of 16 rows x 32 systems) on sizes
    that are not multiples of its tiles, bit for bit against the C restatement
    of thomas_solve_inplace and against the transpose path (exact = 3); odd n
    takes the transpose path (no 16-B row stride for TMA)."""
    import ctypes as C
    import torch
    from oracle.oracle import port_thomas_batch
    from paper_1912_03744_b200 import _native as N
    from paper_1912_03744_b200.tridiagonal import thomas_solve_batch
    rng = np.random.default_rng(n * 1000 + batch)
    a = -rng.random((batch, n))
    c = -rng.random((batch, n))
    a[:, 0] = 0.0
    c[:, -1] = 0.0
    b = 2.05 + np.abs(a) + np.abs(c)
    d = rng.random((batch, n)) * 2 - 1
    host = [np.ascontiguousarray(v).reshape(-1) for v in (a, b, c, d)]
    dev = [torch.from_numpy(h).cuda() for h in host]
    x = torch.empty_like(dev[3])
    thomas_solve_batch(*dev, x, n, batch, 0, exact=True)
    rc, xo, _ = port_thomas_batch(*host, n, batch, 0)
    assert rc == 0
    assert np.array_equal(x.cpu().numpy(), xo)
    x3 = torch.empty_like(dev[3])
    failed = C.c_int64(-1)
    assert N.load().pcgpu_tridiag_batch(*(C.c_void_p(t.data_ptr()) for t in (*dev, x3)), n, batch,
                                        0, 3, None, C.byref(failed)) == N.OK
    assert torch.equal(x, x3)


def test_tridiag_batch_zero_pivot_fused(cuda):
    import torch
    from paper_1912_03744_b200.tridiagonal import thomas_solve_batch
    n, batch = 48, 70
    b = torch.ones(n * batch, dtype=torch.float64, device="cuda")
    b[65 * n + 17] = 0.0
    b[40 * n + 47] = 0.0
    z = torch.zeros_like(b)
    with pytest.raises(LineError) as e:
        thomas_solve_batch(z, b, z, torch.ones_like(b), torch.empty_like(b), n, batch, 0)
    assert e.value.line == 40


def test_tridiag_batch_zero_pivot(cuda):
    import torch
    from paper_1912_03744_b200.tridiagonal import thomas_solve_batch
    n, batch = 5, 8
    b = torch.ones(n * batch, dtype=torch.float64, device="cuda")
    b[3 * n + 2] = 0.0
    b[6 * n] = 0.0
    z = torch.zeros_like(b)
    with pytest.raises(LineError) as e:
        thomas_solve_batch(z, b, z, torch.ones_like(b), torch.empty_like(b), n, batch, 0)
    assert e.value.line == 3


def _rel(a, b, m):
    return float(np.max(np.abs(a[m] - b[m])) / np.max(np.abs(b[m])))


def test_exact_cfg3_full_size_vs_reference(cuda):
    """configs[3] at its full BASELINE size (8192 x 16384, 134M cells): two
    exact-mode steps bit for bit against the reference's own AdiStepper
    (oracle/_ref, on all host cores; the C restatement if the reference library
    is absent) -- fields, tau, iteration counts and last_delta."""
    import torch
    from oracle.oracle import RefStepper, ref_available
    case = configs.cfg3()
    g = case.grid()
    steps = 2
    cpu = (RefStepper(case, workers=os.cpu_count() or 1) if ref_available()
           else PortStepper(case))
    fo = make_field(g, case.solver.T0)
    te_o, _, res_o = cpu.run(fo, 0.0, steps)
    del cpu
    gpu = gpu_stepper(case, "exact")
    fg = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64, device="cuda").t()
    te_g, _, res_g = gpu.run(fg, 0.0, steps, keep_results=True)
    assert te_g == te_o
    assert np.array_equal(_seq(res_g), _seq(res_o))
    assert min(r.radial.iterations for r in res_o) >= 2  # nonlinear Picard work happened
    m = g.mask()
    got = to_host(fg)
    assert np.array_equal(got[m], fo[m])
    assert not np.array_equal(fo[m], make_field(g, case.solver.T0)[m])


# ---------------------------------------------------------------------------
# Partitioned (multi-GPU) stepper, P ranks emulated in-process on one GPU:
# bit-identical to the single-GPU stepper of the same mode; in
# exact mode that is the reference itself.
@pytest.mark.parametrize("name,nranks,steps", [
    ("cfg0", 2, 30), ("cfg0", 3, 30), ("cfg4s", 4, 6), ("cfg4s", 8, 6), ("cfg4s", 1, 4),
])
@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_partitioned_exact_emulated_bitwise(cuda, name, nranks, steps, transport, monkeypatch):
    from paper_1912_03744_b200.dist import PartitionedAdi
    if transport == "nccl":  # all-to-all transposes (memcpy stand-ins when emulated)
        monkeypatch.setenv("PCGPU_DIST_TRANSPORT", "nccl")
    case = configs.cfg0() if name == "cfg0" else \
        configs.scaled(configs.cfg4(), [706, 71, 212, 35], 2048, 1400)
    g = case.grid()
    src = configs.make_source(case, g)
    single = gpu_stepper(case, "exact")
    f1 = to_dev(make_field(g, case.solver.T0))
    _, _, r1 = single.run(f1, 0.0, steps, keep_results=True)
    part = PartitionedAdi(g, case.materials, src, case.timing, case.solver, device=0,
                          emulate=nranks, mode="exact")
    f0 = to_dev(make_field(g, case.solver.T0))
    part.set_field(f0)
    part.enable_timing(True)
    _, _, r2 = part.run(0.0, steps, keep_results=True)
    out = to_dev(make_field(g, 0.0))
    part.get_field(out)
    assert _seq(r1).tolist() == _seq(r2).tolist()
    m = g.mask()
    assert np.array_equal(to_host(out)[m], to_host(f1)[m])
    assert part.transport() == transport
    tm = part.timing()
    assert tm["transposes"] == (3 * steps if transport == "nccl" else 0)
    assert tm["allreduces"] > 0


@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_partitioned_exact_host_fields_bitwise(cuda, transport, monkeypatch):
    """The host-field entry points of the partitioned stepper (each rank moves
    only its state lines): step by step through host memory, as the bench's
    multi-GPU e2e does, against the single-GPU host-field stepper."""
    from paper_1912_03744_b200.dist import PartitionedAdi
    if transport == "nccl":
        monkeypatch.setenv("PCGPU_DIST_TRANSPORT", "nccl")
    case = configs.cfg0()
    g = case.grid()
    src = configs.make_source(case, g)
    single = gpu_stepper(case, "exact")
    f1 = make_field(g, case.solver.T0)
    part = PartitionedAdi(g, case.materials, src, case.timing, case.solver, device=0,
                          emulate=3, mode="exact")
    f2 = make_field(g, case.solver.T0)
    t = 0.0
    for _ in range(12):
        r1 = single.step(f1, t)
        part.set_field_host(f2)
        _, _, r2 = part.run(t, 1, keep_results=True)
        part.get_field_host(f2)
        assert _seq([r1]).tolist() == _seq(r2).tolist()
        t += r1.tau_used
    m = g.mask()
    assert np.array_equal(f2[m], f1[m])
    with pytest.raises(ValueError):
        part.get_field_host(np.zeros((g.nr(), g.nz())))  # C order


@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_partitioned_exact_halving_and_clamps_vs_oracle(cuda, transport, monkeypatch):
    """Partitioned exact run with tau halvings and clamp events, against the
    oracle (the reference's algorithm) directly."""
    from paper_1912_03744_b200.dist import PartitionedAdi
    if transport == "nccl":
        monkeypatch.setenv("PCGPU_DIST_TRANSPORT", "nccl")
    case = _cfg4s()
    g = case.grid()
    f = make_field(g, case.solver.T0)
    f[10:12, 20:23] = 3.9
    f[46, 30:32] = 3.95
    f[50:52, 5:7] = 3.95
    port = PortStepper(case)
    fo = f.copy(order="F")
    _, _, res_o = port.run(fo, 0.0, 6)
    assert sum(r.halvings for r in res_o) > 0
    part = PartitionedAdi(g, case.materials, configs.make_source(case, g), case.timing,
                          case.solver, device=0, emulate=3, mode="exact")
    part.set_field(to_dev(f))
    _, _, res_p = part.run(0.0, 6, keep_results=True)
    out = to_dev(make_field(g, 0.0))
    part.get_field(out)
    assert np.array_equal(_seq(res_p), _seq(res_o))
    m = g.mask()
    assert np.array_equal(to_host(out)[m], fo[m])


# ---------------------------------------------------------------------------
# BASELINE growth controller (configs[2]/[4]): identical decisions on GPU and
# the oracle, bit for bit.
@pytest.mark.parametrize("name", ["cfg2s", "cfg4s"])
def test_growth_controller_matches_oracle(cuda, name, stepper_path):
    from paper_1912_03744_b200.solver import GrowthPolicy
    base = configs.cfg2() if name == "cfg2s" else configs.cfg4()
    case = configs.scaled(base, [44, 5, 13, 3], 128, 87 if name == "cfg4s" else 128)
    g = case.grid()
    pol = GrowthPolicy()
    port = PortStepper(case)
    fo = make_field(g, case.solver.T0)
    t_o, st_o, res_o = port.run_growth(fo, 0.0, 0.35, 400, pol)
    assert st_o["steps"] > 50 and max(r.tau_used for r in res_o) > 1e-4  # it grew
    gpu = gpu_stepper(case, "exact")
    fg = to_dev(make_field(g, case.solver.T0))
    t_g, st_g, res_g = gpu.run_growth(fg, 0.0, 0.35, 400, pol, keep_results=True)
    sg, so = _seq(res_g), _seq(res_o)
    assert t_g == t_o and np.array_equal(sg, so)  # dt, halvings, iterations, last_delta
    assert np.array_equal(to_host(fg)[g.mask()], fo[g.mask()])


def test_growth_controller_cfg2_full_size_vs_reference(cuda):
    """configs[2] at its full BASELINE size (1024 x 2048) for 200 growth-
    controller steps: the B200 against the reference's OWN half-steps under
    the same controller (pcref_run_growth, all host cores) -- identical
    accepted-dt / halving / Picard-iteration / last_delta sequences and a
    bit-identical field (north star: identical sequences, <= 1e-6)."""
    from oracle.oracle import RefStepper, ref_available
    from paper_1912_03744_b200.solver import GrowthPolicy
    if not ref_available():
        pytest.skip("the reference library (oracle/_ref) is not built")
    case = configs.cfg2()
    g = case.grid()
    steps = 200
    ref = RefStepper(case, workers=os.cpu_count() or 1)
    fo = make_field(g, case.solver.T0)
    t_o, _, res_o = ref.run_growth(fo, 0.0, case.t_end, steps, GrowthPolicy())
    del ref
    gpu = gpu_stepper(case, "exact")
    fg = to_dev(make_field(g, case.solver.T0))
    t_g, _, res_g = gpu.run_growth(fg, 0.0, case.t_end, steps, GrowthPolicy(), keep_results=True)
    assert len(res_o) == len(res_g) == steps and t_g == t_o
    assert np.array_equal(_seq(res_g), _seq(res_o))
    assert max(r.tau_used for r in res_o) > 1e-5  # the controller grew tau
    assert np.array_equal(to_host(fg)[g.mask()], fo[g.mask()])


@pytest.mark.parametrize("name,steps", [("cfg2", 8), ("cfg4", 4)])
def test_growth_controller_full_size_exact(cuda, name, steps):
    """configs[2] (1024 x 2048) and configs[4] (2048 x 4096 stepped cell) at their
    full BASELINE sizes: the first steps of the growth controller, exact mode,
    bit for bit against the C restatement (fields, dt, halvings, iterations,
    last_delta)."""
    case = configs.cfg2() if name == "cfg2" else configs.cfg4()
    g = case.grid()
    port = PortStepper(case)
    fo = make_field(g, case.solver.T0)
    t_o, _, res_o = port.run_growth(fo, 0.0, case.t_end, steps)
    gpu = gpu_stepper(case, "exact")
    fg = to_dev(make_field(g, case.solver.T0))
    t_g, _, res_g = gpu.run_growth(fg, 0.0, case.t_end, steps, keep_results=True)
    assert t_g == t_o and len(res_g) == steps
    assert np.array_equal(_seq(res_g), _seq(res_o))
    assert np.array_equal(to_host(fg)[g.mask()], fo[g.mask()])


# ---- exact mode on the kernel variants the large configs select -------------
def _cfg4s():
    return configs.scaled(configs.cfg4(), [44, 5, 13, 3], 128, 87)


def test_exact_selects_ws_and_exact_x_for_configs(cuda):
    gpu = gpu_stepper(_cfg4s(), "exact")
    assert gpu.describe().startswith("mode=exact lines=ws lookups=exact-lean steps=resident:")
    gpu = gpu_stepper(configs.step_cell(True), "exact")
    assert gpu.describe().startswith("mode=exact lines=ws")


@pytest.fixture(params=["exact-lean", "exact-x"])
def lookup_kind(request, monkeypatch):
    """Both exact lookup variants the BASELINE configs can select (exact-x is
    what tables with per-layer knot grids get)."""
    if request.param == "exact-x":
        monkeypatch.setenv("PCGPU_NO_EXACTLEAN", "1")
    return request.param


def test_exact_x_out_of_range_clamp_events_bitwise(cuda, lookup_kind):
    """Cells below the power-law tables (4..300 K) in every layer: clamp events
    are counted per layer exactly as the reference counts them, and the fields
    stay bit-identical. (A hot spot above 300 K in a 4.2 K cell makes the
    reference itself fail its tau floor, so only the lower clamp is driven.)"""
    case = _cfg4s()
    g = case.grid()
    f = make_field(g, case.solver.T0)
    f[10:12, 20:23] = 3.9
    f[46, 30:32] = 3.95
    f[50:52, 5:7] = 3.95
    f[63, 40] = 3.97
    port, gpu = PortStepper(case), gpu_stepper(case, "exact")
    assert f"lookups={lookup_kind} " in gpu.describe()
    fo = f.copy(order="F")
    te_o, _, res_o = port.run(fo, 0.0, 6)
    fg = to_dev(f)
    te_g, _, res_g = gpu.run(fg, 0.0, 6, keep_results=True)
    assert te_g == te_o
    assert np.array_equal(_seq(res_g), _seq(res_o))
    m = g.mask()
    assert np.array_equal(to_host(fg)[m], fo[m])
    assert gpu.clamp_events() == port.clamp_events()
    assert sum(port.clamp_events()) > 0
    assert sum(1 for c in port.clamp_events() if c) >= 2


def test_exact_x_strict_range_lowest_line(cuda, lookup_kind):
    case = _cfg4s()
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


# ---- host-field steps with the copy-in pipelined into the radial sweep ----
def _host_steps(port, gpu, f, t0, n):
    """n steps through pcgpu_step_host (gpu) and the oracle on copies of f."""
    fo, fg = f.copy(order="F"), f.copy(order="F")
    res_o, res_g, t = [], [], t0
    for _ in range(n):
        ro = port.step(fo, t)
        rg = gpu.step(fg, t)
        res_o.append(ro)
        res_g.append(rg)
        t += ro.tau_used
    return fo, fg, res_o, res_g


@pytest.mark.parametrize("name", ["cfg0_nz1024", "cfg4s", "coarse_halving"])
def test_host_step_pipelined_bitwise(cuda, monkeypatch, name):
    """pcgpu_step_host with the field copied in as row blocks while K3 and the
    first radial iterations run on the blocks already there: bit-identical to
    the oracle step by step (fields, tau / halvings / iterations / deltas),
    including the steps whose iteration count changes (redo path)."""
    monkeypatch.setenv("PCGPU_PIPELINE_MIN_NZ", "1")
    monkeypatch.setenv("PCGPU_RESIDENT", "0")  # the host-driven path takes host fields in blocks
    if name == "cfg0_nz1024":
        case, f0, t0, n = configs.scaled(configs.cfg0(), [69, 7, 21, 3], 1024), None, 0.0, 30
    elif name == "cfg4s":
        case, f0, t0, n = _cfg4s(), None, 0.0, 25
    else:
        case = configs.scaled(configs.cfg0(), [23, 3, 7, 2], 48)
        case.solver.tau_source_divisor = 10.0
        case.solver.max_iter = 6
        f0, t0, n = None, 0.02, 25
    g = case.grid()
    f = make_field(g, case.solver.T0) if f0 is None else f0
    port, gpu = PortStepper(case), gpu_stepper(case, "exact")
    fo, fg, res_o, res_g = _host_steps(port, gpu, f, t0, n)
    assert np.array_equal(_seq(res_g), _seq(res_o))
    m = g.mask()
    assert np.array_equal(fg[m], fo[m])
    assert gpu.clamp_events() == port.clamp_events()
    ps = gpu.pipeline_stats()
    assert ps["steps"] == n
    if name == "cfg0_nz1024":  # the iteration count ramps up from T0: redo path taken
        assert 1 <= ps["fallbacks"] < n
    if name == "coarse_halving":
        assert sum(r.halvings for r in res_o) > 0


def test_host_step_pipelined_clamps_and_strict(cuda, monkeypatch):
    """Clamp events counted only for the iterations the reference runs, and
    the reference's first failing line under the strict range policy."""
    monkeypatch.setenv("PCGPU_PIPELINE_MIN_NZ", "1")
    monkeypatch.setenv("PCGPU_RESIDENT", "0")
    case = _cfg4s()
    g = case.grid()
    f = make_field(g, case.solver.T0)
    f[10:12, 20:23] = 3.9
    f[46, 30:32] = 3.95
    f[50:52, 5:7] = 3.95
    port, gpu = PortStepper(case), gpu_stepper(case, "exact")
    fo, fg, res_o, res_g = _host_steps(port, gpu, f, 0.0, 6)
    assert np.array_equal(_seq(res_g), _seq(res_o))
    assert np.array_equal(fg[g.mask()], fo[g.mask()])
    assert gpu.clamp_events() == port.clamp_events() and sum(port.clamp_events()) > 0
    case2 = _cfg4s()
    case2.solver.range_policy = RangePolicy.Strict
    f2 = make_field(g, case2.solver.T0)
    f2[40, 70] = 500.0
    f2[20, 12] = 1.0
    port2, gpu2 = PortStepper(case2), gpu_stepper(case2, "exact")
    with pytest.raises(OracleError) as eo:
        port2.step(f2.copy(order="F"), 0.0)
    with pytest.raises(LineError) as eg:
        gpu2.step(f2.copy(order="F"), 0.0)
    assert eg.value.line == eo.value.line
    assert gpu2.pipeline_stats()["steps"] == 1
