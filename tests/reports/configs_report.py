"""TEST INFRASTRUCTURE (a report, not a test): every BASELINE.json config on one B200, next to the reference's own CPU path
on the same box's host cores. Prints one JSON object; the
committed copies live in profiles/ (r0N_configs_report.json).

  cfg0  100 x 200, tau 1e-4, 2000 steps: the whole run on the GPU (pcgpu_run)
        -- the resident stepper (one launch) and the host-driven path -- and
        the whole run through the reference's AdiStepper on all host cores;
        final fields compared bit for bit.
  paper the reference's own paper_cell.json (1210 x 100, transient pulse),
        3000 steps on the GPU and through the reference, bit for bit.
  cfg1  131072 x 1024 batched Thomas, both layouts (tools/bench_tridiag.py);
        the reference's thomas_solve_inplace over a bounded sample of systems
        on all host cores.
  cfg2  1024 x 2048, BASELINE growth controller, 5 pulse periods on the GPU;
        the first steps checked bit for bit against the C restatement's
        controller (the whole run against the reference's own half-steps is
        adaptive_full_parity.py); the reference AdiStepper timed on a bounded
        number of steps (its own tau controller) on all host cores.
  cfg4  2048 x 4096 stepped cell, growth controller, 10 periods; same checks.
cfg3 is bench.py's workload.

    python tests/reports/configs_report.py [--only cfg0,cfg2] [--periods-scale 1.0]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1912_03744_b200 import configs  # noqa: E402
from paper_1912_03744_b200.solver import AdiStepper, DevicePlan, make_field  # noqa: E402

CORES = os.cpu_count() or 1


def _gpu_stepper(case, g):
    return AdiStepper(g, case.materials, configs.make_source(case, g), case.timing, case.solver,
                      DevicePlan(0, "exact"))


def _dev_field(g, value):
    return torch.full((g.nz(), g.nr()), value, dtype=torch.float64, device="cuda").t()


def _host(f):
    return f.t().contiguous().cpu().numpy().T


def _ref_rate(case, steps, t0=0.0):
    """The reference AdiStepper (oracle/_ref) on all host cores: `steps` step()
    calls after one untimed warm-up step (bench.cpp:12-25)."""
    from oracle.oracle import RefStepper
    g = case.grid()
    ref = RefStepper(case, workers=CORES)
    f = make_field(g, case.solver.T0)
    t, _, _ = ref.run(f, t0, 1)
    s0 = time.perf_counter()
    _, st, _ = ref.run(f, t, steps)
    dt = time.perf_counter() - s0
    return {"value": st["cell_updates"] / dt, "unit": "cell-updates/s", "cores": CORES,
            "kind": "reference", "seconds": dt,
            "sample": f"{steps} step() calls after 1 warm-up ({st['cell_updates']:.3e} "
                      "cell-updates, the reference's own tau controller)"}


def _fixed_run(case, path):
    """The whole fixed-dt run on the GPU: `path` "resident" (one cooperative /
    cluster launch per batch) or "host" (host-driven Picard batches)."""
    os.environ["PCGPU_RESIDENT"] = "1" if path == "resident" else "0"
    g = case.grid()
    st = _gpu_stepper(case, g)
    f = _dev_field(g, case.solver.T0)
    st.run(_dev_field(g, case.solver.T0), 0.0, 5)  # warm-up (separate field)
    torch.cuda.synchronize()
    s0 = time.perf_counter()
    t_end, stats, _ = st.run(f, 0.0, case.steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - s0
    os.environ.pop("PCGPU_RESIDENT")
    return f, t_end, stats, dt, st.describe(), st.launch_count()


def cfg0(case=None, sample="the whole 2000-step run"):
    from oracle.oracle import RefStepper
    case = case or configs.cfg0()
    g = case.grid()
    fh, _, hstats, hdt, hdesc, _ = _fixed_run(case, "host")
    f, t_end, stats, dt, desc, launches = _fixed_run(case, "resident")
    ref = RefStepper(case, workers=CORES)
    fr = make_field(g, case.solver.T0)
    r0 = time.perf_counter()
    t_ref, rstats, _ = ref.run(fr, 0.0, case.steps)
    rdt = time.perf_counter() - r0
    m = g.mask()
    same = bool(np.array_equal(_host(f)[m], fr[m]))
    same_host = bool(np.array_equal(_host(fh)[m], fr[m]))
    return {"grid": f"{g.nr()}x{g.nz()}", "steps": case.steps, "t_end": t_end,
            "gpu": {"seconds": dt, "cell_updates": stats["cell_updates"],
                    "value": stats["cell_updates"] / dt, "unit": "cell-updates/s",
                    "radial_iters": stats["radial_iterations"],
                    "axial_iters": stats["axial_iterations"], "halvings": stats["halvings"],
                    "kernels": desc, "kernel_launches": launches,
                    "timing": "wall clock around pcgpu_run (resident stepper)"},
            "gpu_host_driven": {"seconds": hdt, "value": hstats["cell_updates"] / hdt,
                                "unit": "cell-updates/s", "kernels": hdesc,
                                "final_field_bitwise_vs_reference": same_host},
            "cpu_reference": {"seconds": rdt, "value": rstats["cell_updates"] / rdt,
                              "unit": "cell-updates/s", "cores": CORES, "kind": "reference",
                              "sample": sample},
            "parity": {"final_field_bitwise_vs_reference": same,
                       "iterations_equal": (rstats["radial_iterations"],
                                            rstats["axial_iterations"]) ==
                       (stats["radial_iterations"], stats["axial_iterations"])},
            "hbm_fraction": "not claimed (working set is cache-resident, SURVEY 8(d))"}


def cfg1(cpu_systems=16384):
    from tools.bench_tridiag import generate, run
    from oracle.oracle import ref_thomas_batch
    gpu = run(check=256)
    n = 1024
    bands = [v.ravel() for v in generate(cpu_systems, n)]  # std::mt19937_64(2024)
    ref_thomas_batch(*bands, n, cpu_systems, 0, workers=CORES)  # warm-up
    s0 = time.perf_counter()
    ref_thomas_batch(*bands, n, cpu_systems, 0, workers=CORES)
    dt = time.perf_counter() - s0
    return {"gpu": gpu,
            "cpu_reference": {"rows_per_s": cpu_systems * n / dt, "seconds": dt, "cores": CORES,
                              "kind": "reference",
                              "sample": f"{cpu_systems} x {n} contiguous systems, "
                                        "thomas_solve_inplace per system over a LinePool"}}


def _growth_case(case, check_steps, cpu_steps):
    from oracle.oracle import PortStepper
    g = case.grid()
    st = _gpu_stepper(case, g)
    # parity: the first check_steps steps of the growth controller, bit for bit
    fg = _dev_field(g, case.solver.T0)
    _, _, res_g = st.run_growth(fg, 0.0, case.t_end, check_steps, keep_results=True)
    port = PortStepper(case)
    fo = make_field(g, case.solver.T0)
    _, _, res_o = port.run_growth(fo, 0.0, case.t_end, check_steps)
    seq = lambda rs: [(r.tau_used, r.halvings, r.radial.iterations, r.axial.iterations)
                      for r in rs]
    m = g.mask()
    parity = {"steps_checked": check_steps,
              "sequence_equal": seq(res_g) == seq(res_o),
              "final_field_bitwise_vs_oracle": bool(np.array_equal(_host(fg)[m], fo[m]))}
    # the whole simulation on the GPU
    f = _dev_field(g, case.solver.T0)
    torch.cuda.synchronize()
    s0 = time.perf_counter()
    t_end, stats, _ = st.run_growth(f, 0.0, case.t_end, 10_000_000)
    torch.cuda.synchronize()
    dt = time.perf_counter() - s0
    cpu = _ref_rate(case, cpu_steps)
    return {"grid": f"{g.nr()}x{g.nz()}", "active_cells": int(m.sum()), "t_end": t_end,
            "gpu": {"seconds": dt, "steps": stats["steps"], "halvings": stats["halvings"],
                    "radial_iters": stats["radial_iterations"],
                    "axial_iters": stats["axial_iterations"],
                    "cell_updates": stats["cell_updates"],
                    "value": stats["cell_updates"] / dt, "unit": "cell-updates/s",
                    "timing": "wall clock around pcgpu_run_growth (whole simulation)"},
            "cpu_reference": cpu, "parity": parity}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg0,paper,cfg1,cfg2,cfg4")
    ap.add_argument("--periods-scale", type=float, default=1.0)
    a = ap.parse_args()
    out = {"device": torch.cuda.get_device_name(0), "host_cores": CORES}
    want = a.only.split(",")
    if "cfg0" in want:
        out["cfg0"] = cfg0()
    if "paper" in want:
        out["paper_cell"] = cfg0(configs.paper_cell(3000), "the whole 3000-step run")
    if "cfg1" in want:
        out["cfg1"] = cfg1()
    if "cfg2" in want:
        out["cfg2"] = _growth_case(configs.cfg2(5.0 * a.periods_scale), 8, 20)
    if "cfg4" in want:
        out["cfg4"] = _growth_case(configs.cfg4(10.0 * a.periods_scale), 4, 8)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
