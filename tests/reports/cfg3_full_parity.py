"""TEST INFRASTRUCTURE (a report, not a test): configs[3] in full -- 8192 x 16384, tau = 1e-5, 200 steps -- on the B200 in
exact mode and through the reference's own AdiStepper (oracle/_ref, all host
cores), compared bit for bit: final field, and per step tau, halvings, Picard
iteration counts and last_delta. Prints one JSON object (committed as
profiles/r01_cfg3_full_parity.json). The CPU leg takes ~15-25 min on 16 cores.

    python tests/reports/cfg3_full_parity.py [--steps 200]
"""
import argparse
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1912_03744_b200 import configs  # noqa: E402
from paper_1912_03744_b200.solver import AdiStepper, DevicePlan, make_field  # noqa: E402


def seq(results):
    return [(r.tau_used, r.halvings, r.radial.iterations, r.axial.iterations,
             r.radial.last_delta, r.axial.last_delta) for r in results]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    from oracle.oracle import RefStepper, ref_available
    case = configs.cfg3(a.steps)
    g = case.grid()
    m = g.mask()
    gpu = AdiStepper(g, case.materials, configs.make_source(case, g), case.timing, case.solver,
                     DevicePlan(0, "exact"))
    f = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64, device="cuda").t()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    te_g, st_g, res_g = gpu.run(f, 0.0, a.steps, keep_results=True)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    fg = np.asfortranarray(f.t().contiguous().cpu().numpy().T)
    del gpu, f
    torch.cuda.empty_cache()

    cores = os.cpu_count() or 1
    kind = "reference" if ref_available() else "port"
    if kind == "reference":
        cpu = RefStepper(case, workers=cores)
    else:
        from oracle.oracle import PortStepper
        cpu, cores = PortStepper(case), 1
    fo = make_field(g, case.solver.T0)
    t0 = time.perf_counter()
    te_o, st_o, res_o = cpu.run(fo, 0.0, a.steps)
    cpu_s = time.perf_counter() - t0

    diff = fg[m] != fo[m]
    out = {
        "config": f"configs[3]: {g.nr()} x {g.nz()}, tau 1e-5, {a.steps} steps, exact mode",
        "bitwise_field": bool(not diff.any()),
        "cells_differing": int(diff.sum()),
        "sequence_equal": seq(res_g) == seq(res_o),
        "t_end_equal": te_g == te_o,
        "field_sha256": hashlib.sha256(np.ascontiguousarray(fg).tobytes()).hexdigest(),
        "field_min_max": [float(fg[m].min()), float(fg[m].max())],
        "iterations": {"radial": st_g["radial_iterations"], "axial": st_g["axial_iterations"],
                       "halvings": st_g["halvings"]},
        "gpu": {"seconds": gpu_s, "cell_updates_per_s": st_g["cell_updates"] / gpu_s,
                "timing": "wall clock around pcgpu_run"},
        "cpu": {"seconds": cpu_s, "cell_updates_per_s": st_o["cell_updates"] / cpu_s,
                "cores": cores, "kind": kind},
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
