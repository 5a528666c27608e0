"""Wall-clock of whole runs on the resident stepper vs host-driven steps
(PCGPU_RESIDENT=1/0), per BASELINE config. Each measurement runs in a fresh
process so the env switch applies at stepper creation.

  python tools/res_timing.py [--configs cfg0,cfg2,cfg4] [--out gpurun_out/res_timing.json]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RUNS = {
    # name: (builder expression, kind, steps or (t_end, max_steps))
    "cfg0": "run", "cfg2": "growth", "cfg4": "growth", "paper": "run",
}


def one(name: str, steps: int) -> dict:
    import torch
    from paper_1912_03744_b200 import configs
    from paper_1912_03744_b200.solver import AdiStepper, DevicePlan, GrowthPolicy
    case = {"cfg0": lambda: configs.cfg0(2000), "cfg2": configs.cfg2, "cfg4": configs.cfg4,
            "paper": getattr(configs, "paper_cell", configs.cfg0)}[name]()
    g = case.grid()
    st = AdiStepper(g, case.materials, configs.make_source(case, g), case.timing, case.solver,
                    DevicePlan(device=0))
    f = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64, device="cuda").t()
    kind = RUNS[name]
    # warm-up (allocations, first launch)
    if kind == "run":
        st.run(f, 0.0, 2)
    else:
        st.run_growth(f, 0.0, 1.0, 2, GrowthPolicy())
    f.fill_(case.solver.T0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if kind == "run":
        t_end, stats, _ = st.run(f, 0.0, steps)
    else:
        t_end, stats, _ = st.run_growth(f, 0.0, case.t_end, steps, GrowthPolicy())
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    res = st.resident_stats()
    launches = st.launch_count()
    del st  # prints the phase profile with PCGPU_RES_PROF=1
    import gc
    gc.collect()
    return {"config": name, "grid": f"{g.nr()}x{g.nz()}", "steps": stats["steps"],
            "seconds": sec, "us_per_step": 1e6 * sec / max(1, stats["steps"]),
            "cell_updates_per_s": stats["cell_updates"] / sec,
            "radial_iters": stats["radial_iterations"], "axial_iters": stats["axial_iterations"],
            "halvings": stats["halvings"], "t_end": t_end, "resident": res,
            "launches": launches}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg0,cfg2,cfg4")
    ap.add_argument("--steps", default="cfg0:2000,cfg2:1000,cfg4:300,paper:200")
    ap.add_argument("--out", default=None)
    ap.add_argument("--child", default=None)
    a = ap.parse_args()
    steps = dict((k, int(v)) for k, v in (kv.split(":") for kv in a.steps.split(",")))
    if a.child:
        print(json.dumps(one(a.child, steps[a.child])))
        return
    rows = []
    for name in a.configs.split(","):
        for path in ("1", "0"):
            env = dict(os.environ, PCGPU_RESIDENT=path)
            r = subprocess.run([sys.executable, __file__, "--child", name, "--steps", a.steps],
                               env=env, capture_output=True, text=True, cwd=ROOT)
            line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
            row = json.loads(line[-1]) if line else {"config": name, "error": r.stderr[-800:]}
            row["path"] = "resident" if path == "1" else "host"
            prof = [ln for ln in r.stderr.splitlines() if "resident profile" in ln]
            if prof:
                row["profile"] = prof[-1]
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
