"""TEST INFRASTRUCTURE (a report, not a test): whole-run adaptive-dt parity at
BASELINE size (north star: identical accepted-dt and Picard-iteration-count
sequence, final field within 1e-6 relative -- exact mode is bitwise).

The BASELINE growth policy (start 1e-5 s, halve on non-convergence, x1.2 after
5 easy steps, cap 1e-3 s) runs on the B200 (pcgpu_run_growth) and through the
reference's OWN half-steps under the same controller (pcref_run_growth:
AdiStepper::radial_half_step / axial_half_step, solver.hpp:70-78, the way
acceptance_main.cpp:311-332 drives them), on all host cores.

  # both legs in one process (cfg2: 5 periods, ~4 min of CPU on 16 cores)
  python tests/reports/adaptive_full_parity.py --config cfg2 --out profiles/r02_adaptive_full_parity.json
  # split legs (the GPU leg on the B200, the CPU leg elsewhere), then compare
  python tests/reports/adaptive_full_parity.py --config cfg4 --t-end 1.0 --leg gpu --save g.npz
  python tests/reports/adaptive_full_parity.py --config cfg4 --t-end 1.0 --leg ref --save r.npz
  python tests/reports/adaptive_full_parity.py --compare g.npz r.npz --out ...
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1912_03744_b200 import configs  # noqa: E402
from paper_1912_03744_b200.solver import GrowthPolicy, make_field  # noqa: E402


def seq(results):
    return np.array([[r.tau_used, r.halvings, r.radial.iterations, r.axial.iterations,
                      r.radial.last_delta, r.axial.last_delta] for r in results])


def build(name):
    return {"cfg2": configs.cfg2, "cfg4": configs.cfg4}[name]()


def leg(name, which, t_end, max_steps):
    case = build(name)
    g = case.grid()
    t_end = case.t_end if t_end is None else t_end
    pol = GrowthPolicy()
    t0 = time.perf_counter()
    if which == "gpu":
        import torch
        from paper_1912_03744_b200.solver import AdiStepper, DevicePlan
        st = AdiStepper(g, case.materials, configs.make_source(case, g), case.timing,
                        case.solver, DevicePlan(0))
        f = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64,
                       device="cuda").t()
        te, stats, res = st.run_growth(f, 0.0, t_end, max_steps, pol, keep_results=True)
        torch.cuda.synchronize()
        field = np.asfortranarray(f.t().contiguous().cpu().numpy().T)
        extra = {"resident": st.resident_stats()}
        cores = None
    else:
        from oracle.oracle import RefStepper
        cores = os.cpu_count() or 1
        st = RefStepper(case, workers=cores)
        field = make_field(g, case.solver.T0)
        te, stats, res = st.run_growth(field, 0.0, t_end, max_steps, pol)
        extra = {}
    sec = time.perf_counter() - t0
    m = g.mask()
    return {"config": name, "leg": which, "t_end_requested": t_end, "t_end": te,
            "steps": int(stats["steps"]), "halvings": int(stats["halvings"]),
            "cell_updates": float(stats["cell_updates"]), "seconds": sec, "cores": cores,
            "seq": seq(res), "field": field,
            "sha256_masked": hashlib.sha256(np.ascontiguousarray(field[m]).tobytes()).hexdigest(),
            **extra}


def compare(a, b, mask):
    sa, sb = a["seq"], b["seq"]
    n = min(len(sa), len(sb))
    first_diff = next((k for k in range(n) if not np.array_equal(sa[k], sb[k])), None)
    fa, fb = a["field"][mask], b["field"][mask]
    rel = float(np.max(np.abs(fa - fb)) / np.max(np.abs(fb)))
    return {
        "steps": len(sb), "steps_checked": n if first_diff is None else first_diff,
        "sequence_equal": bool(len(sa) == len(sb) and first_diff is None),
        "dt_iterations_equal": bool(len(sa) == len(sb) and np.array_equal(sa[:, :4], sb[:, :4])),
        "first_differing_step": first_diff,
        "t_end_equal": bool(a["t_end"] == b["t_end"]),
        "final_field_bitwise": bool(np.array_equal(fa, fb)),
        "final_field_rel_linf": rel, "north_star_tolerance": 1e-6,
        "cells_differing": int(np.count_nonzero(fa != fb)),
    }


def summary(r):
    return {k: v for k, v in r.items() if k not in ("seq", "field")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--t-end", type=float, default=None)
    ap.add_argument("--max-steps", type=int, default=2_000_000)
    ap.add_argument("--leg", choices=["both", "gpu", "ref"], default="both")
    ap.add_argument("--save", default=None)
    ap.add_argument("--compare", nargs=2, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    if a.compare:
        ga, ra = (dict(np.load(p, allow_pickle=True)) for p in a.compare)
        ga = {k: (v.item() if v.shape == () else v) for k, v in ga.items()}
        ra = {k: (v.item() if v.shape == () else v) for k, v in ra.items()}
        mask = build(str(ga["config"])).grid().mask()
        out = {"gpu": summary(ga), "reference": summary(ra), **compare(ga, ra, mask)}
    else:
        legs = ["gpu", "ref"] if a.leg == "both" else [a.leg]
        rs = {w: leg(a.config, w, a.t_end, a.max_steps) for w in legs}
        if a.save:
            r = rs[legs[0]]
            np.savez_compressed(a.save, **{k: (np.asarray(v) if not isinstance(v, dict)
                                               else np.asarray(json.dumps(v)))
                                           for k, v in r.items()})
        if a.leg != "both":
            print(json.dumps(summary(rs[legs[0]]), default=str))
            return
        mask = build(a.config).grid().mask()
        out = {"gpu": summary(rs["gpu"]), "reference": summary(rs["ref"]),
               **compare(rs["gpu"], rs["ref"], mask)}
    out["what"] = ("BASELINE growth policy, B200 (pcgpu_run_growth) vs the reference's own "
                   "half-steps under the same controller (pcref_run_growth)")
    s = json.dumps(out, indent=1, default=str)
    print(s)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
