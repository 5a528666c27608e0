"""Run a few ADI steps of a named configuration on cuda:0 (profiling driver).

    python tools/run_case.py --config cfg3 --mode fast --steps 1
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1912_03744_b200 import configs  # noqa: E402
from paper_1912_03744_b200.solver import AdiStepper, DevicePlan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=0)
    ap.add_argument("--dist", type=int, default=0,
                    help="run the partitioned stepper with this many emulated ranks")
    a = ap.parse_args()
    extra = {"stepcell": configs.step_cell, "paper_small": configs.paper_like_small,
             "cfg4_small": lambda: configs.scaled(configs.cfg4(), [44, 5, 13, 3], 128, 87)}
    case = (configs.CONFIGS.get(a.config) or extra[a.config])()
    g = case.grid()
    if a.dist:
        return run_dist(a, case, g)
    st = AdiStepper(g, case.materials, configs.make_source(case, g), case.timing, case.solver,
                    DevicePlan(0, a.mode))
    f = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64, device="cuda").t()
    t = 0.0
    if a.warmup:
        t, _, _ = st.run(f, t, a.warmup)
    torch.cuda.synchronize()
    st.enable_kernel_timing(True)
    t0 = time.perf_counter()
    t, stats, res = st.run(f, t, a.steps, keep_results=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{a.config} {a.mode}: {a.steps} steps in {dt*1e3:.1f} ms, "
          f"{stats['cell_updates']/dt:.3e} cell-updates/s, iters r/a "
          f"{stats['radial_iterations']}/{stats['axial_iterations']}, halvings {stats['halvings']}")
    kt = st.kernel_timing()
    print(f"  line kernels: radial {kt['radial_ms']:.2f} ms / {kt['radial_launches']} launches, "
          f"axial {kt['axial_ms']:.2f} ms / {kt['axial_launches']} launches; launches total "
          f"{st.launch_count()}")


def run_dist(a, case, g):
    from paper_1912_03744_b200.dist import PartitionedAdi
    part = PartitionedAdi(g, case.materials, configs.make_source(case, g), case.timing,
                          case.solver, device=0, emulate=a.dist, mode=a.mode)
    f = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64, device="cuda").t()
    part.set_field(f)
    t = 0.0
    if a.warmup:
        t, _, _ = part.run(t, a.warmup)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t, stats, _ = part.run(t, a.steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{a.config} {a.mode} dist x{a.dist} ({part.transport()}): {a.steps} steps in "
          f"{dt*1e3:.1f} ms, {stats['cell_updates']/dt:.3e} cell-updates/s, iters r/a "
          f"{stats['radial_iterations']}/{stats['axial_iterations']}")


if __name__ == "__main__":
    main()
