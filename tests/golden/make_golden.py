"""Regenerate the golden fixtures from the REFERENCE ITSELF.

Runs the reference's own AdiStepper / thomas_solve_inplace, compiled unchanged
from /root/reference/proj/src into oracle/_ref/libpcref.so (oracle/Makefile),
on the cases below and stores inputs + outputs under tests/golden/*.npz.
Run in the build container (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import RefStepper, ref_thomas_batch  # noqa: E402
from paper_1912_03744_b200 import configs  # noqa: E402
from paper_1912_03744_b200.solver import make_field  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

def _coarse_cfg0():
    c = configs.scaled(configs.cfg0(), [23, 3, 7, 2], 48)
    c.solver.tau_source_divisor = 10.0  # tau = 0.01 outside the transient windows
    c.solver.max_iter = 6
    return c


# (name, case builder, initial field, steps, t0)
CASES = [
    ("stepcell_nonlinear", lambda: configs.step_cell(True), "smooth", 25, 0.0),
    ("stepcell_linear", lambda: configs.step_cell(False), "smooth", 25, 0.0),
    ("stepcell_maxiter1", lambda: configs.step_cell(True, max_iter=1), "smooth20", 3, 0.001),
    ("stepcell_bigtau", lambda: configs.step_cell(True, tau_transient_divisor=1.0,
                                                  tau_source_divisor=1.0, max_iter=8),
     "smooth20", 20, 0.05),
    ("paper_small_transient", configs.paper_like_small, "T0", 40, 0.0),
    ("cfg0_200steps", lambda: configs.cfg0(200), "T0", 200, 0.0),
    ("cfg0_coarse_halving", _coarse_cfg0, "T0", 40, 0.02),
    ("cfg4_small", lambda: configs.scaled(configs.cfg4(), [44, 5, 13, 3], 128, 87), "T0", 60,
     0.0),
]


def initial(case, kind):
    g = case.grid()
    if kind == "smooth":
        return configs.smooth_field(g)
    if kind == "smooth20":
        return configs.smooth_field(g, 20.0)
    return make_field(g, case.solver.T0)


def main():
    for name, build, init, steps, t0 in CASES:
        case = build()
        ref = RefStepper(case)
        f = initial(case, init)
        f0 = f.copy(order="F")
        t_end, stats, res = ref.run(f, t0, steps)
        seq = np.array([[r.tau_used, r.halvings, r.radial.iterations, r.axial.iterations,
                         r.radial.last_delta, r.axial.last_delta] for r in res])
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), initial=f0, final=f,
                            seq=seq, t0=t0, t_end=t_end, steps=steps,
                            clamp=np.array(ref.clamp_events(), dtype=np.uint64))
        print(name, case.grid().nr(), case.grid().nz(), steps, "t_end", t_end)
    # Tridiagonal known answers: random strictly dominant systems (the shape of
    # the acceptance suite's thomas_oracle, acceptance_main.cpp:107-120) solved
    # by the reference thomas_solve_inplace, both layouts.
    rng = np.random.default_rng(2024)
    n, batch = 64, 96
    lo = rng.uniform(-1.0, 0.0, (batch, n)); lo[:, 0] = 0.0
    up = rng.uniform(-1.0, 0.0, (batch, n)); up[:, -1] = 0.0
    dg = 2.05 + np.abs(lo) + np.abs(up)
    rhs = rng.uniform(-1.0, 1.0, (batch, n))
    flat = [np.ascontiguousarray(v.reshape(-1)) for v in (lo, dg, up, rhs)]
    rc, x, _ = ref_thomas_batch(*flat, n, batch, 0)
    assert rc == 0
    np.savez_compressed(os.path.join(HERE, "thomas_batch.npz"), lower=lo, diag=dg, upper=up,
                        rhs=rhs, x=x.reshape(batch, n))
    print("thomas_batch", n, batch)


if __name__ == "__main__":
    main()
