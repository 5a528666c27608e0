"""Diagnostic: fast vs exact half-steps on a configuration; prints where the
largest differences are (profiling/debug helper, not part of the product)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1912_03744_b200 import configs  # noqa: E402
from paper_1912_03744_b200.solver import AdiStepper, DevicePlan  # noqa: E402


def stepper(case, mode):
    g = case.grid()
    return AdiStepper(g, case.materials, configs.make_source(case, g), case.timing, case.solver,
                      DevicePlan(0, mode))


def dev_field(g, val):
    return torch.full((g.nz(), g.nr()), val, dtype=torch.float64, device="cuda").t()


def report(name, a, b, g):
    m = torch.from_numpy(g.mask()).cuda()
    d = ((a - b).abs() * m)
    v, idx = d.flatten().max(0)
    # flatten of the (nr, nz) view with strides (1, nr) follows logical (i, j) order
    i, j = divmod(int(idx), g.nz())
    rows = d.max(dim=1).values.cpu().numpy()
    cols = d.max(dim=0).values.cpu().numpy()
    top_i = np.argsort(-rows)[:8]
    top_j = np.argsort(-cols)[:8]
    print(f"{name}: max |diff| {float(v):.3e} at (i={i}, j={j}); T there {float(b[i, j]):.6f}; "
          f"top rows i {top_i.tolist()} top cols j {top_j.tolist()}")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    case = configs.CONFIGS[name]() if name in configs.CONFIGS else configs.cfg3()
    g = case.grid()
    ex, fa = stepper(case, "exact"), stepper(case, "fast")
    f0 = dev_field(g, case.solver.T0)
    # one step of exact to get a nontrivial field
    ex.run(f0, 0.0, 1)
    tau = ex.initial_tau(1e-5)
    h_e, h_f = dev_field(g, 0.0), dev_field(g, 0.0)
    r1 = ex.radial_half_step(f0, 1e-5, tau, h_e)
    r2 = fa.radial_half_step(f0, 1e-5, tau, h_f)
    print("radial outcomes", r1, r2)
    report("radial half-step", h_f, h_e, g)
    n_e, n_f = dev_field(g, 0.0), dev_field(g, 0.0)
    a1 = ex.axial_half_step(h_e, 1e-5, tau, n_e)
    a2 = fa.axial_half_step(h_e, 1e-5, tau, n_f)
    print("axial outcomes", a1, a2)
    report("axial half-step (same input)", n_f, n_e, g)
    incr = ((h_e - f0).abs() * torch.from_numpy(g.mask()).cuda()).max()
    print(f"max |radial increment| {float(incr):.3e}")


if __name__ == "__main__" and not os.environ.get("DIAG_RUNS"):
    main()


def runs(name="cfg3", steps=(1, 2)):
    case = configs.CONFIGS[name]()
    g = case.grid()
    for n in steps:
        out = {}
        for mode in ("exact", "fast"):
            st = stepper(case, mode)
            f = dev_field(g, case.solver.T0)
            _, stats, res = st.run(f, 0.0, n, keep_results=True)
            out[mode] = (f, [(r.radial.iterations, r.axial.iterations, r.radial.last_delta, r.axial.last_delta) for r in res])
            del st
        print(n, "steps:", out["exact"][1], out["fast"][1])
        report(f"run {n} steps", out["fast"][0], out["exact"][0], g)
        # half-steps from T0 at t=0
    st_e, st_f = stepper(case, "exact"), stepper(case, "fast")
    f0 = dev_field(g, case.solver.T0)
    tau = st_e.initial_tau(0.0)
    h_e, h_f = dev_field(g, 0.0), dev_field(g, 0.0)
    print(st_e.radial_half_step(f0, 0.0, tau, h_e), st_f.radial_half_step(f0, 0.0, tau, h_f))
    report("radial from T0", h_f, h_e, g)
    n_e, n_f = dev_field(g, 0.0), dev_field(g, 0.0)
    print(st_e.axial_half_step(h_e, 0.0, tau, n_e), st_f.axial_half_step(h_e, 0.0, tau, n_f))
    report("axial from exact half", n_f, n_e, g)
    # fast step() API vs exact step()
    fe, ff = dev_field(g, case.solver.T0), dev_field(g, case.solver.T0)
    print(st_e.step(fe, 0.0), st_f.step(ff, 0.0))
    report("step() API", ff, fe, g)
    report("step() vs manual half-steps (exact)", fe, n_e, g)


if __name__ == "__main__" and os.environ.get("DIAG_RUNS"):
    runs(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
