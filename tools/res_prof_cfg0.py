"""configs[0] (2000 steps) on the resident stepper with $PCGPU_RES_PROF=1: the
per-phase device times and the solver warp's cycle split, printed to stderr
when the stepper is destroyed; plus the wall clock of the run."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1912_03744_b200 import configs  # noqa: E402
from paper_1912_03744_b200.solver import AdiStepper, DevicePlan  # noqa: E402

c = configs.cfg0(2000)
g = c.grid()
s = AdiStepper(g, c.materials, configs.make_source(c, g), c.timing, c.solver, DevicePlan(0))
f = torch.full((g.nz(), g.nr()), c.solver.T0, dtype=torch.float64, device="cuda").t()
s.run(f, 0.0, 2)
torch.cuda.synchronize()
f.fill_(c.solver.T0)
t0 = time.perf_counter()
s.run(f, 0.0, 2000)
torch.cuda.synchronize()
print(f"cfg0 2000 steps: {time.perf_counter() - t0:.4f} s", s.resident_stats(), flush=True)
del s
