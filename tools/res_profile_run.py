"""One resident-stepper batch on configs[0] (50 steps) -- the program the ncu
capture of k_resident runs (tools/r02_prof.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1912_03744_b200 import configs  # noqa: E402
from paper_1912_03744_b200.solver import AdiStepper, DevicePlan  # noqa: E402

c = configs.cfg0(50)
g = c.grid()
s = AdiStepper(g, c.materials, configs.make_source(c, g), c.timing, c.solver, DevicePlan(0))
f = torch.full((g.nz(), g.nr()), c.solver.T0, dtype=torch.float64, device="cuda").t()
s.run(f, 0.0, 50)
torch.cuda.synchronize()
assert s.resident_stats()["batches"] == 1
print("ok")
