"""A few host-driven configs[2] steps (the 8-producer line kernel, one CTA per
SM: chain-bound) -- the program ncu captures for the solver-warp stall view."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PCGPU_RESIDENT"] = "0"
import torch  # noqa: E402

from paper_1912_03744_b200 import configs  # noqa: E402
from paper_1912_03744_b200.solver import AdiStepper, DevicePlan  # noqa: E402

c = configs.CONFIGS["cfg2"]()
g = c.grid()
s = AdiStepper(g, c.materials, configs.make_source(c, g), c.timing, c.solver, DevicePlan(0))
f = torch.from_numpy(configs.smooth_field(g, 20.0).T.copy()).cuda().t()
t = 0.0
for _ in range(3):
    t += s.step(f, t).tau_used
torch.cuda.synchronize()
print("ok", s.describe())
