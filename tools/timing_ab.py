import os, sys
sys.path.insert(0, os.getcwd())
import torch
from bench import gpu_stepper_for
from paper_1912_03744_b200 import configs
case = configs.CONFIGS["cfg3"]()
g = case.grid()
s = gpu_stepper_for(case, 0)
f = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64, device="cuda").t()
t, _, _ = s.run(f, 0.0, 3)
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(s.stream(), device="cuda:0")
for timing in (True, False, True, False):
    s.enable_kernel_timing(timing)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    t, stats, _ = s.run(f, t, 20)
    e1.record(st)
    torch.cuda.synchronize()
    print("timing", timing, round(e0.elapsed_time(e1) / 20, 3), "ms/step", stats["radial_iterations"], stats["axial_iterations"])
    s.enable_kernel_timing(False)
