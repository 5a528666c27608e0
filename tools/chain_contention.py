"""Timing experiment (results are wrong; A/B build with -DPCGPU_TSPROF): how
fast the line solver's pivot chain runs with the producer warps beside it
doing all, part or none of their work (pcgpu_debug_set_exp modes), on the
host-driven radial and axial sweeps of a grid (default configs[0]) -- ms per
Picard-iteration launch from the stepper's kernel timing."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PCGPU_RESIDENT"] = "0"
import torch  # noqa: E402

from paper_1912_03744_b200 import _native, configs  # noqa: E402
from paper_1912_03744_b200.solver import AdiStepper, DevicePlan, make_field  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg0"
c = configs.CONFIGS[name]()
c.solver.max_iter = 20
g = c.grid()
s = AdiStepper(g, c.materials, configs.make_source(c, g), c.timing, c.solver, DevicePlan(0))
lib = C.CDLL(_native.LIB_PATH)
f = configs.smooth_field(g, 20.0)
out = make_field(g, 0.0)
fd = torch.from_numpy(f.T.copy()).cuda().t()
od = torch.from_numpy(out.T.copy()).cuda().t()
for mode in (0, 1, 2, 3, 0):
    assert lib.pcgpu_debug_set_exp(mode) == 0
    s.radial_half_step(fd, 0.0, 1e-4, od)  # warm
    s.enable_kernel_timing(True)
    for _ in range(5):
        s.radial_half_step(fd, 0.0, 1e-4, od)
        s.axial_half_step(fd, 0.0, 1e-4, od)
    torch.cuda.synchronize()
    kt = s.kernel_timing()
    s.enable_kernel_timing(False)
    for ax in (0, 1):
        nb = 64
        import numpy as np
        w = np.zeros((nb, 2), dtype=np.uint64)
        if lib.pcgpu_debug_fwait(ax, w.ctypes.data_as(C.c_void_p), nb) == 0:
            m = w[:, 0] > 0
            if m.any():
                print(f"   {'axial' if ax else 'radial'} forward: work {w[m, 0].mean() / 1e3:.1f} us, "
                      f"barrier waits {w[m, 1].mean() / 1e3:.1f} us (mean over CTAs)")
    print(f"{name} mode {mode}: radial {kt['radial_ms'] / max(kt['radial_launches'], 1) * 1e3:.1f} us "
          f"x {kt['radial_launches']}, axial {kt['axial_ms'] / max(kt['axial_launches'], 1) * 1e3:.1f} us "
          f"x {kt['axial_launches']}", flush=True)
