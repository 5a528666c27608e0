"""Per-CTA timeline (tile0: the solver starts the pivot chain) of the resident stepper's last radial and axial Picard
phase on configs[0] (A/B build with -DPCGPU_TSPROF selected by PCGPU_LIB, run
with PCGPU_RES_PROF=1): phase start -> line entry -> forward end -> bulk copy
end -> back substitution end -> line end -> phase barrier, in microseconds."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1912_03744_b200 import _native, configs  # noqa: E402
from paper_1912_03744_b200.solver import AdiStepper, DevicePlan  # noqa: E402

c = configs.CONFIGS[sys.argv[1]]() if len(sys.argv) > 1 else configs.cfg0(50)
g = c.grid()
s = AdiStepper(g, c.materials, configs.make_source(c, g), c.timing, c.solver, DevicePlan(0))
f = torch.full((g.nz(), g.nr()), c.solver.T0, dtype=torch.float64, device="cuda").t()
s.run(f, 0.0, 20)
torch.cuda.synchronize()
lib = C.CDLL(_native.LIB_PATH)
names = ["start", "entry", "fwd", "bulk", "back", "line", "barrier", "tile0"]
for axial in (0, 1):
    buf = np.zeros((64, 8), dtype=np.uint64)
    assert lib.pcgpu_debug_rts(axial, buf.ctypes.data_as(C.c_void_p)) == 0
    rows = [r for r in range(64) if buf[r, 0] and buf[r, 6]]
    t0 = min(int(buf[r, 0]) for r in rows)
    print("axial" if axial else "radial", "(us from the earliest phase start)")
    print("  cta " + " ".join(f"{n:>8}" for n in names))
    for r in rows:
        vals = [(int(buf[r, k]) - t0) / 1e3 if buf[r, k] else float("nan") for k in range(8)]
        print(f"  {r:3d} " + " ".join(f"{v:8.2f}" for v in vals))
