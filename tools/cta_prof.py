"""Per-CTA placement and phases of the last radial ws launch on configs[3] (A/B build
`make -C paper_1912_03744_b200/csrc VARIANT=tsprof EXTRA=-DPCGPU_TSPROF`, PCGPU_LIB):
SM id, entry, forward end, end (%globaltimer), grouped by the SM's CTA count."""
import collections
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import gpu_stepper_for  # noqa: E402
from paper_1912_03744_b200 import _native, configs  # noqa: E402

case = configs.CONFIGS["cfg3"]()
g = case.grid()
s = gpu_stepper_for(case, 0)
f = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64, device="cuda").t()
t, _, _ = s.run(f, 0.0, 3)
s.run(f, t, 1)
torch.cuda.synchronize()
lib = C.CDLL(_native.LIB_PATH)
buf = np.zeros((1024, 4), dtype=np.uint64)
assert lib.pcgpu_debug_ctaprof(buf.ctypes.data_as(C.c_void_p), 1024) == 0
b = buf[buf[:, 1] > 0]
t0 = b[:, 1].min()
per_sm = collections.defaultdict(list)
for r in b:
    per_sm[int(r[0])].append([(float(x) - t0) / 1e3 for x in r[1:]])
print("CTAs:", len(b), "SMs:", len(per_sm))
for k in sorted({len(v) for v in per_sm.values()}):
    rows = np.array([x for v in per_sm.values() if len(v) == k for x in v])
    print(f"SMs with {k} line blocks: {sum(1 for v in per_sm.values() if len(v) == k)}; "
          f"forward end {rows[:, 1].mean():.0f} us (max {rows[:, 1].max():.0f}), "
          f"end {rows[:, 2].mean():.0f} us (max {rows[:, 2].max():.0f})")
