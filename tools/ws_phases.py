"""Phase timeline of the host-driven ws line launches on configs[3] (needs the
A/B build `make -C paper_1912_03744_b200/csrc VARIANT=tsprof EXTRA=-DPCGPU_TSPROF`,
selected with PCGPU_LIB). Per CTA: entry, end of the forward elimination, end,
from %globaltimer; prints the spread of the starts, the forward and backward
durations, and the launch span for the last radial and axial launch of a step."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import gpu_stepper_for  # noqa: E402
from paper_1912_03744_b200 import _native, configs  # noqa: E402


def main():
    case = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]()
    g = case.grid()
    s = gpu_stepper_for(case, 0)
    f = torch.full((g.nz(), g.nr()), case.solver.T0, dtype=torch.float64, device="cuda").t()
    t, _, _ = s.run(f, 0.0, 3)
    s.run(f, t, 1)
    torch.cuda.synchronize()
    lib = C.CDLL(_native.LIB_PATH)
    for axial, name in ((0, "radial"), (1, "axial")):
        nblk = (g.nz() if axial == 0 else g.nr()) // 32
        buf = np.zeros((nblk, 3), dtype=np.uint64)
        assert lib.pcgpu_debug_tsprof(axial, buf.ctypes.data_as(C.c_void_p), nblk) == 0
        b = buf.astype(np.float64)
        t0 = b[:, 0].min()
        st, fe, en = (b[:, 0] - t0) / 1e3, (b[:, 1] - t0) / 1e3, (b[:, 2] - t0) / 1e3
        fwd, back = fe - st, en - fe

        def q(x):
            return " ".join(f"{v:7.1f}" for v in np.percentile(x, [0, 10, 50, 90, 100]))
        print(f"{name}: {nblk} CTAs, span {en.max():.1f} us (percentiles 0/10/50/90/100)")
        print(f"  start     {q(st)}")
        print(f"  fwd dur   {q(fwd)}")
        print(f"  fwd end   {q(fe)}")
        print(f"  back dur  {q(back)}")
        print(f"  end       {q(en)}")


if __name__ == "__main__":
    main()
