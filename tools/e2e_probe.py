"""Where the time of a host-field step goes on configs[3] (pcgpu_step_host):
the bare pinned copies of one field each way, device-resident steps, and
host-field steps (wall clock per call; each call synchronizes)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import gpu_stepper_for  # noqa: E402
from paper_1912_03744_b200 import configs  # noqa: E402


def main():
    case = configs.CONFIGS["cfg3"]()
    g = case.grid()
    nr, nz = g.nr(), g.nz()
    s = gpu_stepper_for(case, 0)
    f = torch.full((nz, nr), case.solver.T0, dtype=torch.float64, device="cuda").t()
    t, _, _ = s.run(f, 0.0, 3)
    torch.cuda.synchronize()
    pinned = torch.empty((nz, nr), dtype=torch.float64).pin_memory()
    pinned.copy_(f.t())
    dev = torch.empty_like(f.t())
    for name, fn in (("H2D 1 GiB", lambda: dev.copy_(pinned, non_blocking=True)),
                     ("D2H 1 GiB", lambda: pinned.copy_(dev, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        print(f"{name}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms", flush=True)
    for _ in range(2):
        t0 = time.perf_counter()
        t, _, _ = s.run(f, t, 1)
        torch.cuda.synchronize()
        print(f"device step: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
    hp = pinned.numpy().T
    for _ in range(4):
        t0 = time.perf_counter()
        r = s.step(hp, t)
        t += r.tau_used
        print(f"host step ({r.radial.iterations}+{r.axial.iterations} it): "
              f"{(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
    print("pipeline", s.pipeline_stats(), os.environ.get("PCGPU_NO_PIPELINE"))


if __name__ == "__main__":
    main()
