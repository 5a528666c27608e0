"""Host<->device copy bandwidth of this box (pinned and pageable), 1 GiB."""
import time

import torch

n = 1 << 27  # 1 GiB of float64
dev = torch.empty(n, dtype=torch.float64, device="cuda")
for pinned in (True, False):
    h = torch.empty(n, dtype=torch.float64, pin_memory=pinned)
    h.fill_(1.0)
    for name, fn in (("H2D", lambda: dev.copy_(h, non_blocking=True)),
                     ("D2H", lambda: h.copy_(dev, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{'pinned' if pinned else 'pageable'} {name}: {n * 8 / ms / 1e6:.1f} GB/s")
