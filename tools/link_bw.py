"""Pinned / pageable host<->device copy bandwidth of this box (torch copies, 1 GiB)."""
import time
import torch
n = 1 << 27
for pin in (True, False):
    h = torch.empty(n, dtype=torch.float64, pin_memory=pin)
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for direction in ("h2d", "d2h"):
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if direction == "h2d":
                d.copy_(h, non_blocking=pin)
            else:
                h.copy_(d, non_blocking=pin)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"pinned={pin} {direction}: {n * 8 / dt / 1e9:.1f} GB/s")
