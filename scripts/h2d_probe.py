"""Raw pinned H2D bandwidth for the cfg 2 batch size (240 MB): one copy, and the
same bytes split over S concurrent streams."""
import time

import torch

x = torch.empty(500_000 * 120, dtype=torch.float32, pin_memory=True)
d = torch.empty_like(x, device="cuda")
for _ in range(3):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    d.copy_(x, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"H2D 240 MB: {ms:.3f} ms = {x.numel() * 4 / ms / 1e6:.1f} GB/s")
for S in (2, 4):
    streams = [torch.cuda.Stream() for _ in range(S)]
    parts = x.numel() // S
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * parts:(i + 1) * parts].copy_(x[i * parts:(i + 1) * parts], non_blocking=True)
        torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 10 * 1e3
    print(f"H2D 240 MB over {S} streams: {ms:.3f} ms = {x.numel() * 4 / ms / 1e6:.1f} GB/s (wall)")
