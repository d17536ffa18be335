"""Raw pinned H2D bandwidth for the cfg 2 batch size (240 MB)."""
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
