"""Dense TF32 tensor-core throughput on this GPU (torch.matmul fp32 with TF32
enabled, 8192^3, best of 10, CUDA events): the tcgen05 peak of the fp32 input
dtype, written beside MEASURED_PEAKS.json's bf16 figure."""
import json
import sys

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a @ b
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
tf = 2.0 * n ** 3 / (best * 1e-3) / 1e12
out = {"tf32_tflops": round(tf, 1), "how": "torch.matmul fp32 (allow_tf32) 8192^3, best of 10, CUDA events",
       "gpu": torch.cuda.get_device_name()}
print(json.dumps(out))
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(json.dumps(out) + "\n")
