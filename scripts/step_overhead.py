"""Host overhead per build_detect step (dev tool): device time with and
without per-phase timing events, and the host wall time of the calls."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = W.CONFIGS[cfg]
n = w.n
x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
W.device_rows(cfg, 0, n, x.data_ptr())
fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
sk = ace.AceSketch(fam, ace.CounterWidth.k32)
stream = torch.cuda.current_stream()
sk.set_stream(stream.cuda_stream)
flags = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
for timing in (1, 0, 1, 0):
    N.dev().ace_sketch_set_timing(sk.handle, timing)
    for _ in range(3):
        sk.reset(); sk.build_detect(x, flags_out=flags)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 50
    host = 0.0
    e0.record(stream)
    for _ in range(steps):
        t0 = time.perf_counter()
        sk.reset()
        t1 = time.perf_counter()
        sk.build_detect(x, flags_out=flags)
        host += t1 - t0
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"timing={timing} device ms/step {e0.elapsed_time(e1) / steps:.4f}  reset call {host / steps * 1e6:.1f} us")
# python wrapper cost without GPU work: a zero-row-ish call is rejected, so time the ctypes layer alone
t0 = time.perf_counter()
for _ in range(1000):
    N.dev().ace_kernel_launches()
print(f"ctypes call overhead {(time.perf_counter() - t0) * 1e3:.1f} us per call x1000 -> {(time.perf_counter() - t0):.4f} ms/call")
