"""Stream throughput and per-batch latency vs hashing group size (cfg 5, 16M rows)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

w = W.CONFIGS[5]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16 * 1024 * 1024
x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
W.device_rows(5, 0, n, x.data_ptr())
fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
flags = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
for g in (1, 2, 4, 8):
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.set_option(N.ACE_OPT_STREAM_GROUP, g)
    sk.set_stream(torch.cuda.current_stream().cuda_stream)
    for _ in range(2):
        sk.reset()
        sk.stream_run(x, w.batch, w.alpha, flags_out=flags)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        sk.reset()
        sk.stream_run(x, w.batch, w.alpha, flags_out=flags, latencies=False)
    torch.cuda.synchronize()
    e0.record()
    reps = 3
    for _ in range(reps):
        sk.reset()
        sk.stream_run(x, w.batch, w.alpha, flags_out=flags, latencies=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    sk.reset()
    _, lat, _ = sk.stream_run(x, w.batch, w.alpha, flags_out=flags)
    print(f"group {g}: {n / ms * 1e3:.3e} pts/s, {ms / (n / w.batch) * 1e3:.1f} us/batch, "
          f"latency p50 {np.percentile(lat, 50):.3f} p99 {np.percentile(lat, 99):.3f} ms")
