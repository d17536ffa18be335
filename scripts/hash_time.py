"""Device time of the projection alone (ace_family_buckets, phase timing off):
CUDA events around repeated hashing of one config's rows."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

tag = sys.argv[1] if len(sys.argv) > 1 else "lib"
out = []
for cfg, rows in ((5, 262144), (2, None), (3, 2000000)):
    w = W.CONFIGS[cfg]
    n = rows or w.n
    x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
    W.device_rows(cfg, 0, n, x.data_ptr())
    fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.set_stream(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        sk.score_sums(x[:8]) if False else fam.buckets(x[:1024])
    import ctypes as C
    from paper_1706_06664_b200 import _native as N
    ids = torch.empty((w.num_tables, n), dtype=torch.int32, device="cuda")
    st = N.AceHashStats()
    fn = N.dev().ace_family_buckets
    def run():
        fn(fam.handle, x.data_ptr(), N.ACE_F32, n, w.dim, N.ACE_DEVICE, ids.data_ptr(), N.ACE_DEVICE, C.byref(st))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    out.append(f"cfg{cfg}:{e0.elapsed_time(e1) / reps * 1e3:.1f}us")
print(tag, " ".join(out))
