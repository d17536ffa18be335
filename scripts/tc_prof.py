"""Section cycles of the projection kernel (a -DACE_TC_PROF=1 build of
libace_dev.so): per CTA and point tile, for one config's hashing."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rows = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = W.CONFIGS[cfg]
n = rows or w.n
x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
W.device_rows(cfg, 0, n, x.data_ptr())
fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
out = (C.c_ulonglong * 24)()
if not hasattr(N.dev(), "ace_debug_tc_prof"):  # a regular build: just run the hashing (ncu target)
    for _ in range(8):
        fam.buckets(x)
    torch.cuda.synchronize()
    sys.exit(0)
f = N.dev().ace_debug_tc_prof
f.argtypes = [C.c_void_p, C.c_int]
for _ in range(3):
    fam.buckets(x)
f(out, 1)
reps = 5
for _ in range(reps):
    fam.buckets(x)
f(out, 1)
tiles = (n + 127) // 128
ctas = min(148, tiles)
per = [v / reps / ctas for v in out]
tpc = tiles / ctas
names = {0: "mma wait A", 1: "mma wait acc-empty", 2: "mma wait W", 3: "mma loop total",
         5: "conv wait raw", 6: "conv pass1", 7: "conv wait A/thr free", 8: "conv pass2", 9: "conv publish",
         10: "epi wait thr + sgn free", 11: "epi wait acc-full", 12: "epi TMEM ld + process", 13: "epi sign words",
         14: "pack buckets", 15: "pack wait sgn", 16: "kernel total (thread 0)"}
print(f"cfg {cfg} n {n}: {tpc:.1f} tiles per CTA; cycles per CTA (per tile)")
if out[22]:
    c = out[22]
    print(f"  per CTA from entry: prologue {out[17] / c:.0f}, first MMA {out[18] / c:.0f}, tail start {out[19] / c:.0f}, "
          f"tail end {out[20] / c:.0f}, kernel end {out[21] / c:.0f} cycles")
for k, nm in names.items():
    print(f"  {nm:26s} {per[k]:10.0f} ({per[k] / tpc:7.0f})")
