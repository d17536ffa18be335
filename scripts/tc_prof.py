"""Wait-cycle breakdown of the tcgen05 projection kernel (ACE_TC_PROF=1)."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["ACE_TC_PROF"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = W.CONFIGS[cfg]
n = min(w.n, 2_000_000)
x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
W.device_rows(cfg, 0, n, x.data_ptr())
fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
sk = ace.AceSketch(fam, ace.CounterWidth.k32)
for _ in range(3):
    sk.reset()
    sk.build_detect(x)
out = (C.c_ulonglong * 8)()
N.dev().ace_debug_tc_prof.argtypes = [C.c_void_p]
N.dev().ace_debug_tc_prof(out)
grid = 148
names = ["prod a_empty", "prod w_empty", "mma a_full", "mma acc_empty", "mma w_full", "epi acc_full(x4 warps)", "total(prod warp)"]
tot = out[6] / grid
print(f"cfg {cfg} n={n} kernel cycles per CTA ~ {tot:.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:24s} {out[i] / grid:12.0f} cycles/CTA  ({100 * out[i] / grid / tot:5.1f}% of kernel)")
