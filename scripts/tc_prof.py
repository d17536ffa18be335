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
out = (C.c_ulonglong * 32)()
N.dev().ace_debug_tc_prof.argtypes = [C.c_void_p]
N.dev().ace_debug_tc_prof(out)
grid = 148
names = ["prod a_empty", "prod w_empty", "mma a_full", "mma acc_empty", "mma w_full", "epi acc_full(x8 warps)",
         "producer end", "mma end", "epilogue loop end (w2)", "epilogue tail end (w2)"]
tot = out[9] / grid
print(f"cfg {cfg} n={n} kernel cycles per CTA ~ {tot:.0f}; globaltimer span {(out[11] - out[10]) / 1e3:.1f} us")
for i, nm in enumerate(names):
    print(f"  {nm:24s} {out[i] / grid:12.0f} cycles/CTA  ({100 * out[i] / grid / tot:5.1f}% of kernel)")
print(f"  max over CTAs: tail end {out[12]}  loop end {out[13]}  near items {out[14]} (avg {out[15] if False else 0})")
print("  epilogue warp 2 per CTA: TMEM ld+wait %.0f  processing %.0f  arrive+pair barrier %.0f  extraction %.0f  acc_full wait %.0f" % (
    out[16] / grid, out[17] / grid, out[18] / grid, out[19] / grid, out[5] / grid / 8))
if out[21]:
    print("  MMA warp: %d groups of 12 MMAs per CTA, %.0f cycles issue time per group (%.1f per MMA)" % (out[21] / grid, out[20] / out[21], out[20] / out[21] / 12))
print("  MMA lane per CTA: loop %.0f = issue %.0f + A copies %.0f + waits %.0f + other %.0f" % (out[23] / grid, out[20] / grid, out[22] / grid, out[24] / grid, (out[23] - out[20] - out[22] - out[24]) / grid))
print("  MMA lane per CTA: tcgen05 fence after acc_empty %.0f" % (out[25] / grid))
if out[21]:
    print("  MMA issuing lane per CTA: W-full waits %.0f  commits %.0f  (per group: %.0f / %.0f)" % (
        out[26] / grid, out[27] / grid, out[26] / out[21], out[27] / out[21]))
print("  near-tie slots per CTA: pushed %.0f, reached by the recheck warps during the main loop %.0f" % (out[29] / grid, out[28] / grid))
