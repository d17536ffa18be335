"""Phase marks of the stream kernel (a -DACE_SP_PROF=1 build of libace_dev.so):
average ns from a CTA's start to each mark, phase-A and phase-B CTAs."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

w = W.CONFIGS[5]
n = 40 * w.batch
x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
W.device_rows(5, 0, n, x.data_ptr())
fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
sk = ace.AceSketch(fam, ace.CounterWidth.k32)
flags = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
f = N.dev().ace_debug_sp_prof
f.argtypes = [C.c_void_p, C.c_int]
out = (C.c_ulonglong * 16)()
sk.stream_run(x, w.batch, w.alpha, flags_out=flags)
f(out, 1)
sk.reset()
sk.stream_run(x, w.batch, w.alpha, flags_out=flags)
f(out, 1)
na, nb = out[14], out[15]
names = {0: "A start", 1: "A staged", 2: "A items done", 3: "A cluster sync 1", 4: "A merged", 5: "A cluster sync 2"}
for k, nm in names.items():
    print(f"  {nm:20s} {out[k] / max(na, 1) / 1e3:8.2f} us after CTA start")
print(f"  B start {out[8] / max(nb, 1) / 1e3:8.2f}  B end {out[9] / max(nb, 1) / 1e3:8.2f} us  (A CTAs {na}, B CTAs {nb})")
