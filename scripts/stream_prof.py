"""Phase timeline of the cooperative stream step (ACE_TAIL_PROF=1): scores, insert."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["ACE_TAIL_PROF"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

w = W.CONFIGS[5]
n = 8 * w.batch
x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
W.device_rows(5, 0, n, x.data_ptr())
fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
sk = ace.AceSketch(fam, ace.CounterWidth.k32)
sk.stream_run(x, w.batch, w.alpha)
torch.cuda.synchronize()
out = (C.c_ulonglong * 8)()
N.dev().ace_debug_tail_prof.argtypes = [C.c_void_p]
N.dev().ace_debug_tail_prof(out)
t = list(out)
print(f"stream step (last batch): scores+barrier {(t[6] - t[5]) / 1e3:.1f} us, insert {(t[7] - t[6]) / 1e3:.1f} us")
