"""Phase timeline of the fused detect tail (ACE_TAIL_PROF=1): counts, gather, scores + threshold, flags."""
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

for cfg in [int(c) for c in (sys.argv[1:] or ["2"])]:
    w = W.CONFIGS[cfg]
    n = min(w.n, 10_000_000)
    x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
    W.device_rows(cfg, 0, n, x.data_ptr())
    fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    out = (C.c_ulonglong * 8)()
    N.dev().ace_debug_tail_prof.argtypes = [C.c_void_p]
    rows = []
    for _ in range(4):
        sk.reset()
        sk.build_detect(x)
        N.dev().ace_debug_tail_prof(out)
        t = list(out)
        rows.append([(t[i] - t[i - 1]) / 1e3 if t[i] and t[i - 1] else 0.0 for i in range(1, 5)])
    r = rows[-1]
    print(f"cfg {cfg} n={n}: counts {r[0]:.1f} us, gather {r[1]:.1f} us, scores+threshold {r[2]:.1f} us, flags {r[3]:.1f} us")
    del x, sk
