"""Phase marks of the group stream kernels (a -DACE_SP_PROF=1 build of
libace_dev.so), per batch and phase-A CTA: pair kernel (pipe 0) and the
one-CTA-per-table kernel beside the projection (pipe P)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

w = W.CONFIGS[5]
G = 8
n = 40 * w.batch
x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
W.device_rows(5, 0, n, x.data_ptr())
fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
f = N.dev().ace_debug_sp_prof
f.argtypes = [C.c_void_p, C.c_int]
pair = None
for pipe in [int(v) for v in sys.argv[1:]] or [0, 88]:
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.set_option(N.ACE_OPT_STREAM_GROUP, G)
    sk.set_option(N.ACE_OPT_STREAM_PIPE, pipe)
    flags = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
    out = (C.c_ulonglong * 16)()
    sk.stream_run(x, w.batch, w.alpha, flags_out=flags)
    f(out, 1)
    sk.reset()
    sk.stream_run(x, w.batch, w.alpha, flags_out=flags)
    f(out, 1)
    na, nb = max(out[14], 1), max(out[15], 1)
    m = [out[k] / na / 1e3 for k in range(8)]   # us per A CTA (marks 2..5 summed over the group's batches)
    if pipe == 0:
        pair = (m, na)
    elif pair is not None:
        # the pipelined run's last group goes through the pair kernel (2 L CTAs per run): take their share out
        npair = 2 * w.num_tables
        m = [(m[k] * na - pair[0][k] * npair) / (na - npair) for k in range(8)]
    rows = m[2] - m[1] - (m[5] - m[6])
    print(f"pipe {pipe}{' (one CTA per table; the pair-kernel CTAs of the last group taken out)' if pipe and pair else ''}: per phase-A CTA and group of {G} batches (us): staged {m[1]:.1f}; row loops {rows:.1f} "
          f"({rows / G:.2f}/batch); sync1 {m[3] - m[2]:.1f}; merge {m[4] - m[3]:.1f}; sync2+clear {m[5] - m[4]:.1f}; "
          f"phase A end {m[6]:.1f}; B CTAs end {out[9] / nb / 1e3:.1f} (A CTAs {out[14]}, B CTAs {out[15]})")
