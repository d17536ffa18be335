"""Per-phase device time of the stream path (cfg 5 rows through
ace_sketch_stream_batch with phase timing) at several batch sizes: hash,
phase A (counts at batch start + insert), phase B (scores + flags)."""
import sys
import ctypes as C
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

w = W.CONFIGS[5]
tag = sys.argv[1] if len(sys.argv) > 1 else "lib"
x = torch.empty((48 * w.batch, w.dim), dtype=torch.float32, device="cuda")
W.device_rows(5, 0, 48 * w.batch, x.data_ptr())
fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
for bs in (16384, 65536, 262144):
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    flags = torch.empty(bs // 32, dtype=torch.int32, device="cuda")
    nb = x.shape[0] // bs
    ms = (C.c_double * 5)()
    acc = []
    for b in range(nb):
        if b == nb // 3:
            N.dev().ace_sketch_set_timing(sk.handle, 1)
        sk.stream_batch(x[b * bs:(b + 1) * bs], w.alpha, flags_out=flags)
        if b >= nb // 3:
            N.dev().ace_sketch_timings(sk.handle, ms)
            acc.append(list(ms))
    a = np.array(acc).mean(0) * 1e3
    print(f"{tag} batch {bs}: hash {a[0]:.1f} us  phaseA {a[1]:.1f} us  phaseB {a[2]:.1f} us")
