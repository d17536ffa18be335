"""Insert/detect timing on skewed inputs (many identical rows), for the
shared-histogram merge policy: python scripts/skew_bench.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1706_06664_b200 import ace

n, d = 2_000_000, 32
rng = np.random.default_rng(0)
for name, uniq in (("all-same", 1), ("8-distinct", 8), ("1k-distinct", 1000), ("random", n)):
    base = rng.standard_normal((uniq, d)).astype(np.float32)
    x = torch.from_numpy(base[rng.integers(0, uniq, n)]).cuda()
    fam = ace.SrpFamily(ace.SrpConfig(dim=d, k_bits=15, num_tables=50, seed=1))
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    ts = []
    for rep in range(5):
        sk.reset()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sk.build_detect(x)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name:12s} build_detect {min(ts[1:]):.3f} ms")
