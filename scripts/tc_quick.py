"""Quick tcgen05-path check against the C oracle (dev tool)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from oracle import Oracle
from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

o = Oracle()
for (d, k, l, n) in [(40, 15, 50, 1000), (120, 15, 50, 5000), (64, 15, 50, 300), (128, 16, 100, 3000), (200, 18, 64, 700), (7, 3, 5, 100), (300, 15, 20, 500), (1000, 18, 64, 700), (4096, 18, 64, 300)]:
    fam = ace.SrpFamily(ace.SrpConfig(dim=d, k_bits=k, num_tables=l, seed=3))
    x = np.random.default_rng(d).standard_normal((n, d)).astype(np.float32)
    st = N.AceHashStats()
    t0 = time.time()
    ids = fam.buckets(x, stats=st)
    ref, near = o.buckets(fam.directions, x, k, l, rel_eps=1e-6)
    bad = int((ids != ref).sum())
    print(f"d={d} K={k} L={l} n={n} kernel={fam.kernel()} mismatches={bad} rechecked={st.rechecked} "
          f"flipped={st.flipped} near1e-6={near} t={time.time()-t0:.2f}s", flush=True)
    if bad:
        r, c = np.nonzero(ids != ref)
        print("  first:", r[:5], c[:5], ids[r[:5], c[:5]], ref[r[:5], c[:5]])
