"""e2e (pinned host rows -> build_detect -> flags on the host) wall time per call for one
ACE_H2D_CHUNKS setting (read once by the library: one setting per process)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = W.CONFIGS[cfg]
n = w.n
x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
W.device_rows(cfg, 0, n, x.data_ptr())
xh = torch.empty((n, w.dim), dtype=torch.float32, pin_memory=True)
xh.copy_(x)
xnp = xh.numpy()
fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
sk = ace.AceSketch(fam, ace.CounterWidth.k32)
for _ in range(3):
    sk.reset()
    ace._detect(sk, xnp, build=True)
torch.cuda.synchronize()
ts = []
for _ in range(15):
    t0 = time.perf_counter()
    sk.reset()
    ace._detect(sk, xnp, build=True)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
ts.sort()
print(f"chunks={os.environ.get('ACE_H2D_CHUNKS', '8')} cfg{cfg} e2e median {ts[len(ts)//2]*1e3:.3f} ms "
      f"min {ts[0]*1e3:.3f} ms -> {n / ts[len(ts)//2]:.4g} points/s")
