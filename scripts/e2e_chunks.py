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

# the C-ABI call alone (host rows in, host flag bitmap out), as a C/C++ caller makes it
import ctypes as C
import numpy as np
from paper_1706_06664_b200 import _native as N
p = ace._Points(xnp, w.dim)
bits = np.zeros((n + 31) // 32, dtype=np.uint32)
rep = N.AceBatchReport()
st = N.AceHashStats()
fn = N.dev().ace_sketch_build_detect
ts = []
for _ in range(15):
    t0 = time.perf_counter()
    sk.reset()
    assert fn(sk._h, p.ptr, p.dtype, p.n, p.ld, p.where, bits.ctypes.data, None, N.ACE_HOST, C.byref(rep), C.byref(st)) == 0
    ts.append(time.perf_counter() - t0)
ts.sort()
print(f"C-ABI call: median {ts[len(ts)//2]*1e3:.3f} ms min {ts[0]*1e3:.3f} ms -> {n / ts[len(ts)//2]:.4g} points/s")
