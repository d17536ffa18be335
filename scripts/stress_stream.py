"""Repeat the pipelined stream driver over the whole config-5 stream and compare
flag and counter digests between repetitions (and with the un-pipelined run)."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
w = W.CONFIGS[5]
n = w.n
x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
for r0 in range(0, n, 8 << 20):
    m = min(8 << 20, n - r0)
    W.device_rows(5, r0, m, x[r0:r0 + m].data_ptr())
fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
flags = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")


def run(sk):
    sk.reset()
    flags.zero_()
    _, _, rep = sk.stream_run(x, w.batch, w.alpha, flags_out=flags, latencies=False)
    return (hashlib.sha256(flags.cpu().numpy().tobytes()).hexdigest()[:16],
            hashlib.sha256(sk.counters_u32().tobytes()).hexdigest()[:16], int(rep.reported), sk.mean())


base = ace.AceSketch(fam, ace.CounterWidth.k32)
base.set_option(N.ACE_OPT_STREAM_GROUP, 8)
base.set_option(N.ACE_OPT_STREAM_PIPE, 0)
want = run(base)
print("un-pipelined:", want)
bad = 0
for g, p in ((8, 90), (8, 84), (3, 94), (16, 90)):
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.set_option(N.ACE_OPT_STREAM_GROUP, g)
    sk.set_option(N.ACE_OPT_STREAM_PIPE, p)
    for i in range(reps):
        got = run(sk)
        if got != want:
            bad += 1
            print("MISMATCH", g, p, i, got)
    print(f"G {g} P {p}: {reps} runs done, mismatches so far {bad}")
print("stress:", "OK" if bad == 0 else f"{bad} MISMATCHES")

# pinned host rows (eager launches, H2D copies of the next group on the copy stream)
m = 16 * 1024 * 1024 + 4160
xh = torch.empty((m, w.dim), dtype=torch.float32, pin_memory=True)
xh.copy_(x[:m])
xd = x[:m]
ref = None
bad = 0
for g, p, src in ((8, 0, "dev"), (8, 90, "pin"), (8, 0, "pin"), (5, 92, "pin")):
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.set_option(N.ACE_OPT_STREAM_GROUP, g)
    sk.set_option(N.ACE_OPT_STREAM_PIPE, p)
    for i in range(8):
        sk.reset()
        fl, _, rep = sk.stream_run(xd if src == "dev" else xh.numpy(), w.batch, w.alpha, latencies=False)
        got = (hashlib.sha256(np.packbits(fl).tobytes()).hexdigest()[:16],
               hashlib.sha256(sk.counters_u32().tobytes()).hexdigest()[:16], int(rep.reported))
        ref = ref or got
        if got != ref:
            bad += 1
            print("MISMATCH", g, p, src, i, got)
    print(f"G {g} P {p} {src}: ok so far, mismatches {bad}")
print("host-rows stress:", "OK" if bad == 0 else f"{bad} MISMATCHES")
