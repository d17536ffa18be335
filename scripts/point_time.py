"""Per-point API (ace_point_bench: detect_stream + insert per query through
include/ace/*.hpp) against the reference's per-point loop (oracle/_ref,
ref_time_point) on the same rows: rate, latency, and whether the scores and
flags agree."""
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import Reference  # noqa: E402
from paper_1706_06664_b200 import workloads as W  # noqa: E402

NB, NQ = 65536, int(sys.argv[1]) if len(sys.argv) > 1 else 10000
for cfg in (5, 2):
    w = W.CONFIGS[cfg]
    x, _ = W.host_rows(cfg, 0, NB + NQ)
    with tempfile.TemporaryDirectory() as td:
        f = Path(td) / "rows.f32"
        o = Path(td) / "out.bin"
        x.astype(np.float32).tofile(f)
        r = subprocess.run([str(ROOT / "paper_1706_06664_b200/lib/ace_point_bench"), str(w.dim), str(w.k_bits),
                            str(w.num_tables), str(w.w_seed), repr(w.alpha), str(NB), "0", str(NQ), str(f), str(o)],
                           capture_output=True, text=True, check=True)
        sec, rep, p50, p99, tdet, nl = r.stdout.split()
        raw = o.read_bytes()
        sc = np.frombuffer(raw[:8 * NQ], dtype=np.float64)
        fl = np.frombuffer(raw[8 * NQ:], dtype=np.uint8)
    rs, rrep, rsc, rfl = Reference().time_point(w.w_seed, x, NB, w.k_bits, w.num_tables, w.alpha, outputs=True)
    print(f"cfg{cfg}: b200 {NQ / float(sec):.0f} pts/s (p50 {p50} us p99 {p99} us, in detect_stream {tdet} us, reported {rep}) | "
          f"reference {NQ / rs:.0f} pts/s (reported {rrep}) | scores equal {np.array_equal(sc, rsc)} "
          f"flags equal {np.array_equal(fl, rfl)}", flush=True)
