"""Full-size parity: BASELINE configurations 3, 4 and 5 at their full sizes
(10M rows, 1M rows at d = 4096, all 1,526 stream batches of 100M rows) against
tests/golden/golden_full.json, made by tests/golden/make_golden_full.py with
the C oracle (pinned to the compiled reference; sketch.cpp:50-72,
detect.cpp:12-74, detect.cpp:76-84).

Compared bit for bit: SHA-256 of every bucket id, the final counters, the
integer score sums, the scores, the flags (per batch for the stream), the
near-tie count |p| < 1e-6 |x||w|, n and the exact mean; the detect_batch
statistics within 1e-9 relative (the reference's are order-dependent binary64
sums); the stream's per-batch mean within 1e-9 relative of the reference's
rounded recurrence.  Rows are generated on the device by the same generator
that made the fixture on the host (bit-identical, csrc/datagen_core.h)."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "golden_full.json").read_text())["configs"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rel_close(a, b, tol=1e-9):
    return abs(a - b) <= tol * max(abs(a), abs(b), 1e-300)


def family(cfg):
    w = W.CONFIGS[cfg]
    return ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))


@pytest.mark.parametrize("cfg", [3, 4])
def test_full_batch_config_matches_oracle(cuda, cfg):
    torch = cuda
    g = GOLD[str(cfg)]
    w = W.CONFIGS[cfg]
    fam = family(cfg)
    assert sha(fam.directions) == g["w_sha256"]
    xd = torch.empty((w.n, w.dim), dtype=torch.float32, device="cuda")
    W.device_rows(cfg, 0, w.n, xd.data_ptr())
    # bucket ids, chunk by chunk as the fixture digests them
    h = hashlib.sha256()
    near = 0
    for r0 in range(0, w.n, g["ids_chunk_rows"]):
        st = N.AceHashStats()
        ids = fam.buckets(xd[r0:r0 + g["ids_chunk_rows"]], stats=st)
        near += st.near_ties
        h.update(ids.tobytes())
    assert h.hexdigest() == g["ids_sha256"]
    assert near == g["near_tie_1e6"]
    # build_sketch + detect_batch in one call
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    scores = torch.empty(w.n, dtype=torch.float64, device="cuda")
    flags = torch.zeros((w.n + 31) // 32, dtype=torch.int32, device="cuda")
    rep = sk.build_detect(xd, flags_out=flags, scores_out=scores)
    assert sha(sk.counters_u32()) == g["counters_sha256"]
    assert sk.size() == g["size"]
    assert sk.mean() == float.fromhex(g["mean_exact"])
    assert rel_close(sk.mean(), float.fromhex(g["mean"]))
    assert sha(scores.cpu().numpy()) == g["scores_sha256"]
    bits = flags.cpu().numpy().view(np.uint32)
    fl = ((bits[:, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool).reshape(-1)[:w.n]
    assert sha(np.packbits(fl, bitorder="little")) == g["flags_sha256"]
    assert rep.reported == g["reported"]
    assert rel_close(rep.score_mean, float.fromhex(g["det_mean"]))
    assert rel_close(rep.score_stddev, float.fromhex(g["det_sd"]))
    assert rel_close(rep.threshold, float.fromhex(g["det_thr"]))
    # integer score sums against the final counters
    assert sha(sk.score_sums(xd)) == g["sums_sha256"]
    del xd
    torch.cuda.empty_cache()


def test_full_stream_config5_matches_oracle(cuda):
    torch = cuda
    g = GOLD["5"]
    w = W.CONFIGS[5]
    fam = family(5)
    assert sha(fam.directions) == g["w_sha256"]
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    chunk = g["ids_chunk_batches"] * w.batch
    h_ids, h_sc = hashlib.sha256(), hashlib.sha256()
    near = reported = ambiguous = 0
    b = 0
    xd = torch.empty((chunk, w.dim), dtype=torch.float32, device="cuda")
    for c0 in range(0, w.n, chunk):
        m = min(chunk, w.n - c0)
        W.device_rows(5, c0, m, xd.data_ptr())
        for b0 in range(0, m, w.batch):  # ids digested batch by batch, as the fixture
            st = N.AceHashStats()
            h_ids.update(fam.buckets(xd[b0:min(m, b0 + w.batch)], stats=st).tobytes())
            near += st.near_ties
        for b0 in range(0, m, w.batch):
            fl, sc, rep = sk.stream_batch(xd[b0:min(m, b0 + w.batch)], w.alpha, scores=True)
            fsha, frep, mean_after = g["per_batch"][b]
            assert sha(np.packbits(fl, bitorder="little"))[:16] == fsha, f"batch {b}"
            assert rep.reported == frep, f"batch {b}"
            assert rel_close(sk.mean(), float.fromhex(mean_after)), f"batch {b}"
            h_sc.update(sc.tobytes())
            reported += rep.reported
            ambiguous += rep.ambiguous
            b += 1
    assert b == g["batches"]
    assert h_ids.hexdigest() == g["ids_sha256"]
    assert h_sc.hexdigest() == g["scores_sha256"]
    assert near == g["near_tie_1e6"]
    assert reported == g["reported"]
    assert sha(sk.counters_u32()) == g["counters_sha256"]
    assert sk.size() == g["size"]
    assert sk.mean() == float.fromhex(g["mean_exact"])
    # the exact-mean cut flags what the reference's rounded recurrence flags
    # on this stream (fixture: 0 rows differ), and no score sits inside the
    # stream's ambiguity band
    assert g["exact_vs_reference_mean"]["rows_flagged_differently_under_exact_cut"] == 0
    assert ambiguous == 0


@pytest.mark.parametrize("group,pipe", [(4, 0), (8, 90)])
def test_full_stream_run_config5_matches_oracle(cuda, group, pipe):
    """The streaming driver (ace_sketch_stream_run; one stream launch per
    hashing group, and pipelined: the next group's projection on `pipe` SMs
    beside the one-CTA-per-table stream kernel) over all 100M rows at once:
    per-batch flag digests, counters and n as the oracle's."""
    torch = cuda
    g = GOLD["5"]
    w = W.CONFIGS[5]
    sk = ace.AceSketch(family(5), ace.CounterWidth.k32)
    sk.set_option(N.ACE_OPT_STREAM_GROUP, group)
    sk.set_option(N.ACE_OPT_STREAM_PIPE, pipe)
    xd = torch.empty((w.n, w.dim), dtype=torch.float32, device="cuda")
    chunk = 8 * 1024 * 1024
    for r0 in range(0, w.n, chunk):
        m = min(chunk, w.n - r0)
        W.device_rows(5, r0, m, xd[r0:r0 + m].data_ptr())
    flags = torch.zeros((w.n + 31) // 32, dtype=torch.int32, device="cuda")
    _, lat, rep = sk.stream_run(xd, w.batch, w.alpha, flags_out=flags)
    del xd
    torch.cuda.empty_cache()
    bits = flags.cpu().numpy().view(np.uint32)
    words = w.batch // 32
    for b in range(g["batches"]):
        wb = bits[b * words:(b + 1) * words]
        rows = min(w.batch, w.n - b * w.batch)
        fl = ((wb[:, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool).reshape(-1)[:rows]
        assert sha(np.packbits(fl, bitorder="little"))[:16] == g["per_batch"][b][0], f"batch {b}"
    assert rep.reported == g["reported"]
    assert rep.ambiguous == 0
    assert sha(sk.counters_u32()) == g["counters_sha256"]
    assert sk.size() == g["size"]
    assert sk.mean() == float.fromhex(g["mean_exact"])
    assert len(lat) == g["batches"] and float(np.max(lat)) > 0.0
