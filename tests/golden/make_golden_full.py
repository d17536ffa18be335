"""Generate tests/golden/golden_full.json: digests of every hot-path output of
BASELINE configurations 3, 4 and 5 at FULL size (10M rows, 1M rows, and all
1,526 stream batches of 100M rows).

Checker only (test infrastructure).  The CPU side is the C oracle
(oracle/ace_oracle.c), which tests/test_cpu_oracle.py and
tests/golden/golden.json pin to the compiled reference:
  - bucket ids: ora_buckets_fast, the reference's sequential binary64 fold
    (srp.cpp:78-113) with 64 rows side by side as vector lanes (bit-identical
    to the scalar fold; checked here again on the first rows of every config
    against the compiled reference's own SrpFamily::bucket when
    oracle/_ref/libaceref.so is present);
  - counters, n and the reference's rounded mean recurrence: ora_insert_batch
    (sketch.cpp:50-72), rows in index order (estimators.cpp:79-92);
  - scores: ora_score_batch (sketch.cpp:108-116);
  - detect_batch statistics and flags: ora_detect_batch_from_scores
    (detect.cpp:44-68);
  - the stream: ora_stream_batch per 65,536-row batch (detect.cpp:76-84 on
    the counts at batch start, then insert; ace_cli.cpp:173-186).
Also recorded per stream batch: the exact mean T/(nL) (T = sum of squared
counters, no saturation at k32) next to the reference's rounded one, and how
many rows of the next batch would flip between the two cuts (mean - alpha) —
the evidence that a device path using the exact mean flags exactly what the
reference flags on this stream.

Inputs come from the synthetic generators (csrc/datagen_core.h), which are
bit-identical on the host and the device, so the GPU test regenerates the
same rows in HBM.

Run in the dev container:  python tests/golden/make_golden_full.py [cfg ...]
(about 10 minutes on 8 cores).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from fractions import Fraction
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import REF_SO, Oracle, Reference, detect_from_scores  # noqa: E402
from paper_1706_06664_b200 import workloads as W  # noqa: E402

OUT = ROOT / "tests" / "golden" / "golden_full.json"
CHUNK = 1 << 20          # rows per ids digest chunk (batch configs)
STREAM_CHUNK_BATCHES = 16  # batches per device generation chunk of the GPU test (ids digested per batch)
NEAR_EPS = 1e-6          # BASELINE.json near-tie measure |<x,w>| < 1e-6 |x||w|


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def exact_mean(counters: np.ndarray, n: int, l: int) -> Fraction:
    c = counters.astype(np.uint64)
    t = int((c * c).sum(dtype=np.uint64))  # < 2^64 at these sizes
    return Fraction(t, n * l)


def pin_prefix(cfg: int, o: Oracle, wmat, rows: int = 256) -> bool:
    """The fast fold against the compiled reference's SrpFamily::bucket."""
    if not REF_SO.exists():
        return False
    w = W.CONFIGS[cfg]
    x, _ = W.host_rows(cfg, 0, rows)
    ref = Reference().buckets(w.w_seed, x, w.k_bits, w.num_tables)
    ids, _ = o.buckets(wmat, x, w.k_bits, w.num_tables)
    if not np.array_equal(ref, ids):
        raise SystemExit(f"cfg {cfg}: fast oracle differs from the compiled reference")
    return True


def batch_config(cfg: int, o: Oracle) -> dict:
    w = W.CONFIGS[cfg]
    n = w.n
    wmat = o.directions(w.w_seed, w.dim, w.k_bits, w.num_tables)
    pinned = pin_prefix(cfg, o, wmat)
    ids = np.empty((w.num_tables, n), dtype=np.uint32)
    h_ids = hashlib.sha256()
    near = 0
    lab_count = 0
    labels = np.empty(n, dtype=np.uint8)
    for r0 in range(0, n, CHUNK):
        m = min(CHUNK, n - r0)
        x, lab = W.host_rows(cfg, r0, m)
        labels[r0:r0 + m] = lab
        lab_count += int((lab != 0).sum())
        part, nr = o.buckets(wmat, x, w.k_bits, w.num_tables, rel_eps=NEAR_EPS)
        near += nr
        h_ids.update(part.tobytes())
        ids[:, r0:r0 + m] = part
        print(f"  cfg {cfg}: rows {r0 + m}/{n}", flush=True)
    sk = o.sketch(w.k_bits, w.num_tables, 32)
    sk.insert_ids(ids)
    scores, sums = sk.score_ids(ids)
    mean, sd, thr, flags = detect_from_scores(o, scores)
    counters = sk.counters().astype(np.uint32)
    em = exact_mean(counters, n, w.num_tables)
    return dict(
        n=n, dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, w_seed=w.w_seed,
        data_seed=w.data_seed, w_sha256=sha(wmat), ids_chunk_rows=CHUNK, ids_sha256=h_ids.hexdigest(),
        near_tie_1e6=near, pinned_to_reference_prefix=pinned,
        counters_sha256=sha(counters), size=int(sk.size()), mean=float(sk.mean()).hex(),
        mean_exact=float(em).hex(), sums_sha256=sha(sums), scores_sha256=sha(scores),
        det_mean=float(mean).hex(), det_sd=float(sd).hex(), det_thr=float(thr).hex(),
        reported=int(flags.sum()), flags_sha256=sha(np.packbits(flags, bitorder="little")),
        correctly_reported=int((flags & (labels != 0)).sum()), labeled=lab_count)


def stream_config(o: Oracle) -> dict:
    w = W.CONFIGS[5]
    wmat = o.directions(w.w_seed, w.dim, w.k_bits, w.num_tables)
    pinned = pin_prefix(5, o, wmat)
    sk = o.sketch(w.k_bits, w.num_tables, 32)
    nb = (w.n + w.batch - 1) // w.batch
    h_ids, h_scores = hashlib.sha256(), hashlib.sha256()
    per = []
    near = 0
    reported = 0
    min_gap = None   # smallest |score - cut| over the stream, in units of 1/L
    flips_exact = 0  # rows whose flag differs under the exact mean's cut
    max_rel = 0.0    # max |mean_ref - mean_exact| / mean_exact
    for b in range(nb):
        r0 = b * w.batch
        m = min(w.batch, w.n - r0)
        x, _ = W.host_rows(5, r0, m)
        ids, nr = o.buckets(wmat, x, w.k_bits, w.num_tables, rel_eps=NEAR_EPS)
        near += nr
        h_ids.update(ids.tobytes())
        n_before = int(sk.size())
        mean_before = float(sk.mean())
        if n_before:
            c = sk.counters().astype(np.uint32)
            em = exact_mean(c, n_before, w.num_tables)
            emf = float(em)
            max_rel = max(max_rel, abs(mean_before - emf) / emf if emf else 0.0)
        fl, sc = sk.stream_ids(ids, w.alpha)
        h_scores.update(sc.tobytes())
        if n_before:
            # flags under the exact cut (exact rational comparison S/L <= mean - alpha)
            S = np.rint(sc * w.num_tables).astype(np.int64)
            cut_exact = em - Fraction(w.alpha)
            # S/L <= cut  <=>  S <= floor(cut * L)
            lim = (cut_exact * w.num_tables).numerator // (cut_exact * w.num_tables).denominator
            fl_exact = S <= lim
            flips_exact += int((fl_exact != fl).sum())
            cut_ref = Fraction(mean_before) - Fraction(w.alpha)
            gaps = np.abs(S.astype(np.float64) - float(cut_ref * w.num_tables))
            g = float(gaps.min())
            min_gap = g if min_gap is None else min(min_gap, g)
        reported += int(fl.sum())
        per.append([sha(np.packbits(fl, bitorder="little"))[:16], int(fl.sum()), float(sk.mean()).hex()])
        if b % 100 == 0 or b == nb - 1:
            print(f"  cfg 5: batch {b + 1}/{nb} reported {reported}", flush=True)
    c = sk.counters().astype(np.uint32)
    return dict(
        n=w.n, dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, w_seed=w.w_seed, data_seed=w.data_seed,
        batch=w.batch, alpha=w.alpha, batches=nb, w_sha256=sha(wmat),
        ids_chunk_batches=STREAM_CHUNK_BATCHES, ids_sha256=h_ids.hexdigest(), scores_sha256=h_scores.hexdigest(),
        near_tie_1e6=near, pinned_to_reference_prefix=pinned, reported=reported,
        per_batch_fields=["flags_sha256[:16]", "reported", "mean_after (reference recurrence, hex)"],
        per_batch=per, counters_sha256=sha(c), size=int(sk.size()), mean=float(sk.mean()).hex(),
        mean_exact=float(exact_mean(c, w.n, w.num_tables)).hex(),
        exact_vs_reference_mean={"max_rel_diff": max_rel, "rows_flagged_differently_under_exact_cut": flips_exact,
                                 "min_score_to_cut_gap_in_1_over_L": min_gap})


def main() -> None:
    cfgs = [int(a) for a in sys.argv[1:]] or [3, 4, 5]
    out = json.loads(OUT.read_text()) if OUT.exists() else {
        "generator": "tests/golden/make_golden_full.py",
        "checker": "C oracle (oracle/ace_oracle.c), pinned to the compiled reference", "configs": {}}
    o = Oracle()
    for cfg in cfgs:
        t0 = time.time()
        e = stream_config(o) if cfg == 5 else batch_config(cfg, o)
        e["seconds"] = round(time.time() - t0, 1)
        e["threads"] = os.cpu_count()
        out["configs"][str(cfg)] = e
        OUT.write_text(json.dumps(out, indent=1))
        print(cfg, e["reported"], e["seconds"], "s", flush=True)


if __name__ == "__main__":
    main()
