"""CPU tests: the C oracle is pinned to the compiled reference and to the
committed golden digests; the synthetic generators are deterministic."""
import hashlib

import numpy as np
import pytest

from oracle import detect_from_scores
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_host_w_generator_matches_oracle(oracle_c):
    # libace.so's SrpFamily W (rng.hpp:36-58, srp.cpp:36-48) == the C oracle
    for (d, k, l, s) in [(40, 15, 50, 1), (7, 5, 6, 321), (3, 4, 2, 77), (128, 16, 3, 9)]:
        assert np.array_equal(ace.generate_directions(s, d, k, l), oracle_c.directions(s, d, k, l))


def test_oracle_w_matches_golden(oracle_c, golden):
    for cfg, e in golden["configs"].items():
        w = oracle_c.directions(e["w_seed"], e["dim"], e["k_bits"], e["num_tables"])
        assert sha(w) == e["w_sha256"], cfg


def test_datagen_deterministic_and_prefix_consistent():
    for cfg in (1, 2, 3, 5):
        x, lab = W.host_rows(cfg, 0, 300)
        y, lab2 = W.host_rows(cfg, 100, 50, threads=1)
        assert np.array_equal(x[100:150], y) and np.array_equal(lab[100:150], lab2)
        assert np.isfinite(x).all()
    x, _ = W.host_rows(4, 0, 3)
    assert x.shape == (3, 4096) and np.isfinite(x).all()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_oracle_against_golden_batch(oracle_c, golden, cfg):
    """C oracle reproduces the reference's ids, counters, mean, scores and
    detect_batch flags for the golden rows (configs 3/4 on a sub-prefix to
    keep the CPU suite short; the GPU suite covers the full golden rows)."""
    e = golden["configs"][str(cfg)]
    n = e["n"]
    x, lab = W.host_rows(cfg, 0, n)
    assert sha(x) == e["x_sha256"], "synthetic generator drifted"
    w = oracle_c.directions(e["w_seed"], e["dim"], e["k_bits"], e["num_tables"])
    ids, _ = oracle_c.buckets(w, x, e["k_bits"], e["num_tables"])
    assert sha(ids) == e["ids_sha256"]
    sk = oracle_c.sketch(e["k_bits"], e["num_tables"], 32)
    sk.insert_ids(ids)
    assert sha(sk.counters().astype(np.uint32)) == e["counters_sha256"]
    assert sk.mean() == float.fromhex(e["mean"])
    sc, _ = sk.score_ids(ids)
    assert sha(sc) == e["scores_sha256"]
    m, s, t, fl = detect_from_scores(oracle_c, sc)
    assert (m, s, t) == (float.fromhex(e["det_mean"]), float.fromhex(e["det_sd"]),
                         float.fromhex(e["det_thr"]))
    assert sha(np.packbits(fl, bitorder="little")) == e["flags_sha256"]
    assert int(fl.sum()) == e["reported"]


def test_oracle_against_golden_stream(oracle_c, golden):
    e = golden["configs"]["5"]
    w = oracle_c.directions(e["w_seed"], e["dim"], e["k_bits"], e["num_tables"])
    sk = oracle_c.sketch(e["k_bits"], e["num_tables"], 32)
    for b, pb in enumerate(e["per_batch"][:2]):
        x, _ = W.host_rows(5, b * e["batch"], e["batch"])
        assert sha(x) == pb["x_sha256"]
        ids, _ = oracle_c.buckets(w, x, e["k_bits"], e["num_tables"])
        fl, sc = sk.stream_ids(ids, e["alpha"])
        assert sha(np.packbits(fl, bitorder="little")) == pb["flags_sha256"]
        assert sha(sc) == pb["scores_sha256"]
        assert sk.mean() == float.fromhex(pb["mean_after"])


def test_oracle_pinned_to_compiled_reference(oracle_c, reference):
    """Where the compiled reference is present: random shapes, the C oracle
    equals the reference bit-for-bit (ids, counters, mean, detect, stream)."""
    rng = np.random.default_rng(5)
    for (d, k, l, seed) in [(5, 3, 4, 99), (9, 15, 50, 1), (33, 7, 11, 12345)]:
        x = (rng.standard_normal((3000, d)) * rng.uniform(0.1, 10)).astype(np.float32)
        x[::97] = 0.0  # zero rows: sign(0) -> 1
        w = oracle_c.directions(seed, d, k, l)
        assert np.array_equal(w, reference.directions(seed, d, k, l))
        ids, _ = oracle_c.buckets(w, x, k, l)
        assert np.array_equal(ids, reference.buckets(seed, x, k, l))
        rs = reference.sketch(seed, d, k, l, 32)
        rs.insert(x)
        os_ = oracle_c.sketch(k, l, 32)
        os_.insert_ids(ids)
        assert np.array_equal(rs.counters(), os_.counters())
        assert rs.mean() == os_.mean()
        det = rs.detect_batch(x)
        m, s, t, fl = detect_from_scores(oracle_c, os_.score_ids(ids)[0])
        assert (det["mean"], det["sd"], det["thr"]) == (m, s, t)
        assert np.array_equal(det["flags"], fl)
        # stream order
        rs2 = reference.sketch(seed, d, k, l, 32)
        os2 = oracle_c.sketch(k, l, 32)
        for part in np.array_split(np.arange(3000), 3):
            f1, s1 = rs2.stream_batch(x[part], 1.0)
            f2, s2 = os2.stream_ids(ids[:, part], 1.0)
            assert np.array_equal(f1, f2) and np.array_equal(s1, s2)
        assert rs2.mean() == os2.mean()


def test_oracle_k16_saturation_matches_reference(oracle_c, reference):
    d, k, l, seed = 3, 2, 2, 4
    x = np.tile(np.array([[0.5, -1.0, 2.0]], dtype=np.float32), (70000, 1))
    rs = reference.sketch(seed, d, k, l, 16)
    rs.insert(x)
    w = oracle_c.directions(seed, d, k, l)
    ids, _ = oracle_c.buckets(w, x, k, l)
    os_ = oracle_c.sketch(k, l, 16)
    os_.insert_ids(ids)
    assert rs.saturated() and os_.saturated()
    assert np.array_equal(rs.counters(), os_.counters())
    assert rs.mean() == os_.mean()
