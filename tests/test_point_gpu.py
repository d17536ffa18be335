"""The per-point path (point_kernel: insert / score / detect_stream one query
at a time, sketch.hpp:33,42, detect.hpp:34-36) against the C oracle: the
reference's per-point loop (ace_cli.cpp:173-183) restated as one-row stream
batches (detect_stream on the counts before the row, then insert), bit-exact
scores and flags; the C++ drop-in's loop (tests/cpp/point_bench.cpp) the
same; asynchronous inserts seen by every later call; counter() reads one
element."""
import subprocess

import numpy as np
import pytest

from oracle import Oracle
from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _family(cfg):
    w = W.CONFIGS[cfg]
    return w, ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))


def _oracle_loop(w, fam, x, nb):
    """Scores and flags of rows nb.. under the one-query-at-a-time loop."""
    o = Oracle()
    wm = o.directions(w.w_seed, w.dim, w.k_bits, w.num_tables)
    ids, _ = o.buckets(wm, x, w.k_bits, w.num_tables)
    sk = o.sketch(w.k_bits, w.num_tables, 32)
    sk.insert_ids(np.ascontiguousarray(ids[:, :nb]))
    sc, fl = [], []
    for i in range(nb, x.shape[0]):
        f, s = sk.stream_ids(np.ascontiguousarray(ids[:, i:i + 1]), w.alpha)
        sc.append(s[0])
        fl.append(bool(f[0]))
    return np.array(sc), np.array(fl), sk


@pytest.mark.parametrize("cfg,dtype", [(5, np.float64), (2, np.float32)])
def test_point_loop_matches_oracle(cuda, cfg, dtype):
    w, fam = _family(cfg)
    nb, nq = 4096, 400
    x, _ = W.host_rows(cfg, 0, nb + nq)
    want_sc, want_fl, osk = _oracle_loop(w, fam, x, nb)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.insert(x[:nb])
    xs = x.astype(dtype)
    sc, fl = [], []
    for i in range(nb, nb + nq):
        est, flag = ace.detect_stream(sk, xs[i], w.alpha)
        sc.append(est.value)
        fl.append(flag)
        sk.insert(xs[i])
    assert np.array_equal(np.array(sc), want_sc)
    assert np.array_equal(np.array(fl), want_fl)
    assert sk.size() == nb + nq
    assert np.array_equal(sk.counters_u32(), osk.counters().astype(np.uint32))


def test_point_async_inserts_seen_by_later_calls(cuda):
    w, fam = _family(5)
    x, _ = W.host_rows(5, 0, 64)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    ref = ace.AceSketch(fam, ace.CounterWidth.k32)
    for i in range(40):  # per-point inserts (no waits), then a batch call
        sk.insert(x[i])
    sk.insert(x[40:64])   # <= 32 host rows: one point launch
    ref.insert(x)         # general path, one batch
    assert sk.size() == 64 and sk.mean() == ref.mean()
    c = ref.counters_u32()
    assert np.array_equal(sk.counters_u32(), c)
    cfgk = fam.config()
    for t, b in ((0, int(np.argmax(c[:1 << cfgk.k_bits]))), (cfgk.num_tables - 1, 5)):
        assert sk.counter(t, b) == int(c[(t << cfgk.k_bits) + b])
    # scores of single points (point path) equal the batch path's
    s_pt = np.array([sk.score(x[i]).value for i in range(8)])
    assert np.array_equal(s_pt, ref.score_batch(x[:8]))
    # remove after asynchronous inserts: exact inverse
    sk.remove(x[:10])
    ref.remove(x[:10])
    assert np.array_equal(sk.counters_u32(), ref.counters_u32()) and sk.size() == ref.size()


def test_point_detect_stream_contract(cuda):
    _, fam = _family(5)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    q = np.zeros(fam.config().dim)
    with pytest.raises(ace.ContractViolation, match="alpha"):
        ace.detect_stream(sk, q, -1.0)
    with pytest.raises(ace.ContractViolation, match="empty sketch"):
        ace.detect_stream(sk, q, 1.0)
    with pytest.raises(ace.ContractViolation, match="empty sketch"):  # reported before the size check
        ace.detect_stream(sk, np.zeros(3), 1.0)
    sk.insert(q)
    with pytest.raises(ace.ContractViolation):
        ace.detect_stream(sk, np.zeros(3), 1.0)
    est, flag = ace.detect_stream(sk, q, 0.0)
    assert est.value == 1.0 and flag  # score 1 <= mean 1 - 0


def test_cpp_point_bench_matches_oracle(cuda, tmp_path):
    exe = N.LIB_DIR / "ace_point_bench"
    assert exe.exists(), "built by __graft_entry__.build()"
    w, fam = _family(5)
    nb, nq = 4096, 300
    x, _ = W.host_rows(5, 0, nb + nq)
    want_sc, want_fl, _ = _oracle_loop(w, fam, x, nb)
    f = tmp_path / "rows.f32"
    out = tmp_path / "out.bin"
    x.astype(np.float32).tofile(f)
    r = subprocess.run([str(exe), str(w.dim), str(w.k_bits), str(w.num_tables), str(w.w_seed), repr(w.alpha),
                        str(nb), "0", str(nq), str(f), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    raw = out.read_bytes()
    assert np.array_equal(np.frombuffer(raw[:8 * nq], dtype=np.float64), want_sc)
    assert np.array_equal(np.frombuffer(raw[8 * nq:], dtype=np.uint8).astype(bool), want_fl)
    f_ = r.stdout.split()
    assert int(f_[1]) == int(want_fl.sum())
    assert int(f_[5]) == nq + 1  # one point kernel per query, plus the last deferred insert


def test_point_deferred_insert_with_other_calls(cuda):
    """detect_stream(q); insert(q) defers the insert (no launch) into the next
    point kernel; every other call applies it first."""
    torch = cuda
    w, fam = _family(5)
    x, _ = W.host_rows(5, 0, 96)
    xd = torch.from_numpy(x).cuda()  # the reference sketch takes the batch path (device rows)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    ref = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.insert(x[:32])
    ref.insert(xd[:32])
    for i in range(32, 96):
        est, _ = ace.detect_stream(sk, x[i], 0.5)
        assert est.value == ref.score_batch(xd[i:i + 1])[0]
        sk.insert(x[i])  # deferred
        ref.insert(xd[i:i + 1])
        k = i % 6
        if k == 0:
            assert sk.size() == ref.size() and sk.mean() == ref.mean()
        elif k == 1:
            ids = fam.buckets(x[i:i + 1])
            assert sk.counter(3, int(ids[3, 0])) == ref.counter(3, int(ids[3, 0]))
        elif k == 2:  # the same row again: applied after the deferred one
            sk.insert(x[i])
            ref.insert(xd[i:i + 1])
        elif k == 3:
            c = sk.copy()
            assert np.array_equal(c.counters_u32(), ref.counters_u32())
        elif k == 4:
            assert np.array_equal(sk.score_batch(x[:40]), ref.score_batch(xd[:40]))
    assert np.array_equal(sk.counters_u32(), ref.counters_u32())
    assert sk.size() == ref.size() and sk.mean() == ref.mean()
    fl, _, _ = sk.stream_batch(x[:64], 0.5)
    fr, _, _ = ref.stream_batch(xd[:64], 0.5)
    assert np.array_equal(fl, fr)
    assert np.array_equal(sk.counters_u32(), ref.counters_u32())
