"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden digests made by the compiled reference) and the C oracle.

Bar: bit-exact bucket ids, counters, scores and flags; sketch mean and the
detect statistics within 1e-9 relative (the reference's binary64 recurrences
are order-dependent; the device keeps exact integers)."""
import hashlib

import numpy as np
import pytest

from oracle import detect_from_scores
from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace
from paper_1706_06664_b200 import workloads as W

pytestmark = pytest.mark.gpu
REL = 1e-9


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def family(cfg):
    w = W.CONFIGS[cfg]
    return ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables,
                                       seed=w.w_seed))


def close(a, b, rel=REL):
    return abs(a - b) <= rel * max(1.0, abs(b))


@pytest.mark.parametrize("cfg,kernel", [(1, "auto"), (2, "auto"), (3, "auto"), (4, "auto"),
                                        (1, "simt"), (2, "simt"), (3, "simt")])
def test_batch_pipeline_matches_reference(cuda, golden, cfg, kernel):
    e = golden["configs"][str(cfg)]
    x, lab = W.host_rows(cfg, 0, e["n"])
    assert sha(x) == e["x_sha256"]
    fam = family(cfg)
    fam.set_kernel(kernel)
    ids = fam.buckets(x)
    assert sha(ids) == e["ids_sha256"], "bucket ids differ from the reference"
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    xd = cuda.from_numpy(x).cuda()
    rep = sk.build_detect(xd)
    assert rep.stats.rechecked >= rep.stats.flipped
    assert sha(sk.counters_u32()) == e["counters_sha256"]
    assert sk.size() == e["size"]
    assert close(sk.mean(), float.fromhex(e["mean"]))
    assert int(rep.reported) == e["reported"]
    assert sha(np.packbits(rep.flags, bitorder="little")) == e["flags_sha256"]
    assert close(rep.score_mean, float.fromhex(e["det_mean"]))
    assert close(rep.score_stddev, float.fromhex(e["det_sd"]))
    assert close(rep.threshold, float.fromhex(e["det_thr"]))
    # scores bit-exact (S / L with integer S)
    assert sha(sk.score_batch(xd)) == e["scores_sha256"]
    # host-memory input path gives the same counters
    sk2 = ace.AceSketch(fam, ace.CounterWidth.k32)
    rep2 = sk2.build_detect(x)
    assert np.array_equal(sk2.counters_u32(), sk.counters_u32())
    assert np.array_equal(rep2.flags, rep.flags)


@pytest.mark.parametrize("kernel", ["auto", "simt"])
def test_stream_matches_reference(cuda, golden, kernel):
    e = golden["configs"]["5"]
    fam = family(5)
    fam.set_kernel(kernel)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    for b, pb in enumerate(e["per_batch"]):
        x, _ = W.host_rows(5, b * e["batch"], e["batch"])
        assert sha(x) == pb["x_sha256"]
        flags, scores, rep = sk.stream_batch(x, e["alpha"], scores=True)
        assert sha(np.packbits(flags, bitorder="little")) == pb["flags_sha256"], b
        assert int(flags.sum()) == pb["reported"]
        assert sha(scores) == pb["scores_sha256"], b
        assert rep.ambiguous == 0
        assert close(sk.mean(), float.fromhex(pb["mean_after"]))
    assert sha(sk.counters_u32()) == e["counters_sha256"]
    assert sk.size() == e["size"]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("kernel", ["tc", "simt"])
def test_near_tie_stress_exact(cuda, oracle_c, dtype, kernel):
    """Points built to sit within ~1e-9 of many hyperplanes: the fast path's
    margin routes them to the FP64 recheck and every id still matches."""
    d, k, l, seed = 96, 15, 50, 7
    fam = ace.SrpFamily(ace.SrpConfig(dim=d, k_bits=k, num_tables=l, seed=seed))
    fam.set_kernel(kernel)
    w = fam.directions
    rng = np.random.default_rng(3)
    n = 4096
    x = rng.standard_normal((n, d))
    r = rng.integers(0, k * l, n)
    wr = w[r]
    eps = rng.choice([0.0, 1e-12, -1e-12, 1e-9, -1e-9, 1e-7], n)
    x = x - ((x * wr).sum(1) / (wr * wr).sum(1))[:, None] * wr + eps[:, None] * wr
    x = x.astype(dtype)
    st = N.AceHashStats()
    ids = fam.buckets(x, stats=st)
    ref_ids, near = oracle_c.buckets(w, x, k, l, rel_eps=1e-6)
    assert np.array_equal(ids, ref_ids)
    assert st.rechecked >= near  # every sub-1e-6 projection went to the recheck
    assert st.near_ties == near  # the BASELINE near-tie measure, counted as the oracle counts it


@pytest.mark.parametrize("kernel", ["tc", "simt"])
def test_edge_cases(cuda, oracle_c, kernel):
    d, k, l = 10, 4, 6
    fam = ace.SrpFamily(ace.SrpConfig(dim=d, k_bits=k, num_tables=l, seed=11))
    fam.set_kernel(kernel)
    w = fam.directions
    x = np.zeros((77, d), dtype=np.float32)          # zero rows -> all-ones buckets
    x[1] = np.nan                                     # NaN -> p NaN -> bit 0
    x[2, 0] = np.inf
    x[3] = 1e-38                                      # tiny
    x[4] = 3e37                                       # huge
    x[5:] = np.random.default_rng(0).standard_normal((72, d)).astype(np.float32)
    ids = fam.buckets(x)
    ref, _ = oracle_c.buckets(w, x, k, l)
    assert np.array_equal(ids, ref)
    assert (ids[:, 0] == (1 << k) - 1).all()
    # ragged n and strided rows (ld > dim) through torch views
    xt = cuda.from_numpy(np.random.default_rng(1).standard_normal((1001, 2 * d)).astype(np.float32)).cuda()
    view = xt[:, :d]
    ids_v = fam.buckets(view)
    ref_v, _ = oracle_c.buckets(w, view.cpu().numpy(), k, l)
    assert np.array_equal(ids_v, ref_v)
    # empty batch is a no-op; empty detect is a contract violation
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.insert(np.zeros((0, d), dtype=np.float32))
    assert sk.size() == 0
    with pytest.raises(ace.ContractViolation):
        ace.detect_batch(sk, np.zeros((0, d), dtype=np.float32))
    with pytest.raises(ace.ContractViolation):
        sk.insert(np.zeros((3, d + 1), dtype=np.float32))
    with pytest.raises(ace.ContractViolation):
        sk.stream_batch(np.zeros((3, d), dtype=np.float32), -1.0)


@pytest.mark.parametrize("k", [1, 8, 16, 18, 30])
@pytest.mark.parametrize("kernel", ["tc", "simt"])
def test_k_range_packing(cuda, oracle_c, k, kernel):
    d = 12
    l = 3 if k == 30 else 9
    fam = ace.SrpFamily(ace.SrpConfig(dim=d, k_bits=k, num_tables=l, seed=k))
    fam.set_kernel(kernel)
    x = np.random.default_rng(k).standard_normal((513, d)).astype(np.float32)
    ids = fam.buckets(x)
    ref, _ = oracle_c.buckets(fam.directions, x, k, l)
    assert np.array_equal(ids, ref)
    assert int(ids.max()) < (1 << k)


def test_k16_saturation_and_remove(cuda, oracle_c, reference):
    d, k, l, seed = 3, 2, 2, 4
    fam = ace.SrpFamily(ace.SrpConfig(dim=d, k_bits=k, num_tables=l, seed=seed))
    x = np.tile(np.array([[0.5, -1.0, 2.0]], dtype=np.float32), (70000, 1))
    sk = ace.AceSketch(fam, ace.CounterWidth.k16)
    sk.insert(x[:30000])
    sk.insert(x[30000:])
    rs = reference.sketch(seed, d, k, l, 16)
    rs.insert(x)
    assert sk.saturated() and rs.saturated()
    assert np.array_equal(sk.counters_flat(), rs.counters())
    assert close(sk.mean(), rs.mean())


def test_remove_and_inconsistent_delete(cuda, reference):
    d, k, l, seed = 8, 6, 10, 3
    fam = ace.SrpFamily(ace.SrpConfig(dim=d, k_bits=k, num_tables=l, seed=seed))
    rng = np.random.default_rng(2)
    x = rng.standard_normal((500, d)).astype(np.float32)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.insert(x)
    sk.remove(x[:200])
    rs = reference.sketch(seed, d, k, l, 32)
    rs.insert(x)
    assert rs.remove(x[:200]) == 0
    assert np.array_equal(sk.counters_flat(), rs.counters())
    assert sk.size() == rs.size() == 300
    assert close(sk.mean(), rs.mean())
    before = sk.counters_flat()
    never = rng.standard_normal((1, d)).astype(np.float32) * 100
    sk2 = ace.AceSketch(fam, ace.CounterWidth.k32)
    with pytest.raises(ace.InconsistentDelete):
        sk2.remove(never)
    sk.remove(x[200:])
    assert sk.size() == 0 and sk.mean() == 0.0
    assert int(sk.counters_flat().sum()) == 0
    assert before.sum() == 300 * l


def test_restore_clone_roundtrip(cuda):
    w = W.CONFIGS[1]
    fam = family(1)
    x, _ = W.host_rows(1, 0, 5000)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.insert(x)
    c = sk.copy()
    r = ace.AceSketch.restore(fam, ace.CounterWidth.k32, sk.counters_flat(), sk.size(), sk.mean(), False)
    q = x[:100]
    assert np.array_equal(sk.score_batch(q), r.score_batch(q))
    assert np.array_equal(sk.score_batch(q), c.score_batch(q))
    c.insert(x[:10])
    assert c.size() == sk.size() + 10
    assert close(r.mean(), sk.mean())
    with pytest.raises(ace.ContractViolation):
        ace.AceSketch.restore(fam, ace.CounterWidth.k32, np.zeros(5, np.uint64), 0, 0.0, False)
    assert w.dim == 40


@pytest.mark.parametrize("d", [1, 3, 63, 64, 65, 127, 129, 192, 255, 256, 257, 300, 1000, 4096])
def test_tc_dims_and_overflow_path(cuda, oracle_c, d):
    """Every K-chunk count of the tcgen05 kernel (d > 256: the K-streamed
    kernel); list-overflow rows (NaN rows
    force every projection onto the exact path) still give exact ids."""
    k, l = 15, 20
    fam = ace.SrpFamily(ace.SrpConfig(dim=d, k_bits=k, num_tables=l, seed=d))
    assert fam.kernel() == "tc"
    rng = np.random.default_rng(d)
    x = rng.standard_normal((2000, d)).astype(np.float32)
    x[::50] = np.nan
    x[7::61] = 0.0
    ids = fam.buckets(x)
    ref, _ = oracle_c.buckets(fam.directions, x, k, l)
    assert np.array_equal(ids, ref)
    assert (ids[:, 0] == 0).all()  # NaN -> all bits 0


def test_stream_run_matches_reference(cuda, golden):
    """The queued multi-batch driver gives the golden per-batch flags."""
    e = golden["configs"]["5"]
    fam = family(5)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    nb = len(e["per_batch"])
    x, _ = W.host_rows(5, 0, nb * e["batch"])
    flags, lat, rep = sk.stream_run(cuda.from_numpy(x).cuda(), e["batch"], e["alpha"])
    assert len(lat) == nb and (lat > 0).all()
    for b, pb in enumerate(e["per_batch"]):
        fb = flags[b * e["batch"]:(b + 1) * e["batch"]]
        assert sha(np.packbits(fb, bitorder="little")) == pb["flags_sha256"], b
    assert sha(sk.counters_u32()) == e["counters_sha256"]
    assert rep.ambiguous == 0
    with pytest.raises(ace.ContractViolation):
        sk.stream_run(x[:100], 33, 1.0)


@pytest.mark.parametrize("cfg", [1, 2])
def test_repeated_calls_replay_graph(cuda, golden, cfg):
    """build_detect repeated on the same buffers: eager, then captured into a
    CUDA graph, then replayed.  Every repetition must give the reference's
    counters and flags; a call with other arguments must not replay."""
    e = golden["configs"][str(cfg)]
    x, _ = W.host_rows(cfg, 0, e["n"])
    fam = family(cfg)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    xd = cuda.from_numpy(x).cuda()
    flags = cuda.empty((e["n"] + 31) // 32, dtype=cuda.int32, device="cuda")
    for rep_i in range(4):
        sk.reset()
        rep = sk.build_detect(xd, flags_out=flags)
        assert sha(sk.counters_u32()) == e["counters_sha256"], rep_i
        assert int(rep.reported) == e["reported"], rep_i
        bits = flags.cpu().numpy().view(np.uint32)
        fl = np.unpackbits(bits.view(np.uint8), bitorder="little")[: e["n"]].astype(bool)
        assert sha(np.packbits(fl, bitorder="little")) == e["flags_sha256"], rep_i
    # detect_batch (no build) on a prefix: different key, no stale replay
    half = e["n"] // 2
    rep_a = ace.detect_batch(sk, xd[:half])
    rep_b = ace.detect_batch(sk, xd[:half])
    rep_c = ace.detect_batch(sk, xd[:half])
    assert int(rep_a.reported) == int(rep_b.reported) == int(rep_c.reported)
    assert np.array_equal(rep_a.flags, rep_c.flags)
    # pinned host input through the same graph machinery
    xp = cuda.from_numpy(x).pin_memory()
    for _ in range(3):
        sk.reset()
        sk.build_detect(xp)
        assert sha(sk.counters_u32()) == e["counters_sha256"]


def test_fused_gather_path_all_shapes(cuda, golden):
    """The fused count-and-gather pass forced on (ACE_OPT_DEFER_INSERT = 1)
    for configs 1, 2 and the K = 16 prefix of 3 (packed u16 bins), and forced
    off (-1): reference counters and flags either way."""
    torch = cuda
    for cfg in (1, 2, 3):
        e = golden["configs"][str(cfg)]
        w = W.CONFIGS[cfg]
        x, _ = W.host_rows(cfg, 0, e["n"])
        fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
        for mode in (1, -1):
            sk = ace.AceSketch(fam, ace.CounterWidth.k32)
            sk.set_option(N.ACE_OPT_DEFER_INSERT, mode)
            rep = sk.build_detect(torch.from_numpy(x).cuda())
            assert sha(sk.counters_u32()) == e["counters_sha256"], (cfg, mode)
            assert sha(np.packbits(rep.flags, bitorder="little")) == e["flags_sha256"], (cfg, mode)
            assert rep.reported == e["reported"], (cfg, mode)


@pytest.mark.parametrize("chunks", [1, 3, 16])
def test_chunked_h2d_pipeline(cuda, golden, chunks):
    """Pinned host rows of a large batch are copied in chunks on a copy
    stream and hashed as each chunk lands (ACE_OPT_H2D_CHUNKS).  Uneven chunk
    counts on configs 1 and 2, both counter widths, repeated calls (graph
    replay): reference counters, flags and report."""
    torch = cuda
    for cfg in (1, 2):
        e = golden["configs"][str(cfg)]
        w = W.CONFIGS[cfg]
        x, _ = W.host_rows(cfg, 0, e["n"])
        xp = torch.from_numpy(x).pin_memory()
        fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
        for width in (ace.CounterWidth.k32, ace.CounterWidth.k16):
            sk = ace.AceSketch(fam, width)
            sk.set_option(N.ACE_OPT_H2D_CHUNKS, chunks)
            for _ in range(2):
                sk.reset()
                rep = sk.build_detect(xp.numpy())
            assert sha(sk.counters_u32()) == e["counters_sha256"], (cfg, width)
            assert sha(np.packbits(rep.flags, bitorder="little")) == e["flags_sha256"], (cfg, width)
            assert rep.reported == e["reported"], (cfg, width)


def test_hist16_hot_bins_wrap(cuda):
    """K = 16 deferred insert counts 2^16 bins packed two per shared word
    (count_range16): bins hit 65536+ times within one block's id range wrap
    their u16 half and spill to the global counter, a wrapped low half's carry
    into its neighbour is undone.  Two points whose table-0 buckets differ only
    in the last bit (the two halves of one word) alternate over 6M rows (24M
    ids: ~81k hits per bin per block range); the other tables get one or two
    hot bins.  Counters, mean and scores equal the exact counts."""
    torch = cuda
    fam = ace.SrpFamily(ace.SrpConfig(dim=2, k_bits=16, num_tables=4, seed=7))
    w = np.asarray(fam.direction(0, 15), dtype=np.float64)
    perp = np.array([-w[1], w[0]]) / np.linalg.norm(w)
    u = w / np.linalg.norm(w)
    pair = None
    for delta in (1e-2, 1e-3, 1e-4, 1e-5):
        pts = np.stack([perp + delta * u, perp - delta * u]).astype(np.float32)
        b = fam.buckets(pts.astype(np.float64))
        if int(b[0, 0]) ^ int(b[0, 1]) == 1:
            pair = pts
            break
    assert pair is not None, "no point pair straddling only the last hyperplane of table 0"
    n = 6_000_000
    x = np.empty((n, 2), dtype=np.float32)
    x[0::2] = pair[0]
    x[1::2] = pair[1]
    ids = fam.buckets(pair.astype(np.float64))  # (L, 2)
    L, K = 4, 16
    expect = np.zeros((L, 1 << K), dtype=np.uint64)
    for t in range(L):
        expect[t, ids[t, 0]] += n // 2
        expect[t, ids[t, 1]] += n // 2
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    rep = sk.build_detect(torch.from_numpy(x).cuda())
    got = sk.counters_u32().reshape(L, 1 << K).astype(np.uint64)
    assert np.array_equal(got, expect)
    sq = int((expect.astype(object) ** 2).sum())
    assert sk.size() == n
    assert abs(sk.mean() - sq / (n * L)) <= 1e-12 * sq / (n * L)
    s0 = int(sum(expect[t, ids[t, 0]] for t in range(L)))
    s1 = int(sum(expect[t, ids[t, 1]] for t in range(L)))
    assert abs(rep.score_mean - (s0 + s1) / (2 * L)) <= 1e-9 * max(s0, s1)


@pytest.mark.parametrize("gather", [False, True])
def test_tied_scores_replay(cuda, oracle_c, gather):
    """Every row's score sits exactly on the exact threshold (two points, m
    copies each: all scores equal, sd = 0), so the ambiguity band holds every
    row and the detect tail's last block replays the reference's sequential
    binary64 statistics (detect.cpp:44-60).  The flags must be the
    reference's, whichever way its rounding falls; the run with N*L >= 16M
    takes the deferred-insert (gather) path of the tail."""
    torch = cuda
    L = 50 if gather else 4
    fam = ace.SrpFamily(ace.SrpConfig(dim=8, k_bits=15, num_tables=L, seed=11))
    rng = np.random.default_rng(5)
    pts = rng.standard_normal((2, 8)).astype(np.float32)
    m = 200_000 if gather else 3_001
    x = np.repeat(pts, m, axis=0)
    rng.shuffle(x, axis=0)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    rep = sk.build_detect(torch.from_numpy(x).cuda())
    assert rep.ambiguous == 2 * m and rep.replayed
    ids = fam.buckets(x.astype(np.float64))                      # (L, n)
    cnt = sk.counters_u32().reshape(L, -1)
    S = cnt[np.arange(L)[:, None], ids].astype(np.int64).sum(axis=0)
    _, _, thr, flags = detect_from_scores(oracle_c, S / float(L))
    assert np.array_equal(rep.flags, flags)
    assert rep.reported == int(flags.sum())
    assert rep.threshold == thr


@pytest.mark.gpu
@pytest.mark.parametrize("pipe", [0, 64, 90])
def test_stream_run_pipelined_matches_oracle(cuda, pipe):
    """ace_sketch_stream_run with ACE_OPT_STREAM_PIPE (the next group's
    projection beside a one-CTA-per-table stream kernel) against the oracle's
    stream order: clustered rows, then whole batches of one repeated row (a
    bucket taking all 65,536 rows of a batch, the u16 histogram's wrap), a
    ragged last batch."""
    from oracle import Oracle
    w = W.CONFIGS[5]
    batch, nb = 65536, 7
    n = batch * nb - 4001
    x, _ = W.host_rows(5, 0, n)
    x[2 * batch:4 * batch] = x[17]          # two batches of one point
    x[5 * batch:5 * batch + 300] = x[17]
    fam = family(5)
    o = Oracle()
    ids, _ = o.buckets(fam.directions, x, w.k_bits, w.num_tables)
    osk = o.sketch(w.k_bits, w.num_tables, 32)
    want = np.zeros(n, dtype=bool)
    for b in range(nb):
        r0, r1 = b * batch, min(n, (b + 1) * batch)
        want[r0:r1], _ = osk.stream_ids(ids[:, r0:r1], w.alpha)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.set_option(N.ACE_OPT_STREAM_GROUP, 2)
    sk.set_option(N.ACE_OPT_STREAM_PIPE, pipe)
    xd = cuda.from_numpy(x).cuda()
    for rep_i in range(3):  # the third call replays the driver's CUDA graph
        sk.reset()
        flags, lat, rep = sk.stream_run(xd, batch, w.alpha, latencies=(rep_i == 0))
        assert np.array_equal(flags, want), rep_i
        assert np.array_equal(sk.counters_flat(), osk.counters())
        assert sk.size() == n
        assert rep.reported == int(want.sum())


@pytest.mark.gpu
@pytest.mark.parametrize("d,k,l,batch,group,pipe", [
    (24, 8, 10, 1024, 4, 88),     # small tables, many scoring CTAs
    (64, 15, 50, 4096, 3, 64),    # cfg-5 shape, short batches, group not dividing the batch count
    (40, 12, 64, 8192, 2, 80),    # 64 tables + 4 + 80 = 148 SMs: the tightest split
    (33, 4, 7, 256, 8, 100),      # K = 4 (the smallest), batches of one scoring chunk
    (64, 15, 50, 4096, 3, 0),     # the pair kernel on the same stream
])
def test_stream_run_shapes_match_oracle(cuda, d, k, l, batch, group, pipe):
    """The group stream kernels (pair and one CTA per table, pipelined with
    the projection) on other shapes than config 5, device rows and pinned host
    rows, against the oracle's stream order."""
    from oracle import Oracle
    torch = cuda
    nb = 11
    n = batch * nb - 96
    rng = np.random.default_rng(1000 * k + l)
    centres = rng.standard_normal((5, d)) * 3.0
    x = (centres[rng.integers(0, 5, n)] + 0.3 * rng.standard_normal((n, d))).astype(np.float32)
    x[rng.integers(0, n, n // 50)] = (rng.standard_normal((n // 50, d)) * 8.0).astype(np.float32)
    fam = ace.SrpFamily(ace.SrpConfig(dim=d, k_bits=k, num_tables=l, seed=7))
    o = Oracle()
    ids, _ = o.buckets(fam.directions, x, k, l)
    osk = o.sketch(k, l, 32)
    want = np.zeros(n, dtype=bool)
    alpha = 0.5
    for b in range(nb):
        r0, r1 = b * batch, min(n, (b + 1) * batch)
        want[r0:r1], _ = osk.stream_ids(ids[:, r0:r1], alpha)
    for src in ("device", "pinned"):
        sk = ace.AceSketch(fam, ace.CounterWidth.k32)
        sk.set_option(N.ACE_OPT_STREAM_GROUP, group)
        sk.set_option(N.ACE_OPT_STREAM_PIPE, pipe)
        xin = torch.from_numpy(x).cuda() if src == "device" else torch.from_numpy(x).pin_memory().numpy()
        for rep_i in range(3):
            sk.reset()
            flags, _, rep = sk.stream_run(xin, batch, alpha, latencies=(rep_i == 1))
            assert np.array_equal(flags, want), (src, rep_i)
            assert np.array_equal(sk.counters_flat(), osk.counters()), (src, rep_i)
            assert sk.size() == n and rep.reported == int(want.sum())
