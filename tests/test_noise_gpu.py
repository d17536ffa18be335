"""Noisy SRP variant (srp.cpp:93-104, 126-129, sketch.cpp:76-79).

Every noisy bit is RN(p + noise_scale * N(0,1)) with the normal drawn from the
family's aux stream at tick = that family's call counter.  The ticks run in
point / table / bit order, so a sequence of calls on our family must give the
same ids as the same sequence on the compiled reference, bit for bit, once
both aux streams are pinned with reset_noise_stream (or both start from the
seed-derived default).  Sketches copy the family, counter included."""
import numpy as np
import pytest

from paper_1706_06664_b200 import ace

pytestmark = pytest.mark.gpu


def _fam(d, k, l, seed, noise):
    return ace.SrpFamily(ace.SrpConfig(dim=d, k_bits=k, num_tables=l, seed=seed, noise_scale=noise))


def _pts(n, d, seed, dtype=np.float64):
    return np.random.default_rng(seed).standard_normal((n, d)).astype(dtype)


@pytest.mark.parametrize("d,k,l,noise", [(6, 4, 2, 1.5), (16, 8, 10, 0.25), (33, 15, 7, 3.0), (128, 20, 3, 0.01)])
@pytest.mark.parametrize("aux", [None, 4242])
def test_noisy_buckets_match_reference(cuda, reference, d, k, l, noise, aux):
    x = _pts(57, d, d + k)
    f = _fam(d, k, l, 11, noise)
    if aux is not None:
        f.reset_noise_stream(aux)
    got = f.buckets(x)
    want = reference.noisy_calls(11, d, k, l, noise, x, 0, l, aux=aux)
    assert np.array_equal(got, want)
    # the counter moved on: a second batch continues the same stream
    got2 = f.buckets(x)
    f2 = _fam(d, k, l, 11, noise)
    if aux is not None:
        f2.reset_noise_stream(aux)
    both = f2.buckets(np.concatenate([x, x]))
    assert np.array_equal(both[:, 57:], got2)


def test_noisy_single_calls_tick_order(cuda, reference):
    """bucket(t) takes K ticks, bit(t, b) one; a mixed call sequence agrees."""
    d, k, l, noise = 9, 6, 5, 0.8
    x = _pts(12, d, 5)
    f = _fam(d, k, l, 3, noise)
    f.reset_noise_stream(7)
    ops, got = [], []
    for i in range(12):
        for t, b in ((1, 2), (4, -1), (3, 5), (0, -1)):
            ops.append((i, t, b))
            got.append(f.bit(t, b, x[i]) if b >= 0 else f.bucket(t, x[i]))
    want = reference.noisy_sequence(3, d, k, l, noise, 7, x, ops)
    assert np.array_equal(np.array(got, dtype=np.uint32), want)
    # batch calls continue the stream where the single calls left it
    got_batch = f.buckets(x[:4])
    want_all = reference.noisy_sequence(3, d, k, l, noise, 7, x, ops + [(i, t, -1) for i in range(4)
                                                                       for t in range(l)])
    assert np.array_equal(got_batch.T.reshape(-1), want_all[len(ops):])


def test_noisy_sketch_counters_scores_detect(cuda, reference):
    d, k, l, noise = 12, 7, 9, 0.7
    x = _pts(300, d, 1, np.float32)
    q = _pts(80, d, 2, np.float32)
    fam = _fam(d, k, l, 21, noise)
    fam.reset_noise_stream(1234)
    sk = ace.AceSketch(fam, ace.CounterWidth.k32)
    sk.insert(x)
    ref = reference.noisy_sketch(21, d, k, l, noise, width=32, aux=1234)
    ref.insert(x)
    assert np.array_equal(sk.counters_u32(), ref.counters().astype(np.uint32).reshape(sk.counters_u32().shape))
    # the mean is T/(nL) rounded once; the reference's recurrence drifts by a
    # few ulps, held to 1e-9 as for the exact path
    assert sk.size() == ref.size() and abs(sk.mean() - ref.mean()) <= 1e-9 * ref.mean()
    assert np.array_equal(sk.score_batch(q), ref.score(q))
    # detect_batch with one thread: scores in row order, sequential statistics
    rep = ace.detect_batch(sk, x, threads=1, want_scores=True)
    rr = ref.detect_batch(x, threads=1)
    assert (rep.score_mean, rep.score_stddev, rep.threshold, rep.reported) == \
        (rr["mean"], rr["sd"], rr["thr"], rr["reported"])
    # the reference report has no per-row flags (its driver re-scores, which
    # draws fresh noise): check the scores on a twin sketch in the same state
    twin = reference.noisy_sketch(21, d, k, l, noise, width=32, aux=1234)
    twin.insert(x)
    twin.score(q)
    assert np.array_equal(rep.scores, twin.score(x))
    assert np.array_equal(rep.flags, rep.scores < rep.threshold)
    with pytest.raises(ace.UnsupportedOperation):
        sk.remove(x[:1])
