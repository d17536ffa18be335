"""ACE1 sketch files (reference io.cpp:184-244, tests test_io.cpp:100-164).

CPU: the bytes this framework writes for a sketch state are the bytes the
compiled reference's save_sketch writes for that state, and the loader's
error behaviour matches (bad magic, truncation, bad width -> DataError).
GPU: a device sketch saved here loads in the reference (counters, n, mean,
saturation equal) and a reference file restores here with the same counters,
the same mean bit for bit and the same scores."""
import numpy as np
import pytest

from paper_1706_06664_b200 import ace
from paper_1706_06664_b200.sketch_io import ace1_bytes, parse_ace1


def _ref_sketch(reference, seed, dim, k, l, width, n, data_seed):
    x = np.random.default_rng(data_seed).standard_normal((n, dim)).astype(np.float32)
    r = reference.sketch(seed, dim, k, l, width)
    r.insert(x)
    return r, x


@pytest.mark.parametrize("width", [16, 32])
def test_bytes_match_reference_writer(reference, tmp_path, width):
    r, _ = _ref_sketch(reference, 99, 6, 10, 20, width, 120, 17)
    path = tmp_path / "ref.ace"
    r.save(path)
    ref_bytes = path.read_bytes()
    ours = ace1_bytes(6, 10, 20, width, 99, 0.0, r.size(), r.mean(), r.saturated(), r.counters())
    assert ours == ref_bytes
    h, counters = parse_ace1(ref_bytes)
    assert (h["cfg"].dim, h["cfg"].k_bits, h["cfg"].num_tables, h["cfg"].seed) == (6, 10, 20, 99)
    assert h["width"] == width and h["n"] == 120 and h["mean"] == r.mean()
    assert np.array_equal(counters, r.counters())


def test_saturated_k16_flag_round_trips(reference, tmp_path):
    # 70,000 identical rows saturate a 16-bit counter (sticky flag, capped count)
    x = np.ones((70_000, 3), dtype=np.float32)
    r = reference.sketch(2, 3, 4, 2, 16)
    r.insert(x)
    assert r.saturated()
    path = tmp_path / "sat.ace"
    r.save(path)
    h, counters = parse_ace1(path.read_bytes())
    assert h["saturated"] and counters.max() == 65535
    assert ace1_bytes(3, 4, 2, 16, 2, 0.0, r.size(), r.mean(), True, r.counters()) == path.read_bytes()


def test_loader_errors_match_reference(reference, tmp_path):
    bad = tmp_path / "bad.ace"
    bad.write_bytes(b"NOPEnotasketch")
    with pytest.raises(ace.DataError):
        parse_ace1(bad.read_bytes())
    with pytest.raises(ValueError):
        reference.load_sketch(bad)
    r, _ = _ref_sketch(reference, 2, 3, 8, 4, 16, 20, 29)
    whole = tmp_path / "whole.ace"
    r.save(whole)
    data = whole.read_bytes()
    trunc = tmp_path / "trunc.ace"
    trunc.write_bytes(data[:-7])
    with pytest.raises(ace.DataError):
        parse_ace1(trunc.read_bytes())
    with pytest.raises(ValueError):
        reference.load_sketch(trunc)
    badw = tmp_path / "badw.ace"
    badw.write_bytes(data[:16] + bytes([8]) + data[17:])  # width field (bytes 16..19)
    with pytest.raises(ace.DataError):
        parse_ace1(badw.read_bytes())
    with pytest.raises(ValueError):
        reference.load_sketch(badw)


@pytest.mark.gpu
@pytest.mark.parametrize("width", [ace.CounterWidth.k16, ace.CounterWidth.k32])
def test_device_sketch_files_interchange_with_reference(cuda, reference, tmp_path, width):
    dim, k, l, seed, n = 40, 15, 50, 1, 5000
    x = np.random.default_rng(5).standard_normal((n, dim)).astype(np.float32)
    fam = ace.SrpFamily(ace.SrpConfig(dim=dim, k_bits=k, num_tables=l, seed=seed))
    sk = ace.AceSketch(fam, width)
    sk.insert(x)
    # ours -> reference
    p1 = tmp_path / "ours.ace"
    ace.save_sketch(sk, p1)
    r = reference.load_sketch(p1)
    assert np.array_equal(r.counters(), sk.counters_flat())
    assert r.size() == sk.size() and r.mean() == sk.mean() and r.saturated() == sk.saturated()
    # reference -> ours: counters, mean bit for bit, scores
    w_bits = 16 if width == ace.CounterWidth.k16 else 32
    rr = reference.sketch(seed, dim, k, l, w_bits)
    rr.insert(x[:3000])
    p2 = tmp_path / "ref.ace"
    rr.save(p2)
    loaded = ace.load_sketch(p2)
    assert np.array_equal(loaded.counters_flat(), rr.counters())
    assert loaded.size() == rr.size() and loaded.mean() == rr.mean()
    q = x[3000:3500]
    assert np.array_equal(loaded.score_batch(q), rr.score(q))
    # the pinned mean is released by the next update
    loaded.insert(x[3000:3001])
    rr.insert(x[3000:3001])
    assert abs(loaded.mean() - rr.mean()) <= 1e-9 * rr.mean()
