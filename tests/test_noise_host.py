"""Host side of the noisy variant (no GPU): the aux stream's seed, tick
counter, reset and copy semantics (srp.cpp:34, 51-64, 93-104, 126-129)."""
import numpy as np

from paper_1706_06664_b200 import ace


def _fam(noise=0.5, seed=5):
    return ace.SrpFamily(ace.SrpConfig(dim=4, k_bits=3, num_tables=2, seed=seed, noise_scale=noise))


def test_default_aux_seed_and_ticks():
    f = _fam()
    assert f._noise_seed == ace.mix_seed(5, 0x6e6f697365)
    a = f.draw_noise(10)
    assert f._noise_ctr == 10
    f2 = _fam()
    b = np.concatenate([f2.draw_noise(3), f2.draw_noise(7)])
    assert np.array_equal(a, b)  # tick-indexed: chunking does not matter
    assert np.all(np.isfinite(a)) and a.std() > 0


def test_reset_and_scale():
    f = _fam(noise=2.0)
    f.reset_noise_stream(99)
    a = f.draw_noise(6)
    f.reset_noise_stream(99)
    assert np.array_equal(f.draw_noise(6), a)
    g = _fam(noise=1.0)
    g.reset_noise_stream(99)
    assert np.array_equal(2.0 * g.draw_noise(6), a)  # sigma * N(0,1), exact for a power of two


def test_copy_carries_counter():
    f = _fam()
    f.draw_noise(4)
    c = f._copy()
    assert c._noise_ctr == 4
    x = c.draw_noise(2)
    assert f._noise_ctr == 4  # independent counters after the copy
    assert np.array_equal(f.draw_noise(2), x)
