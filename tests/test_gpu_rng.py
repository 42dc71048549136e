"""GPU parity of the device RNG / libm / slowdown against numpy + glibc
known answers (tests/golden/rng_golden.npz), bit-exact."""
import numpy as np
import pytest

from tests import _golden

pytestmark = pytest.mark.gpu


def test_noise_draws_bit_exact():
    from paper_2512_18725_b200 import engine

    R = _golden.load("rng_golden.npz")
    keys = R["noise_keys"].astype(np.int64)
    for sig, ref, n in ((0.05, R["noise_sigma005"], len(keys)), (0.02, R["noise_sigma002"], 400)):
        seeds = keys[:n, 0]
        got = np.zeros(n)
        for s in np.unique(seeds):
            sel = seeds == s
            got[sel] = engine.noise_draws(int(s), sig, keys[:n][sel, 1], keys[:n][sel, 2])
        np.testing.assert_array_equal(got, ref)


def test_rng_streams_bit_exact():
    import oracle as O
    from paper_2512_18725_b200 import engine

    R = _golden.load("rng_golden.npz")
    np.testing.assert_array_equal(engine.rng_stream(O.int_words(*R["uniform_seed"]), 5000, uniform=True), R["uniform"])
    z = engine.rng_stream(O.int_words(*R["normal_seed"]), len(R["normal"]))
    np.testing.assert_array_equal(z, R["normal"])  # includes ziggurat wedge + tail draws


def test_slowdown_hand_example_and_monotone():
    import paper_2512_18725_b200 as p

    noiseless = p.InterferenceOracle(noise_sigma=0.0)
    assert p.oracle_slowdown((0.9, 0.9, 0.9), (0, 0, 0), noiseless) == 1.0
    assert abs(p.oracle_slowdown((0.6, 0.5, 0.4), (0.6, 0.5, 0.4), noiseless) - 1.2) < 1e-12
    with pytest.raises(ValueError):
        p.oracle_slowdown((-0.1, 0.5, 0.5), (0, 0, 0), noiseless)
    o = p.InterferenceOracle(noise_sigma=0.1, seed=5)
    assert o.noise_draw(3, 1) == o.noise_draw(3, 1) != o.noise_draw(3, 2)
