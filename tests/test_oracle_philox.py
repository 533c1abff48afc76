"""P1: the oracle's Philox4x32-10 against the Random123 known-answer vectors.

Pins: tests/golden/philox4x32_10_kat.txt (Salmon et al., SC'11 KATs) — the one
external reference for the RNG both sides implement independently (R#20).
"""
import os

import numpy as np

from oracle import philox4x32_10, sample_actions

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kats():
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        w = [int(x, 16) for x in line.split()]
        yield w[0:4], w[4:6], w[6:10]


def test_philox_known_answers():
    n = 0
    for ctr, key, want in _kats():
        got = philox4x32_10(ctr, key)
        assert [int(x) for x in got] == want, (ctr, key)
        n += 1
    assert n == 3


def test_philox_counter_sensitivity():
    # every counter word and key word changes every output word (avalanche)
    base = philox4x32_10([1, 2, 3, 4], [5, 6])
    for i in range(4):
        c = [1, 2, 3, 4]
        c[i] ^= 1
        assert np.all(philox4x32_10(c, [5, 6]) != base)
    for i in range(2):
        k = [5, 6]
        k[i] ^= 1
        assert np.all(philox4x32_10([1, 2, 3, 4], k) != base)


def test_action_stream_is_uniform_and_shard_invariant():
    # action stream: keyed by the GLOBAL env index, so a shard
    # [begin, begin+n) reproduces the corresponding columns of the full stream.
    full = sample_actions(1, 0, 64, 0, 50, 7)
    part = sample_actions(1, 16, 32, 0, 50, 7)
    assert np.array_equal(full[:, 16:48], part)
    later = sample_actions(1, 0, 64, 10, 40, 7)
    assert np.array_equal(full[10:], later)
    big = sample_actions(1, 0, 4096, 0, 16, 7)
    counts = np.bincount(big.reshape(-1), minlength=7)
    assert counts.max() - counts.min() < 0.05 * counts.mean()
    assert big.max() == 6
