"""P4: the success reward of Eq. (1), read per R#1/R#2.

Pins: tests/golden/p4_reward_bits.json (SURVEY §8c-10 P4 bit patterns, and
S:306's 0.82 at t=19, T=100), plus a bound that does not depend on how the
oracle evaluates it: for every step count of every headline horizon T the
binary32 reward lies within one binary32 ulp of the exact rational
1 - 9*sc/(10*T), is strictly decreasing in sc, and ends at RN32(0.1).
"""
import json
import os
import struct
from fractions import Fraction

import numpy as np

from oracle import success_reward

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bits(x: float) -> int:
    return struct.unpack("<I", struct.pack("<f", x))[0]


def test_p4_golden_bit_patterns():
    g = json.load(open(os.path.join(GOLD, "p4_reward_bits.json")))
    for c in g["cases"]:
        r = success_reward(0, c["sc"], c["T"])
        assert bits(r) == int(c["bits"], 16), c
        assert abs(r - c["value"]) < 1e-7


def test_markovian_mode_is_one():
    # "1 at task completion" in NAVIX's Markovian default
    for T in (100, 256, 640):
        for sc in (1, T // 2, T):
            assert success_reward(1, sc, T) == 1.0


def test_exact_rational_bound_all_step_counts():
    for T in (100, 256, 640, 196, 270):
        prev = None
        for sc in range(1, T + 1):
            r = success_reward(0, sc, T)
            exact = Fraction(1) - Fraction(9 * sc, 10 * T)
            ulp = np.spacing(np.float32(r))
            assert abs(Fraction(r) - exact) <= Fraction(float(ulp)), (sc, T)
            if prev is not None:
                assert r < prev
            prev = r
        assert bits(r) == bits(float(np.float32(0.1)))
