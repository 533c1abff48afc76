"""P3: brute force over every short action sequence on Empty-5x5.

Empty-5x5 has no RNG and nothing to pick up, drop or toggle, so the state is
(x, y, dir) over 36 values.  A DP written here (independent of the oracle's
object-grid simulation) counts, for each L, the length-L sequences over the
7 actions whose FIRST goal arrival is at step L; these must equal the counts
in tests/golden/p3_empty5_first_goal_counts.json.  The
oracle then runs every sequence of length L_MAX as one lane each: the number
of lanes terminating at step L must be count(L) * 7^(L_MAX - L), each with
reward RN32(1 - 0.9*L/100), and no lane may terminate twice (>= 5 steps to
reach the goal again after the autoreset).
"""
import json
import os

import numpy as np

from oracle import OracleEnv, success_reward

GOLD = os.path.join(os.path.dirname(__file__), "golden")
L_MAX = 7


def dp_first_goal_counts(L_max: int) -> dict:
    goal = (3, 3)
    dvec = [(1, 0), (0, 1), (-1, 0), (0, -1)]
    counts = {(1, 1, 0): 1}
    out = {}
    for L in range(1, L_max + 1):
        nxt = {}
        arrived = 0
        for (x, y, d), c in counts.items():
            for a in range(7):
                if a == 0:
                    s = (x, y, (d + 3) % 4)
                elif a == 1:
                    s = (x, y, (d + 1) % 4)
                elif a == 2:
                    fx, fy = x + dvec[d][0], y + dvec[d][1]
                    if (fx, fy) == goal:
                        arrived += c
                        continue
                    if 1 <= fx <= 3 and 1 <= fy <= 3:
                        s = (fx, fy, d)
                    else:
                        s = (x, y, d)  # wall
                else:
                    s = (x, y, d)  # pickup/drop/toggle/done: no-ops here
                nxt[s] = nxt.get(s, 0) + c
        counts = nxt
        out[L] = arrived
    return out


def test_dp_matches_golden_counts():
    g = json.load(open(os.path.join(GOLD, "p3_empty5_first_goal_counts.json")))["counts"]
    dp = dp_first_goal_counts(10)
    for L in range(1, 5):
        assert dp[L] == 0
    for L_str, c in g.items():
        assert dp[int(L_str)] == c


def test_oracle_bruteforce_all_sequences():
    n = 7 ** L_MAX
    lanes = np.arange(n)
    digits = np.stack([(lanes // 7 ** (L_MAX - 1 - t)) % 7 for t in range(L_MAX)]).astype(np.uint8)
    env = OracleEnv("Empty-5x5-v0", n)
    env.reset()
    dp = dp_first_goal_counts(L_MAX)
    term_count = np.zeros(n, np.int64)
    for t in range(L_MAX):
        r, te, tr = env.step_no_obs(digits[t])
        L = t + 1
        assert int(te.sum()) == dp[L] * 7 ** (L_MAX - L), L
        assert not tr.any()
        if te.any():
            want = success_reward(0, L, 100)
            assert np.all(r[te == 1] == np.float32(want))
            assert np.all(r[te == 0] == 0)
        term_count += te
    assert term_count.max() <= 1
