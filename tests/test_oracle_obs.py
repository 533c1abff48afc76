"""Pins of the oracle's observation function O (Table 5, [MG] gen_obs).

P2  worked example: Empty-5x5 reset and after `left` (tests/golden/p2_*.json).
P5  visibility: the oracle's literal [MG] process_vis loops equal an
    independent formulation (row closures of a 7-bit mask, written here) on
    every pattern with <= 3 opaque cells and on random patterns; monotonicity
    (S:229).
P6  rotation: slice + rotate_left^(dir+1) equals the closed form
    world = agent + (6 - vj) * DIR_TO_VEC[dir] + (vi - 3) * DIR_TO_VEC[(dir+1) % 4].
Invariants: out-of-grid cells are never visible (R#12), the agent cell is
always visible, four `left`s give the same observation.
"""
import itertools
import json
import os

import numpy as np
import pytest

from inputgen import random_actions
from oracle import OracleEnv, process_vis7, view_tags

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DIR_TO_VEC = [(1, 0), (0, 1), (-1, 0), (0, -1)]


def test_p2_empty5_reset_observation():
    g = json.load(open(os.path.join(GOLD, "p2_empty5_reset.json")))
    env = OracleEnv("Empty-5x5-v0", 1, seed=0)
    obs = env.reset()[0]
    assert obs[:, :, 0].T.tolist() == g["type_T_reset"]
    gc = g["goal_cell"]
    assert obs[gc["vi"], gc["vj"]].tolist() == gc["value"]
    walls = obs[:, :, 0] == 2
    assert np.all(obs[walls][:, 1] == g["wall_colour"])
    others = ~walls & ~((obs[:, :, 0] == 8))
    assert np.all(obs[others][:, 1] == 0) and np.all(obs[:, :, 2] == 0)
    # agent cell: nothing carried -> empty (1, 0, 0), always visible (R#13)
    assert obs[3, 6].tolist() == [1, 0, 0]
    obs2, r, te, tr = env.step(np.array([0], np.uint8))
    assert obs2[0, :, :, 0].T[5:7].tolist() == g["type_T_after_left_rows_5_6"]
    assert np.all(obs2[0, :, :, 0].T[:5] == 0)


def _closure_vis(opaque: np.ndarray) -> np.ndarray:
    """Independent formulation: per row j (6 -> 0) the visible set is the closure
    of the seeds under 'a visible transparent cell shows its row neighbours',
    and the next row's seeds are the visible transparent cells and their two
    lateral neighbours.  Written as explicit set iteration, not bit tricks."""
    vis = np.zeros((7, 7), bool)
    seeds = {3}
    for j in range(6, -1, -1):
        row = set(seeds)
        changed = True
        while changed:
            changed = False
            for i in list(row):
                if not opaque[i, j]:
                    for k in (i - 1, i + 1):
                        if 0 <= k < 7 and k not in row:
                            row.add(k)
                            changed = True
        for i in row:
            vis[i, j] = True
        seeds = set()
        for i in row:
            if not opaque[i, j]:
                seeds |= {k for k in (i - 1, i, i + 1) if 0 <= k < 7}
    return vis


def test_p5_visibility_exhaustive_up_to_three_opaque():
    cells = [(i, j) for i in range(7) for j in range(7) if (i, j) != (3, 6)]
    n = 0
    for k in range(4):
        for combo in itertools.combinations(cells, k):
            op = np.zeros((7, 7), np.uint8)
            for c in combo:
                op[c] = 1
            got = process_vis7(op).astype(bool)
            want = _closure_vis(op)
            assert np.array_equal(got, want), combo
            n += 1
    assert n == 1 + 48 + 1128 + 17296


def test_p5_visibility_random_and_monotone():
    rng = np.random.default_rng(5)
    for trial in range(3000):
        p = rng.uniform(0.05, 0.7)
        op = (rng.random((7, 7)) < p).astype(np.uint8)
        op[3, 6] = rng.integers(0, 2)  # the agent's own cell may be opaque too
        got = process_vis7(op).astype(bool)
        assert np.array_equal(got, _closure_vis(op))
        assert got[3, 6]
        # monotonicity: removing an opaque cell never shrinks the mask
        ones = np.argwhere(op)
        if len(ones):
            i, j = ones[rng.integers(len(ones))]
            op2 = op.copy()
            op2[i, j] = 0
            got2 = process_vis7(op2).astype(bool)
            assert np.all(got2 >= got)


@pytest.mark.parametrize("W,H", [(5, 5), (8, 8), (7, 7)])
def test_p6_rotation_closed_form(W, H):
    for ax in range(W):
        for ay in range(H):
            for d in range(4):
                tags = view_tags(W, H, ax, ay, d)
                D, R = DIR_TO_VEC[d], DIR_TO_VEC[(d + 1) % 4]
                for vi in range(7):
                    for vj in range(7):
                        x = ax + (6 - vj) * D[0] + (vi - 3) * R[0]
                        y = ay + (6 - vj) * D[1] + (vi - 3) * R[1]
                        want = y * W + x if (0 <= x < W and 0 <= y < H) else -1
                        assert tags[vi, vj] == want, (ax, ay, d, vi, vj)
                assert tags[3, 6] == ay * W + ax  # the agent sits at view (3, 6)


@pytest.mark.parametrize("env_id", ["Empty-8x8-v0", "DoorKey-8x8-v0", "KeyCorridorS3R3-v0",
                                    "LavaGapS7-v0", "Dynamic-Obstacles-8x8-v0"])
def test_four_lefts_cycle_and_oob_never_visible(env_id):
    n = 64
    env = OracleEnv(env_id, n, seed=3)
    env.reset()
    acts = random_actions(11, 40, n, env.spec.n_actions)
    W, H = env.spec.width, env.spec.height
    for t in range(40):
        obs, _, te, tr = env.step(acts[t])
        rec = env.export()
        for e in range(n):
            p = 3 * H * W
            ax, ay, d = int(rec[e, p]), int(rec[e, p + 1]), int(rec[e, p + 2])
            tags = view_tags(W, H, ax, ay, d)
            assert np.all(obs[e][tags < 0] == 0), "an out-of-grid cell was visible"
            assert obs[e, 3, 6, 0] != 0, "agent cell must be visible"
    if env_id.startswith("Dynamic"):
        return  # balls move on every step, so `left` x4 does not return the same frame
    before = env.observe()
    done = env.export()[:, 3 * H * W + 11] == 1
    for _ in range(4):
        obs, _, te, tr = env.step(np.zeros(n, np.uint8))
    still = ~done & (te == 0) & (tr == 0)
    assert np.array_equal(obs[still], before[still])
