"""Pins of the oracle's f3/f4 variants.

f4: reward composition (Table 6 time_cost / action_cost; Code 4 `compose`
P:673-680; R#31) — worked trajectory on Empty-5x5 and the zero-cost identity.
f3: the full-grid `symbolic` observation (Table 5, MiniGrid's
FullyObsWrapper; R#32) — hand-derived Empty-5x5 reset grid and the P2b
DoorKey layout.
"""
import json
import os
import struct

import numpy as np

from inputgen import record_from_map, random_actions
from oracle import OracleEnv

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bits(x):
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


def test_reward_costs_worked_trajectory():
    tc, ac = 0.01, 0.05
    env = OracleEnv("Empty-5x5-v0", 1)
    env.reset()
    env.set_reward_costs(tc, ac)
    rs = [float(env.step(np.array([a], np.uint8))[1][0]) for a in (2, 2, 1, 6, 2, 2)]
    f = np.float32
    step_cost = f(f(0.0) + f(-tc)) + f(-ac)   # event 0, then time cost, then action cost
    done_cost = f(f(0.0) + f(-tc)) + f(0.0)   # `done` pays no action cost
    assert bits(rs[0]) == bits(step_cost) and bits(rs[1]) == bits(step_cost) and bits(rs[2]) == bits(step_cost)
    assert bits(rs[3]) == bits(done_cost)
    success = f(1.0 - 0.9 * (6 / 100))
    assert bits(rs[5]) == bits(f(f(success) + f(-tc)) + f(-ac))
    assert abs(rs[5] - (0.946 - tc - ac)) < 1e-6  # success at step 6: 1 - 0.9*6/100


def test_zero_costs_are_the_identity():
    a = OracleEnv("LavaGapS7-v0", 64, seed=4)
    b = OracleEnv("LavaGapS7-v0", 64, seed=4)
    a.reset()
    b.reset()
    b.set_reward_costs(0.0, 0.0)
    acts = random_actions(3, 200, 64, 7)
    for t in range(200):
        assert np.array_equal(a.step(acts[t])[1].view(np.uint32), b.step(acts[t])[1].view(np.uint32))


def test_full_obs_empty5_reset():
    env = OracleEnv("Empty-5x5-v0", 1)
    env.reset()
    full = env.observe_full()[0]  # [x][y][c]
    assert full.shape == (5, 5, 3)
    for x in range(5):
        for y in range(5):
            if x in (0, 4) or y in (0, 4):
                want = [2, 5, 0]
            elif (x, y) == (3, 3):
                want = [8, 1, 0]
            elif (x, y) == (1, 1):
                want = [10, 0, 0]  # agent, red, facing east
            else:
                want = [1, 0, 0]
            assert full[x, y].tolist() == want, (x, y)


def test_full_obs_doorkey_layout_and_carry_not_drawn():
    g = json.load(open(os.path.join(GOLD, "p2b_doorkey_trace.json")))
    env = OracleEnv("DoorKey-8x8-v0", 1)
    env.reset()
    env.import_(record_from_map(g["map"], g["agent_dir"]).reshape(1, -1))
    full = env.observe_full()[0]
    assert full[1, 1].tolist() == [10, 0, 1]       # agent facing south
    assert full[3, 2].tolist() == [4, 4, 2]        # locked yellow door
    assert full[1, 3].tolist() == [5, 4, 0]        # yellow key
    assert full[6, 6].tolist() == [8, 1, 0]
    assert np.all(full[3, [0, 1, 3, 4, 5, 6, 7], 0] == 2)
    env.step(np.array([2], np.uint8))
    env.step(np.array([3], np.uint8))              # pick up the key
    full = env.observe_full()[0]
    assert full[1, 2].tolist() == [10, 0, 1] and full[1, 3].tolist() == [1, 0, 0]


def _walk_empty5(actions, reward_events, termination_events):
    env = OracleEnv("Empty-5x5-v0", 1)
    env.reset()
    env.set_event_functions(reward_events, termination_events)
    return env, [env.step(np.array([a], np.uint8))[1:] for a in actions]


def test_event_functions_free_reward_and_free_termination():
    # Table 6 / 7 `free` (R#42).  Empty-5x5 from (1,1) east: F (2,1), F (3,1),
    # R (south), F (3,2), F (3,3) = the goal at step 5
    path = [2, 2, 1, 2, 2]
    env, out = _walk_empty5(path, 7, 7)
    assert out[-1][1][0] == 1 and out[-1][0][0] == np.float32(1 - 0.9 * 5 / 100)
    env, out = _walk_empty5(path, 0, 7)             # free reward: the goal still terminates
    assert out[-1][1][0] == 1 and out[-1][0][0] == 0.0
    env, out = _walk_empty5(path, 7, 0)             # free termination: paid, not terminated
    assert out[-1][1][0] == 0 and out[-1][0][0] == np.float32(1 - 0.9 * 5 / 100)
    st = env.stats()
    assert st[0] == 0                              # no episode ended
    # standing on the goal does not pay again; walking off and back on does
    _, r, te, tr = env.step(np.array([0], np.uint8))
    assert r[0] == 0 and te[0] == 0
    for _ in range(100 - 6 - 1):
        _, r, te, tr = env.step(np.array([0], np.uint8))
    _, r, te, tr = env.step(np.array([0], np.uint8))
    assert tr[0] == 1 and te[0] == 0                # only truncation ends it
    st = env.stats()
    assert st[0] == 1 and st[2] == 0 and st[6] == 1


def test_event_functions_lava_and_collision():
    # LavaGap navix mode: lava pays -1 unless deselected; DynObs collision continues if not terminating
    from inputgen import record_from_map
    rows = ["#######", "#.A.V.#", "#.....#", "#.....#", "#.....#", "#....G#", "#######"]
    for rev, tev, want in ((7, 7, (-1.0, 1)), (5, 7, (0.0, 1)), (7, 5, (-1.0, 0)), (0, 0, (0.0, 0))):
        env = OracleEnv("LavaGapS7-v0", 1, reward_mode=1)
        env.reset()
        env.import_(record_from_map(rows, 0).reshape(1, -1))
        env.set_event_functions(rev, tev)
        env.step(np.array([2], np.uint8))
        _, r, te, _ = env.step(np.array([2], np.uint8))   # onto the lava at (4,1)
        assert (float(r[0]), int(te[0])) == want, (rev, tev)
    env = OracleEnv("Dynamic-Obstacles-5x5", 1)
    env.reset()
    env.set_event_functions(7, 3)                          # collisions pay -1 but do not end the episode
    env.import_(record_from_map(["#####", "#A..#", "#..B#", "#.BG#", "#####"], 3,
                                balls=[(3, 2), (2, 3)]).reshape(1, -1))  # facing the wall north
    _, r, te, _ = env.step(np.array([2], np.uint8))
    assert r[0] == -1.0 and te[0] == 0
