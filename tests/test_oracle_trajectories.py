"""Worked trajectories that pin the oracle's step rules (I, mu, R, gamma).

P2b  scripted DoorKey-8x8 trajectory (tests/golden/p2b_doorkey_trace.json):
     pickup, locked door blocks, toggle with the matching key, door open,
     goal reward 1 - 0.9*16/640 (Eq. 1, R#1/R#2).
P2c  DynObs collision with a wall (R#4) and the >=3 -> 0 action map (R#7);
     LavaGap lava termination with 0 / -1 (Table 6, R#3);
     KeyCorridor ball pickup success and the full-pocket no-op (R#8);
     truncation exactly at T and the next-step autoreset (R#18).
Also the SPEC S:399 Empty-5x5 example [F, F, R, F, F] -> reward, terminated.
"""
import json
import os
import struct

import numpy as np

from inputgen import BALL, DOOR, EMPTY, KEY, LOCKED, OPEN, YELLOW, decode_record, record_from_map
from oracle import OracleEnv

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def f32_bits(x) -> int:
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


def test_p2b_doorkey_scripted_trajectory():
    g = json.load(open(os.path.join(GOLD, "p2b_doorkey_trace.json")))
    env = OracleEnv(g["env_id"], 1, seed=0)
    env.reset()
    env.import_(record_from_map(g["map"], g["agent_dir"]).reshape(1, -1))
    for t, a in enumerate(g["actions"], start=1):
        obs, r, te, tr = env.step(np.array([a], np.uint8))
        d = decode_record(env.export()[0], 8, 8)
        if t < g["terminal_step"]:
            assert r[0] == 0 and te[0] == 0 and tr[0] == 0, t
        assert [d["agent"][0], d["agent"][1]] == g["positions_after"][t - 1], t
        assert d["agent"][2] == g["dirs_after"][t - 1], t
        o = obs[0]
        if t == 2:
            assert d["carry"] == (KEY, YELLOW) and d["cells"][3, 1, 0] == EMPTY
        if t in (4, 5):
            assert o[:, :, 0].T.tolist() == g["type_T_t4"], t
            assert o[:, :, 2].T[5].tolist() == g["state_T_t4_row5"]
            assert o[3, 6].tolist() == g["agent_cell_t4"]
        if t == 6:
            assert o[:, :, 0].T.tolist() == g["type_T_t6"]
            assert o[:, :, 2].T[5].tolist() == g["state_T_t6_row5"]
            assert d["cells"][2, 3].tolist() == [DOOR, YELLOW, OPEN]
            assert d["carry"] == (KEY, YELLOW)  # the key is not consumed
        if t == 5:
            assert d["cells"][2, 3].tolist() == [DOOR, YELLOW, LOCKED]
    assert te[0] == 1 and tr[0] == 0
    assert f32_bits(r[0]) == int(g["terminal_reward_f32_bits"], 16)
    # next call: autoreset -> FIRST observation, reward 0, flags 0, episode 1
    obs, r, te, tr = env.step(np.array([2], np.uint8))
    d = decode_record(env.export()[0], 8, 8)
    assert r[0] == 0 and te[0] == 0 and tr[0] == 0
    assert d["step_count"] == 0 and d["episode"] == 1 and d["prev_done"] == 0
    assert env.stats().tolist() == [1, 16, 1, 16, 0, 0, 0, 0]


def test_spec_s399_empty5_shortest_path():
    env = OracleEnv("Empty-5x5-v0", 1)
    env.reset()
    rs = []
    for a in [2, 2, 1, 2, 2]:
        obs, r, te, tr = env.step(np.array([a], np.uint8))
        rs.append((float(r[0]), int(te[0])))
    assert [x[1] for x in rs] == [0, 0, 0, 0, 1]
    assert f32_bits(rs[-1][0]) == 0x3F747AE1  # 0.955 = RN32(1 - 0.9*5/100)


def test_p2c_dynobs_wall_collision_any_seed():
    for seed in range(20):
        for first in (0, 5):  # `toggle` (5) maps to `left` (0) in DynObs (R#7)
            env = OracleEnv("Dynamic-Obstacles-8x8-v0", 4, seed=seed)
            env.reset()
            _, r, te, tr = env.step(np.full(4, first, np.uint8))
            assert np.all(te == 0) and np.all(r == 0)
            _, r, te, tr = env.step(np.full(4, 2, np.uint8))
            assert np.all(te == 1) and np.all(r == -1.0) and np.all(tr == 0)
            rec = env.export()
            for e in range(4):
                d = decode_record(rec[e], 8, 8, 4)
                assert d["agent"][:2] == (1, 1)
            assert env.stats()[5] == 4  # n_failure (collisions)


LAVA_MAP = ["#######",
            "#AV...#",
            "#.V...#",
            "#.....#",
            "#.V...#",
            "#.V..G#",
            "#######"]


def test_p2c_lavagap_lava_terminates():
    for mode, want in ((0, 0.0), (1, -1.0)):
        env = OracleEnv("LavaGapS7-v0", 1, seed=0, reward_mode=mode)
        env.reset()
        env.import_(record_from_map(LAVA_MAP, 0).reshape(1, -1))
        _, r, te, tr = env.step(np.array([2], np.uint8))
        d = decode_record(env.export()[0], 7, 7)
        assert te[0] == 1 and tr[0] == 0 and float(r[0]) == want
        assert d["agent"][:2] == (2, 1)  # lava can be overlapped
        assert env.stats()[4] == 1


KC_MAP = ["#######",
          "#.#.OB#",
          "#D#.###",
          "#.#.D.#",
          "#D#.###",
          "#K#...#",
          "#######"]


def test_p2c_keycorridor_ball_pickup_and_full_pocket():
    # agent standing in the (unlocked, open) doorway (4,1) facing the ball (5,1)
    m = [r.replace("O", "A") for r in KC_MAP]
    rec = record_from_map(m, 0, step_count=9)
    # the agent's cell must be the open door: patch the record (cell (4,1))
    rec[3 * (1 * 7 + 4): 3 * (1 * 7 + 4) + 3] = [DOOR, YELLOW, OPEN]
    env = OracleEnv("KeyCorridorS3R3-v0", 1, seed=0)
    env.reset()
    env.import_(rec.reshape(1, -1))
    obs, r, te, tr = env.step(np.array([3], np.uint8))
    assert te[0] == 1 and abs(float(r[0]) - (1 - 9 * 10 / (10 * 270))) < 1e-7  # Eq. (1), sc = 10
    d = decode_record(env.export()[0], 7, 7)
    assert d["carry"][0] == BALL and obs[0, 3, 6, 0] == BALL
    # carrying the key: pickup facing the ball is a no-op, no event
    rec2 = record_from_map(m, 0, carry=(KEY, YELLOW))
    rec2[3 * (1 * 7 + 4): 3 * (1 * 7 + 4) + 3] = [DOOR, YELLOW, OPEN]
    env.import_(rec2.reshape(1, -1))
    obs, r, te, tr = env.step(np.array([3], np.uint8))
    assert te[0] == 0 and r[0] == 0
    d = decode_record(env.export()[0], 7, 7)
    assert d["carry"] == (KEY, YELLOW) and d["cells"][1, 5, 0] == BALL
    # drop needs an empty front cell: the ball is in front -> no-op
    obs, r, te, tr = env.step(np.array([4], np.uint8))
    d = decode_record(env.export()[0], 7, 7)
    assert d["carry"] == (KEY, YELLOW)


def test_p2c_truncation_and_autoreset():
    env = OracleEnv("Empty-8x8-v0", 3, seed=0)
    env.reset()
    for t in range(1, 257):
        obs, r, te, tr = env.step(np.zeros(3, np.uint8))
        if t < 256:
            assert not tr.any() and not te.any()
    assert tr.all() and not te.any() and np.all(r == 0)
    first = OracleEnv("Empty-8x8-v0", 3, seed=0).reset()
    obs, r, te, tr = env.step(np.full(3, 2, np.uint8))  # action ignored on reset
    assert np.array_equal(obs, first) and not r.any() and not te.any() and not tr.any()
    d = decode_record(env.export()[0], 8, 8)
    assert d["step_count"] == 0 and d["episode"] == 1
    assert env.stats().tolist() == [3, 768, 0, 0, 0, 0, 3, 0]


def test_locked_door_needs_matching_colour():
    m = ["########",
         "#A.L...#",
         "#..#...#",
         "#..#...#",
         "#..#...#",
         "#..#...#",
         "#..#..G#",
         "########"]
    env = OracleEnv("DoorKey-8x8-v0", 1)
    env.reset()
    # wrong colour key in the pocket: toggle does nothing
    rec = record_from_map(m, 0, carry=(KEY, 2))
    env.import_(rec.reshape(1, -1))
    env.step(np.array([2], np.uint8))  # forward to (2,1)
    env.step(np.array([5], np.uint8))  # toggle the locked yellow door
    d = decode_record(env.export()[0], 8, 8)
    assert d["agent"][:2] == (2, 1)
    assert d["cells"][1, 3].tolist() == [DOOR, YELLOW, LOCKED]
    # no key: still locked; matching key: opens, and toggling again closes it
    rec = record_from_map(m, 0, carry=(KEY, YELLOW))
    env.import_(rec.reshape(1, -1))
    env.step(np.array([2], np.uint8))
    env.step(np.array([5], np.uint8))
    d = decode_record(env.export()[0], 8, 8)
    assert d["cells"][1, 3].tolist() == [DOOR, YELLOW, OPEN]
    env.step(np.array([5], np.uint8))
    d = decode_record(env.export()[0], 8, 8)
    assert d["cells"][1, 3].tolist() == [DOOR, YELLOW, 1]  # closed, no longer locked
    env.step(np.array([2], np.uint8))  # closed door blocks
    assert decode_record(env.export()[0], 8, 8)["agent"][:2] == (2, 1)


def test_drop_and_pickup_roundtrip():
    m = ["########",
         "#A.#...#",
         "#..L...#",
         "#K.#...#",
         "#..#...#",
         "#..#...#",
         "#..#..G#",
         "########"]
    env = OracleEnv("DoorKey-8x8-v0", 1)
    env.reset()
    env.import_(record_from_map(m, 1).reshape(1, -1))
    env.step(np.array([2], np.uint8))  # (1,2)
    env.step(np.array([3], np.uint8))  # pickup key at (1,3)
    env.step(np.array([3], np.uint8))  # pickup again: front empty -> no-op
    d = decode_record(env.export()[0], 8, 8)
    assert d["carry"] == (KEY, YELLOW)
    env.step(np.array([4], np.uint8))  # drop onto (1,3)
    d = decode_record(env.export()[0], 8, 8)
    assert d["carry"] == (EMPTY, 0) and d["cells"][3, 1].tolist() == [KEY, YELLOW, 0]
    env.step(np.array([4], np.uint8))  # drop with nothing carried -> no-op
    env.step(np.array([6], np.uint8))  # done -> no-op
    env.step(np.array([200], np.uint8))  # out-of-range action -> no-op (R#15)
    d2 = decode_record(env.export()[0], 8, 8)
    assert np.array_equal(d2["cells"], d["cells"]) and d2["agent"] == d["agent"]
    assert d2["step_count"] == 7
