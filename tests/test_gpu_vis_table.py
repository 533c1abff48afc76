"""The per-pose visibility tables (step_kernel.cuh obs_table_kernel) checked
exhaustively against the oracle's literal process_vis: every agent pose of
every static-layout family (Dynamic-Obstacles with balls scattered, Empty,
Empty-Random, DistShift) and every (pose, wall column, door row, door state)
of DoorKey's generated layouts, imported as states (import recognises the
layouts and sets the table flags) and observed; plus the layouts the tables
must NOT serve (a second door, an extra wall), which take the generic path."""
import numpy as np
import pytest
import torch

from inputgen import BALL, BLUE, DOOR, EMPTY, GOAL, GREY, KEY, LAVA, LOCKED, OPEN, RED, WALL, YELLOW
from oracle import OracleEnv

pytestmark = pytest.mark.gpu


def _record(cells, ax, ay, d, balls=(), sc=3):
    H, W = cells.shape[:2]
    rec = list(cells.reshape(-1)) + [ax, ay, d, EMPTY, 0] + list(int(sc).to_bytes(2, "little"))
    rec += list((5).to_bytes(4, "little")) + [0]
    for bx, by in balls:
        rec += [bx, by]
    return np.array(rec, np.uint8)


def _frame(H, W):
    c = np.zeros((H, W, 3), np.uint8)
    c[:, :] = (EMPTY, 0, 0)
    c[0, :] = c[-1, :] = c[:, 0] = c[:, -1] = (WALL, GREY, 0)
    return c


def _check(env_id, recs):
    from paper_2407_19396_b200 import NavixEnv
    recs = np.stack(recs)
    n = len(recs)
    g = NavixEnv(env_id, n, seed=0)
    o = OracleEnv(env_id, n, seed=0)
    g.import_state(recs)
    o.import_(recs)
    np.testing.assert_array_equal(g.observe().cpu().numpy(), o.observe())
    acts = np.random.default_rng(1).integers(0, 3, size=n).astype(np.uint8)  # turns and forward
    go, *_ = g.step(torch.from_numpy(acts).cuda())
    oo, *_ = o.step(acts)
    np.testing.assert_array_equal(go.cpu().numpy(), oo)


@pytest.mark.parametrize("env_id,S", [("Empty-5x5-v0", 5), ("Empty-8x8-v0", 8), ("Empty-16x16-v0", 16),
                                      ("Empty-Random-6x6", 6), ("Dynamic-Obstacles-8x8-v0", 8),
                                      ("Dynamic-Obstacles-5x5-v0", 5)])
def test_static_layout_every_pose(env_id, S):
    c = _frame(S, S)
    c[S - 2, S - 2] = (GOAL, 1, 0)
    nob = {5: 2, 6: 3, 8: 4, 16: 8}[S] if env_id.startswith("Dynamic") else 0
    rng = np.random.default_rng(S)
    recs = []
    for ay in range(1, S - 1):
        for ax in range(1, S - 1):
            for d in range(4):
                cc = c.copy()
                free = [(x, y) for y in range(1, S - 1) for x in range(1, S - 1)
                        if (x, y) != (ax, ay) and (x, y) != (S - 2, S - 2)]
                balls = [free[i] for i in rng.permutation(len(free))[:nob]]
                for bx, by in balls:
                    cc[by, bx] = (BALL, BLUE, 0)
                recs.append(_record(cc, ax, ay, d, balls))
    _check(env_id, recs)


@pytest.mark.parametrize("env_id,strip2", [("DistShift1-v0", 2), ("DistShift2-v0", 5)])
def test_distshift_every_pose(env_id, strip2):
    c = _frame(7, 9)
    c[1, 7] = (GOAL, 1, 0)
    for x in range(3, 6):
        c[1, x] = c[strip2, x] = (LAVA, RED, 0)
    recs = [_record(c, ax, ay, d) for ay in range(1, 6) for ax in range(1, 8) for d in range(4)]
    _check(env_id, recs)


@pytest.mark.parametrize("S", [5, 6, 8])
def test_doorkey_every_layout_and_pose(S):
    recs = []
    for split in range(2, S - 2):
        for door_y in range(1, S - 2):
            for state in (LOCKED, 1, OPEN):
                c = _frame(S, S)
                c[1:-1, split] = (WALL, GREY, 0)
                c[door_y, split] = (DOOR, YELLOW, state)
                c[S - 2, S - 2] = (GOAL, 1, 0)
                c[S - 2, 1] = (KEY, YELLOW, 0) if split > 1 else c[S - 2, 1]
                for ay in range(1, S - 1):
                    for ax in range(1, S - 1):
                        if ax == split and not (ay == door_y and state == OPEN):
                            continue  # the agent cannot stand in the wall or a closed door
                        if (ax, ay) == (1, S - 2):
                            continue  # the key's cell
                        for d in range(4):
                            recs.append(_record(c, ax, ay, d))
    _check(f"DoorKey-{S}x{S}-v0", recs)


def test_layouts_the_tables_must_not_serve():
    recs = []
    S = 8
    for variant in range(3):
        c = _frame(S, S)
        c[1:-1, 3] = (WALL, GREY, 0)
        c[2, 3] = (DOOR, YELLOW, LOCKED)
        c[6, 6] = (GOAL, 1, 0)
        if variant == 0:
            c[4, 5] = (DOOR, 2, 1)  # a second (closed) door
        elif variant == 1:
            c[5, 5] = (WALL, GREY, 0)  # an extra wall
        else:
            c[5, 3] = (DOOR, 2, OPEN)  # two doors in the wall column
        for ay in range(1, S - 1):
            for ax in (1, 2, 4, 6):
                if c[ay, ax, 0] != EMPTY:
                    continue
                for d in range(4):
                    recs.append(_record(c, ax, ay, d))
    _check("DoorKey-8x8-v0", recs)
    # an Empty grid with an object on it: not the template
    c = _frame(8, 8)
    c[6, 6] = (GOAL, 1, 0)
    c[3, 4] = (WALL, GREY, 0)
    _check("Empty-8x8-v0", [_record(c, ax, ay, d) for ay in (1, 2, 5) for ax in (1, 2, 5) for d in range(4)])


@pytest.mark.parametrize("env_id,S", [("LavaGapS7-v0", 7), ("LavaGapS5-v0", 5), ("Crossings-S9N2-v0", 9),
                                      ("Crossings-S11N5-v0", 11), ("SimpleCrossingS9N1-v0", 9)])
def test_border_opacity_every_pose(env_id, S):
    # lava is see-through: with the border the only opaque cells, the table
    # serves every pose (SimpleCrossing only when an import has no wall river)
    c = _frame(S, S)
    c[S - 2, S - 2] = (GOAL, 1, 0)
    for y in range(1, S - 1):
        if y != 2:
            c[y, 2] = (LAVA, RED, 0)  # a lava river at x = 2 with its opening at y = 2
    if S >= 9:
        for x in range(1, S - 1):
            if x != 5:
                c[4, x] = (LAVA, RED, 0)
    c[1, S - 2] = (KEY, 2, 0)  # a see-through object
    recs = [_record(c, ax, ay, d) for ay in range(1, S - 1) for ax in range(1, S - 1) for d in range(4)
            if c[ay, ax, 0] in (EMPTY, LAVA, GOAL)]
    _check(env_id, recs)
    # a wall or a door inside: the generic path
    c2 = c.copy()
    c2[3, 3] = (WALL, GREY, 0) if S > 5 else (DOOR, 3, 1)
    _check(env_id, [_record(c2, 1, 1, d) for d in range(4)] + [_record(c2, 1, 3, d) for d in range(4)])
