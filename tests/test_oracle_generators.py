"""P8: the oracle's level generators (P0 of reset(key); Table 9).

Structural invariants from the [MG] _gen_grid definitions and S:446-452,
solvability by breadth-first search, and chi-square tests of
every drawn quantity against the uniform laws of DESIGN.md "Level generators"
(R#22/R#23).  10^4 levels per family, each from its own Philox stream
(global env index = counter word 0).
"""
from collections import deque

import numpy as np
import pytest
from scipy.stats import chisquare

from inputgen import BALL, BLUE, DOOR, EMPTY, GOAL, KEY, LAVA, LOCKED, WALL, YELLOW
from oracle import OracleEnv

N = 10_000


def levels(env_id, n=N, seed=7):
    env = OracleEnv(env_id, n, seed=seed)
    env.reset()
    rec = env.export()
    s = env.spec
    H, W = s.height, s.width
    cells = rec[:, : 3 * H * W].reshape(n, H, W, 3)
    p = 3 * H * W
    agent = rec[:, p: p + 3].astype(int)
    return env, cells, agent, rec


def uniform_ok(values, k, lo=0):
    counts = np.bincount(np.asarray(values) - lo, minlength=k)
    assert len(counts) == k, counts
    return chisquare(counts).pvalue > 1e-4


def bfs_reach(cells, start, passable):
    H, W = cells.shape[:2]
    seen = np.zeros((H, W), bool)
    q = deque([start])
    seen[start[1], start[0]] = True
    while q:
        x, y = q.popleft()
        for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            nx, ny = x + dx, y + dy
            if 0 <= nx < W and 0 <= ny < H and not seen[ny, nx] and passable(cells[ny, nx]):
                seen[ny, nx] = True
                q.append((nx, ny))
    return seen


def test_doorkey8_structure_distribution_solvable():
    env, cells, agent, rec = levels("DoorKey-8x8-v0")
    splits, door_ys, dirs, agent_y_at2 = [], [], [], []
    for e in range(N):
        c = cells[e]
        t = c[:, :, 0]
        col = [x for x in range(2, 6) if np.all((t[:, x] == WALL) | (t[:, x] == DOOR))]
        assert len(col) == 1
        split = col[0]
        doors = np.argwhere(t == DOOR)
        assert len(doors) == 1 and doors[0][1] == split
        dy = int(doors[0][0])
        assert 1 <= dy <= 5 and c[dy, split].tolist() == [DOOR, YELLOW, LOCKED]
        keys = np.argwhere(t == KEY)
        assert len(keys) == 1 and keys[0][1] < split and c[keys[0][0], keys[0][1], 1] == YELLOW
        ax, ay, ad = agent[e]
        assert 1 <= ax < split and 1 <= ay <= 6 and t[ay, ax] == EMPTY
        assert (ax, ay) != (int(keys[0][1]), int(keys[0][0]))
        assert t[6, 6] == GOAL
        splits.append(split)
        door_ys.append(dy)
        dirs.append(ad)
        if split == 2:
            agent_y_at2.append(ay)
        # solvable: key reachable on the agent's side, goal reachable through the door
        side = bfs_reach(c, (ax, ay), lambda v: v[0] in (EMPTY, GOAL))
        assert side[keys[0][0], keys[0][1]] or any(
            side[keys[0][0] + dy_, keys[0][1] + dx_]
            for dx_, dy_ in ((1, 0), (-1, 0), (0, 1), (0, -1)))
        allp = bfs_reach(c, (ax, ay), lambda v: v[0] in (EMPTY, GOAL, DOOR, KEY))
        assert allp[6, 6]
    assert uniform_ok(splits, 4, lo=2)
    assert uniform_ok(door_ys, 5, lo=1)
    assert uniform_ok(dirs, 4)
    assert uniform_ok(agent_y_at2, 6, lo=1)
    assert env.stats()[7] == 0


def test_lavagap7_structure_distribution_solvable():
    env, cells, agent, rec = levels("LavaGapS7-v0")
    gx_all, gy_all = [], []
    for e in range(N):
        t = cells[e][:, :, 0]
        lava = np.argwhere(t == LAVA)
        xs = set(int(v) for v in lava[:, 1])
        assert len(xs) == 1 and len(lava) == 4  # one column of 5 interior cells, one gap
        gx = xs.pop()
        assert 2 <= gx <= 4
        gy = [y for y in range(1, 6) if t[y, gx] == EMPTY]
        assert len(gy) == 1
        gx_all.append(gx)
        gy_all.append(gy[0])
        assert tuple(agent[e]) == (1, 1, 0) and t[5, 5] == GOAL
        assert bfs_reach(cells[e], (1, 1), lambda v: v[0] in (EMPTY, GOAL))[5, 5]
    assert uniform_ok(gx_all, 3, lo=2)
    assert uniform_ok(gy_all, 5, lo=1)


def test_dynobs8_structure_distribution():
    env, cells, agent, rec = levels("Dynamic-Obstacles-8x8-v0")
    p = 3 * 64 + 12
    first = []
    for e in range(N):
        t = cells[e][:, :, 0]
        balls = [(int(rec[e, p + 2 * i]), int(rec[e, p + 2 * i + 1])) for i in range(4)]
        assert len(set(balls)) == 4
        for bx, by in balls:
            assert t[by, bx] == BALL and cells[e][by, bx, 1] == BLUE
            assert (bx, by) != (1, 1)
        assert np.count_nonzero(t == BALL) == 4
        assert tuple(agent[e]) == (1, 1, 0) and t[6, 6] == GOAL
        bx, by = balls[0]
        first.append((by - 1) * 6 + (bx - 1))
    # ball 0 is uniform over the 34 empty interior cells (not agent, not goal)
    counts = np.bincount(first, minlength=36)
    assert counts[0] == 0 and counts[35] == 0
    assert chisquare(counts[1:35]).pvalue > 1e-4


def test_keycorridor_s3r3_structure_distribution_solvable():
    env, cells, agent, rec = levels("KeyCorridorS3R3-v0")
    ridx, colours, krows, poses = [], [], [], []
    for e in range(N):
        c = cells[e]
        t = c[:, :, 0]
        locked = np.argwhere((t == DOOR) & (c[:, :, 2] == LOCKED))
        assert len(locked) == 1
        ly, lx = map(int, locked[0])
        assert lx == 4 and ly in (1, 3, 5)
        r = (ly - 1) // 2
        colour = int(c[ly, lx, 1])
        balls = np.argwhere(t == BALL)
        assert len(balls) == 1 and tuple(balls[0]) == (ly, 5)
        keys = np.argwhere(t == KEY)
        assert len(keys) == 1 and keys[0][1] == 1 and c[keys[0][0], 1, 1] == colour
        assert t[2, 3] == EMPTY and t[4, 3] == EMPTY  # the hallway
        ax, ay, ad = agent[e]
        assert ax == 3 and ay in (2, 3, 4)
        front = c[ay + (0, 1, 0, -1)[ad], ax + (1, 0, -1, 0)[ad]]
        # empty or wall when placed; connect_all may since have turned a wall
        # into a closed (unlocked) door
        assert front[0] in (EMPTY, WALL) or (front[0] == DOOR and front[2] == 1)
        # connect_all: every room interior reachable through doors of any state
        allp = bfs_reach(c, (ax, ay), lambda v: v[0] in (EMPTY, DOOR, KEY, BALL))
        for i in range(3):
            for j in range(3):
                assert allp[2 * j + 1, 2 * i + 1], (e, i, j)
        # key reachable without the locked door
        nolock = bfs_reach(c, (ax, ay), lambda v: v[0] == EMPTY or (v[0] == DOOR and v[2] != LOCKED))
        ky, kx = map(int, keys[0])
        assert any(nolock[ky + dy, kx + dx] for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)))
        ridx.append(r)
        colours.append(colour)
        krows.append((int(keys[0][0]) - 1) // 2)
        poses.append(ay)
    assert uniform_ok(ridx, 3)
    assert uniform_ok(colours, 6)
    assert uniform_ok(krows, 3)
    assert env.stats()[7] == 0


@pytest.mark.parametrize("env_id", ["Empty-5x5-v0", "Empty-8x8-v0"])
def test_empty_fixed_layout(env_id):
    env, cells, agent, rec = levels(env_id, n=16)
    S = env.spec.width
    t = cells[:, :, :, 0]
    border = np.ones((S, S), bool)
    border[1:-1, 1:-1] = False
    assert np.all(t[:, border] == WALL)
    assert np.count_nonzero(t[0] == WALL) == 4 * (S - 1)  # 28 for 8x8
    assert np.all(t[:, S - 2, S - 2] == GOAL)
    assert np.all(agent == [1, 1, 0])
    assert np.all(rec == rec[0])


def test_levels_are_reproducible_and_seed_dependent():
    a = levels("DoorKey-8x8-v0", n=256, seed=1)[3]
    b = levels("DoorKey-8x8-v0", n=256, seed=1)[3]
    c = levels("DoorKey-8x8-v0", n=256, seed=2)[3]
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)
