"""Pins of the oracle's further Table 9 families (row f2):
Empty-Random-SxS and DistShift1/2 (Table 9; MiniGrid's EmptyEnv with
agent_start_pos=None and DistShiftEnv; R#33, R#34); the Crossings (Table 8's
SimpleCrossing with wall rivers, Table 9's Crossings with R_2 = MiniGrid's
LavaCrossing, lava rivers; R#35); GoToDoor, FourRooms, DynObs-Random.

DistShift: the layout the MiniGrid source fixes (goal (W-2, 1), lava strips
x = 3..W-4 on rows 1 and 2 (DistShift1) or 5 (DistShift2), agent (1,1) east)
and two hand-walked trajectories whose outcome differs between the two
variants.  Empty-Random: the start state is uniform over the (W-2)(H-2)-1
empty interior cells and the 4 directions (chi-square), never the goal.
"""
import numpy as np
import pytest
from scipy import stats as sps

from inputgen import record_from_map
from oracle import OracleEnv, spec_of

R, L, F = 1, 0, 2  # right, left, forward


@pytest.mark.parametrize("env_id,strip2", [("DistShift1-v0", 2), ("DistShift2-v0", 5)])
def test_distshift_layout(env_id, strip2):
    s = spec_of(env_id)
    assert (s.width, s.height, s.max_steps, s.n_actions) == (9, 7, 4 * 9 * 7, 7)
    env = OracleEnv(env_id, 3, seed=11)
    env.reset()
    full = env.observe_full()
    assert np.all(full == full[0])          # no randomness: every env identical
    f = full[0]                              # [x][y][c]
    for x in range(9):
        for y in range(7):
            if x in (0, 8) or y in (0, 6):
                want = [2, 5, 0]
            elif (x, y) == (7, 1):
                want = [8, 1, 0]
            elif 3 <= x <= 5 and y in (1, strip2):
                want = [9, 0, 0]
            elif (x, y) == (1, 1):
                want = [10, 0, 0]
            else:
                want = [1, 0, 0]
            assert f[x, y].tolist() == want, (x, y)


def _walk(env_id, actions):
    env = OracleEnv(env_id, 1)
    env.reset()
    out = []
    for a in actions:
        _, r, te, tr = env.step(np.array([a], np.uint8))
        out.append((float(r[0]), int(te[0]), int(tr[0])))
    return out


def test_distshift_lava_straight_ahead():
    # east from (1,1): (2,1) then the lava at (3,1) ends the episode with 0
    for env_id in ("DistShift1-v0", "DistShift2-v0"):
        out = _walk(env_id, [F, F])
        assert out[0] == (0.0, 0, 0)
        assert out[1] == (0.0, 1, 0)


def test_distshift_row2_path_separates_the_variants():
    path = [R, F, L] + [F] * 6 + [L, F]      # (1,2) -> east along row 2 -> (7,2) -> north to the goal
    out2 = _walk("DistShift2-v0", path)
    assert all(o == (0.0, 0, 0) for o in out2[:-1])
    r, te, tr = out2[-1]
    assert te == 1 and tr == 0
    assert r == pytest.approx(1 - 0.9 * len(path) / 252, abs=1e-7)
    out1 = _walk("DistShift1-v0", path)
    assert out1[3] == (0.0, 0, 0)            # (2,2) free
    assert out1[4] == (0.0, 1, 0)            # (3,2) is lava in DistShift1


@pytest.mark.parametrize("S", [6, 8, 16])
def test_empty_random_start_is_uniform(S):
    s = spec_of(f"Empty-Random-{S}x{S}-v0")
    assert (s.width, s.height, s.max_steps, s.n_actions) == (S, S, 4 * S * S, 7)
    n = 24000
    env = OracleEnv(f"Empty-Random-{S}x{S}-v0", n, seed=5)
    env.reset()
    full = env.observe_full()                 # [n][x][y][c]
    ag = np.argwhere(full[:, :, :, 0] == 10)
    assert ag.shape == (n, 3) and np.array_equal(ag[:, 0], np.arange(n))
    x, y = ag[:, 1], ag[:, 2]
    assert np.all((x >= 1) & (x <= S - 2) & (y >= 1) & (y <= S - 2))
    assert not np.any((x == S - 2) & (y == S - 2))
    assert np.all(full[:, S - 2, S - 2, 0] == 8)
    k = (S - 2) * (S - 2) - 1
    cnt = np.bincount((y - 1) * (S - 2) + (x - 1), minlength=k + 1)[:k]
    assert sps.chisquare(cnt).pvalue > 1e-4
    d = full[ag[:, 0], x, y, 2]
    assert sps.chisquare(np.bincount(d, minlength=4)).pvalue > 1e-4
    # episodes differ in start state; the same seed reproduces them
    env2 = OracleEnv(f"Empty-Random-{S}x{S}-v0", n, seed=5)
    env2.reset()
    assert np.array_equal(env2.observe_full(), full)


def test_empty_random_goal_reward_from_known_start():
    # import a start next to the goal and step onto it: success reward with T = 4 S^2

    m = ["######",
         "#....#",
         "#....#",
         "#..A.#",
         "#...G#",
         "######"]
    env = OracleEnv("Empty-Random-6x6-v0", 1)
    env.reset()
    env.import_(record_from_map(m, 1).reshape(1, -1))  # facing south, at (3,3)
    env.step(np.array([L], np.uint8))                   # now east
    _, r, te, _ = env.step(np.array([F], np.uint8))     # (4,3)
    assert te[0] == 0
    env.step(np.array([R], np.uint8))                   # south
    _, r, te, _ = env.step(np.array([F], np.uint8))     # goal (4,4)
    assert te[0] == 1 and float(r[0]) == pytest.approx(1 - 0.9 * 4 / 144, abs=1e-7)


def _crossing_levels(env_id, n, seed=7):
    env = OracleEnv(env_id, n, seed=seed)
    env.reset()
    return env.observe_full()[:, :, :, 0]  # [n][x][y] type


def _reachable(t, sx, sy):
    S = t.shape[0]
    seen = np.zeros_like(t, bool)
    st = [(sx, sy)]
    seen[sx, sy] = True
    while st:
        x, y = st.pop()
        for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            u, v = x + dx, y + dy
            if 0 <= u < S and 0 <= v < S and not seen[u, v] and t[u, v] != 2:
                seen[u, v] = True
                st.append((u, v))
    return seen


@pytest.mark.parametrize("env_id,S,N,ob", [("SimpleCrossingS9N1-v0", 9, 1, 2), ("SimpleCrossingS9N2-v0", 9, 2, 2),
                                           ("SimpleCrossingS9N3-v0", 9, 3, 2), ("SimpleCrossingS11N5-v0", 11, 5, 2),
                                           ("Crossings-S9N1-v0", 9, 1, 9), ("Navix-Crossings-S9N3-v0", 9, 3, 9),
                                           ("Crossings-S11N5-v0", 11, 5, 9), ("LavaCrossingS9N2-v0", 9, 2, 9)])
def test_crossing_structure_and_solvable(env_id, S, N, ob):
    s = spec_of(env_id)
    assert (s.width, s.height, s.max_steps, s.n_actions) == (S, S, 4 * S * S, 7)
    levels = _crossing_levels(env_id, 400)
    for t in levels:
        assert t[1, 1] == 10 and t[S - 2, S - 2] == 8
        # a river line holds S-3 obstacles (its one opening excepted); any other
        # interior line holds at most N obstacles (where rivers cross it) < S-3
        cols = [x for x in range(1, S - 1) if np.count_nonzero(t[x, 1:-1] == ob) == S - 3]
        rows = [y for y in range(1, S - 1) if np.count_nonzero(t[1:-1, y] == ob) == S - 3]
        assert all(x % 2 == 0 and 2 <= x <= S - 3 for x in cols)
        assert all(y % 2 == 0 and 2 <= y <= S - 3 for y in rows)
        assert len(cols) + len(rows) == N
        want = np.zeros((S, S), bool)
        for x in cols:
            want[x, 1:-1] = True
        for y in rows:
            want[1:-1, y] = True
        interior = np.pad(np.ones((S - 2, S - 2), bool), 1)
        got = t == ob
        assert not np.any(interior & (t == (9 if ob == 2 else 2)))  # one obstacle kind only
        assert not np.any(got & interior & ~want)      # no obstacle off the rivers
        assert np.count_nonzero(want & ~got) == N      # exactly one opening per river
        assert _reachable(np.where(t == 9, 2, t), 1, 1)[S - 2, S - 2]  # openings connect start and goal


@pytest.mark.parametrize("S,N", [(9, 1), (9, 2), (9, 3), (11, 5)])
def test_lava_crossing_is_simple_crossing_with_lava(S, N):
    # the same draws build the same rivers and openings; only the obstacle differs
    simple = _crossing_levels(f"SimpleCrossingS{S}N{N}-v0", 300, seed=4)
    for lava_id in (f"Crossings-S{S}N{N}-v0", f"LavaCrossingS{S}N{N}-v0"):
        lava = _crossing_levels(lava_id, 300, seed=4)
        inner = np.zeros((S, S), bool)
        inner[1:-1, 1:-1] = True
        want = np.where((simple == 2) & inner[None], 9, simple)
        assert np.array_equal(lava, want)


def test_lava_crossing_terminates_on_lava_and_sees_across():
    # Table 9 R_2 (caption P:972): "-1 when the agent is on the lava
    # square"; all envs terminate when the reward is not 0; MiniGrid's
    # lava pays 0 (R#3).  A vertical lava river at x = 2 with its opening at (2,5).
    m = ["#########",
         "#AV.....#",
         "#.V.....#",
         "#.V.....#",
         "#.V.....#",
         "#.......#",
         "#.V.....#",
         "#.V....G#",
         "#########"]
    for mode, want in ((0, 0.0), (1, -1.0)):
        env = OracleEnv("Crossings-S9N1-v0", 1, seed=0, reward_mode=mode)
        env.reset()
        env.import_(record_from_map(m, 0).reshape(1, -1))
        obs = env.observe()[0]
        # lava is see-through (MiniGrid Lava.see_behind): the cells beyond the
        # river are visible, e.g. (3,1) = view (vi=3, vj=4) facing east
        assert obs[3, 4].tolist() == [1, 0, 0] and obs[3, 5].tolist() == [9, 0, 0]
        _, r, te, tr = env.step(np.array([F], np.uint8))
        assert te[0] == 1 and tr[0] == 0 and float(r[0]) == want
        assert env.stats()[4] == 1
    # the same map with wall rivers (SimpleCrossing): the river occludes
    env = OracleEnv("SimpleCrossingS9N1-v0", 1, seed=0)
    env.reset()
    env.import_(record_from_map([r.replace("V", "#") for r in m], 0).reshape(1, -1))
    obs = env.observe()[0]
    assert obs[3, 5].tolist() == [2, 5, 0] and obs[3, 4].tolist() == [0, 0, 0]
    _, r, te, _ = env.step(np.array([F], np.uint8))
    assert te[0] == 0 and r[0] == 0


def test_crossing_river_subset_and_opening_uniform():
    # S9N2: the 2 rivers are a uniform 2-subset of the 6 candidates (C(6,2) = 15)
    lv = _crossing_levels("SimpleCrossingS9N2-v0", 6000, seed=9)
    keys = []
    for t in lv:
        v = tuple(x for x in (2, 4, 6) if np.count_nonzero(t[x, 1:-1] == 2) >= 5)
        h = tuple(y for y in (2, 4, 6) if np.count_nonzero(t[1:-1, y] == 2) >= 5)
        keys.append((v, h))
    _, cnt = np.unique(np.array([str(k) for k in keys]), return_counts=True)
    assert len(cnt) == 15 and sps.chisquare(cnt).pvalue > 1e-4
    # S9N1 with a vertical river: its opening row is uniform over 1..7
    lv = _crossing_levels("SimpleCrossingS9N1-v0", 8000, seed=10)
    ys = []
    for t in lv:
        for x in (2, 4, 6):
            col = t[x, 1:-1]
            if np.count_nonzero(col == 2) == 6:
                ys.append(1 + int(np.argmax(col != 2)))
    c = np.bincount(ys, minlength=8)[1:]
    assert len(ys) > 3000 and sps.chisquare(c).pvalue > 1e-4


# ---------------------------------------------------------------- GoToDoor
def _gtd(S, n, seed=3):
    env = OracleEnv(f"GoToDoor-{S}x{S}-v0", n, seed=seed)
    env.reset()
    return env, env.observe_full(), env.export()


@pytest.mark.parametrize("S", [5, 6, 8])
def test_gotodoor_structure(S):
    s = spec_of(f"GoToDoor-{S}x{S}-v0")
    assert (s.width, s.height, s.max_steps, s.n_actions, s.export_bytes) == (S, S, 4 * S * S, 7, 3 * S * S + 14)
    n = 3000
    _, full, rec = _gtd(S, n)
    ws, hs, tgt_side, first_col = [], [], [], []
    for k in range(n):
        t, c, st = full[k, :, :, 0], full[k, :, :, 1], full[k, :, :, 2]
        # room: the wall rectangle from (0,0); its size from the top wall's extent
        w = 1 + max(x for x in range(S) if t[x, 0] in (2, 4))
        h = 1 + max(y for y in range(S) if t[0, y] in (2, 4))
        assert 5 <= w <= S and 5 <= h <= S
        ring = [(x, 0) for x in range(w)] + [(x, h - 1) for x in range(w)] + \
               [(0, y) for y in range(1, h - 1)] + [(w - 1, y) for y in range(1, h - 1)]
        doors = [(x, y) for (x, y) in ring if t[x, y] == 4]
        assert len(doors) == 4 and all(t[x, y] == 2 for (x, y) in ring if (x, y) not in doors)
        assert all(st[x, y] == 1 for x, y in doors)                  # closed, not locked
        cols = [int(c[x, y]) for x, y in doors]
        assert len(set(cols)) == 4                                   # distinct colours
        top = [d for d in doors if d[1] == 0 and 0 < d[0] < w - 1]
        bot = [d for d in doors if d[1] == h - 1 and 0 < d[0] < w - 1]
        lef = [d for d in doors if d[0] == 0]
        rig = [d for d in doors if d[0] == w - 1]
        assert len(top) == len(bot) == len(lef) == len(rig) == 1
        assert 2 <= top[0][0] <= w - 3 and 2 <= bot[0][0] <= w - 3
        assert 2 <= lef[0][1] <= h - 3 and 2 <= rig[0][1] <= h - 3
        # everything outside the room is empty, the inside is empty but the agent
        out = np.ones((S, S), bool)
        out[:w, :h] = False
        assert np.all(t[out] == 1)
        ag = np.argwhere(t == 10)
        assert len(ag) == 1 and 1 <= ag[0][0] <= w - 2 and 1 <= ag[0][1] <= h - 2
        tx, ty = int(rec[k, -2]), int(rec[k, -1])
        assert (tx, ty) in doors
        ws.append(w)
        hs.append(h)
        tgt_side.append([top[0], bot[0], lef[0], rig[0]].index((tx, ty)))
        first_col.append(int(c[top[0]]))
    if S == 5:
        assert set(ws) == set(hs) == {5}
    else:
        assert sps.chisquare(np.bincount(ws, minlength=S + 1)[5:]).pvalue > 1e-4
        assert sps.chisquare(np.bincount(hs, minlength=S + 1)[5:]).pvalue > 1e-4
    assert sps.chisquare(np.bincount(tgt_side, minlength=4)).pvalue > 1e-4
    assert sps.chisquare(np.bincount(first_col, minlength=6)).pvalue > 1e-4


ROOM5 = ["##D##",
         "#...#",
         "D.A.D",
         "#...#",
         "##D##"]


def _room(action_seq, agent_dir, target, S=5, rows=ROOM5, reward_mode=0):
    env = OracleEnv(f"GoToDoor-{S}x{S}-v0", 1, reward_mode=reward_mode)
    env.reset()
    env.import_(record_from_map(rows, agent_dir, target=target).reshape(1, -1))
    outs = []
    for a in action_seq:
        o, r, te, tr = env.step(np.array([a], np.uint8))
        outs.append((o[0], float(r[0]), int(te[0]), int(tr[0])))
    return env, outs


def test_gotodoor_done_next_to_target_succeeds():
    # agent (2,2) facing north; target the top door (2,0): forward to (2,1), done
    env, outs = _room([F, 6], 3, (2, 0))
    assert outs[0][1:] == (0.0, 0, 0)
    assert outs[1][2] == 1 and outs[1][1] == pytest.approx(1 - 0.9 * 2 / 100, abs=1e-7)
    st = env.stats()
    assert st[0] == 1 and st[2] == 1 and st[5] == 0
    # navix reward mode: 1
    _, outs = _room([F, 6], 3, (2, 0), reward_mode=1)
    assert outs[1][1:3] == (1.0, 1)


def test_gotodoor_done_elsewhere_and_toggle_fail():
    env, outs = _room([F, 6], 3, (0, 2))   # next to the top door, but the target is the left one
    assert outs[1][1:] == (0.0, 1, 0)
    assert env.stats()[5] == 1             # n_failure
    env, outs = _room([6], 3, (2, 0))      # (2,2) is 2 cells from the target: not adjacent
    assert outs[0][1:] == (0.0, 1, 0)
    # toggle ends the episode (the door it faces is opened first)
    env, outs = _room([F, 5], 3, (2, 0))
    assert outs[1][1:] == (0.0, 1, 0)
    assert env.stats()[5] == 1
    full = env.observe_full()[0]
    assert full[2, 0].tolist() == [4, 4, 0]   # the top door is open now


def test_gotodoor_open_door_on_the_grid_edge_sees_outside_as_wall():
    # after toggling the top door open from (2,1) facing north, the view runs
    # off the grid: [MG] slices out-of-grid cells as Walls, so the cell behind
    # the door is a visible wall and everything further is unseen; the open
    # door's own row-4 neighbours (i +- 1, j - 1) are lit by process_vis too
    _, outs = _room([F, 5], 3, (4, 2))
    obs = outs[1][0]                              # [vi][vj][c], agent at (3, 6)
    assert obs[3, 6].tolist() == [1, 0, 0]        # own cell (carrying nothing)
    assert obs[3, 5].tolist() == [4, 4, 0]        # the open door in front
    assert obs[3, 4].tolist() == [2, 5, 0]        # outside the grid: wall
    assert obs[3, 3].tolist() == [0, 0, 0]        # behind it: unseen
    assert obs[2, 4].tolist() == obs[4, 4].tolist() == [2, 5, 0]
    assert np.count_nonzero(obs[:, :5, 0]) == 3   # rows beyond the door: only those walls


def test_gotodoor_open_edge_walk_blocked_outside():
    # an imported GoToDoor state may have an open grid edge (R#37): walking
    # off the grid is blocked as if by a wall
    rows = ["..D..",
            ".....",
            "A....",
            ".....",
            "....."]
    env = OracleEnv("GoToDoor-5x5-v0", 1)
    env.reset()
    env.import_(record_from_map(rows, 2, target=(2, 0)).reshape(1, -1))  # facing west at x = 0
    _, r, te, _ = env.step(np.array([F], np.uint8))
    rec = env.export()[0]
    assert (rec[75], rec[76]) == (0, 2) and te[0] == 0


@pytest.mark.parametrize("S", [5, 6, 8])
def test_gotodoor_closed_room_never_sees_outside_the_grid(S):
    # R#37: a generated room with its doors closed encloses the agent, and
    # [MG] process_vis only spreads from visible see-through cells, so no view
    # position outside the grid is ever visible (the kernels skip the
    # out-of-grid walls for such rooms).  Every action but toggle (which opens
    # a door and ends the episode); done ends episodes, so new rooms come too.
    n, T = 300, 40
    env = OracleEnv(f"GoToDoor-{S}x{S}-v0", n, seed=5)
    obs = env.reset()
    rng = np.random.default_rng(0)
    vi, vj = np.meshgrid(np.arange(7), np.arange(7), indexing="ij")
    fwd = np.array([(1, 0), (0, 1), (-1, 0), (0, -1)])
    checked = 0
    for _ in range(T):
        rec = env.export().astype(np.int64)
        ax, ay, d = rec[:, 3 * S * S], rec[:, 3 * S * S + 1], rec[:, 3 * S * S + 2]
        fx, fy = fwd[d, 0][:, None, None], fwd[d, 1][:, None, None]
        lx, ly = -fy, fx  # view column vi lies at lateral offset vi - 3, row vj at distance 6 - vj
        x = ax[:, None, None] + (6 - vj) * fx + (vi - 3) * lx
        y = ay[:, None, None] + (6 - vj) * fy + (vi - 3) * ly
        out = (x < 0) | (x >= S) | (y < 0) | (y >= S)
        assert not obs[out].any()
        checked += int(out.sum())
        obs, *_ = env.step(rng.choice([0, 1, 2, 3, 4, 6], size=n).astype(np.uint8))
    assert checked > 10000


# ---------------------------------------------------------------- FourRooms
def test_fourrooms_structure_and_uniform_placement():
    s = spec_of("Navix-FourRooms-v0")
    assert (s.width, s.height, s.max_steps, s.n_actions) == (17, 17, 100, 7)   # Table 9 size, [MG] T (R#38)
    n = 20000
    env = OracleEnv("FourRooms-v0", n, seed=2)
    env.reset()
    full = env.observe_full()
    t = full[:, :, :, 0]
    ag_cells, goal_cells, gaps = [], [], []
    for k in range(0, n):
        tk = t[k]
        border = np.ones((17, 17), bool)
        border[1:-1, 1:-1] = False
        assert np.all(tk[border] == 2)
        if k < 300:
            segs = {"v_top": [(8, y) for y in range(1, 8)], "v_bot": [(8, y) for y in range(9, 16)],
                    "h_left": [(x, 8) for x in range(1, 8)], "h_right": [(x, 8) for x in range(9, 16)]}
            for cells in segs.values():
                assert sum(tk[c] != 2 for c in cells) == 1     # exactly one opening per segment
            assert tk[8, 8] == 2
            inner = tk[1:-1, 1:-1]
            walls = np.count_nonzero(inner == 2)
            assert walls == 15 + 15 - 1 - 4
            # every free cell is reachable from the agent
            seen = _reachable(np.where(tk == 2, 2, 1), *np.argwhere(tk == 10)[0])
            assert np.all(seen[tk != 2])
            gaps.append([c for cells in segs.values() for c in cells if tk[c] != 2])
        (ax, ay), = np.argwhere(tk == 10)
        (gx, gy), = np.argwhere(tk == 8)
        ag_cells.append((ax, ay))
        goal_cells.append((gx, gy))
    # agent and goal uniform over the 200 free cells (cells are free in the
    # rooms' interiors; wall rows/columns only through their openings)
    room = [(x, y) for y in range(1, 16) for x in range(1, 16) if x != 8 and y != 8]
    idx = {c: i for i, c in enumerate(room)}
    a = np.bincount([idx[c] for c in ag_cells if c in idx], minlength=len(room))
    g = np.bincount([idx[c] for c in goal_cells if c in idx], minlength=len(room))
    assert sps.chisquare(a).pvalue > 1e-4 and sps.chisquare(g).pvalue > 1e-4
    assert all(a_ != g_ for a_, g_ in zip(ag_cells, goal_cells))


def test_fourrooms_truncates_at_100():
    env = OracleEnv("FourRooms-v0", 4, seed=1)
    env.reset()
    for t in range(100):
        _, r, te, tr = env.step(np.zeros(4, np.uint8))   # turning left forever
        assert not te.any()
        assert tr.all() == (t == 99)
    _, r, te, tr = env.step(np.zeros(4, np.uint8))
    assert env.export()[:, 3 * 289 + 5].tolist() == [0, 0, 0, 0]  # auto-reset: step_count 0


def test_gotodoor_navix_mode_on_door_done():
    # Table 6/7 `on_door_done` (R#39): only done *in front of* the mission's
    # door rewards (+1) and terminates; toggle and other dones continue
    env, outs = _room([F, 6], 3, (2, 0), reward_mode=1)        # (2,1) facing the target door
    assert outs[1][1:] == (1.0, 1, 0)
    env, outs = _room([F, 1, 6], 3, (2, 0), reward_mode=1)     # adjacent but facing east
    assert outs[2][1:] == (0.0, 0, 0)
    env, outs = _room([F, 5, 6], 3, (2, 0), reward_mode=1)     # toggle opens it, no termination; done still counts
    assert outs[1][1:] == (0.0, 0, 0)
    assert outs[2][1:] == (1.0, 1, 0)
    env, outs = _room([F, 6], 3, (0, 2), reward_mode=1)        # facing a door of another colour
    assert outs[1][1:] == (0.0, 0, 0)
    assert env.stats()[0] == 0


@pytest.mark.parametrize("S,nob", [(5, 2), (6, 3), (8, 4)])
def test_dynobs_random_start(S, nob):
    # [MG] DynamicObstaclesEnv(agent_start_pos=None) (R#40): agent uniform over
    # the empty interior cells and directions, then the balls avoid it
    env_id = f"Dynamic-Obstacles-Random-{S}x{S}"
    s = spec_of(env_id)
    assert (s.width, s.max_steps, s.n_actions, s.n_obstacles) == (S, 4 * S * S, 3, nob)
    n = 20000
    env = OracleEnv(env_id, n, seed=4)
    env.reset()
    full = env.observe_full()
    ag = np.argwhere(full[:, :, :, 0] == 10)
    assert np.array_equal(ag[:, 0], np.arange(n))
    x, y = ag[:, 1], ag[:, 2]
    k = (S - 2) * (S - 2) - 1
    cnt = np.bincount((y - 1) * (S - 2) + (x - 1), minlength=k + 1)
    assert cnt[k] == 0 and sps.chisquare(cnt[:k]).pvalue > 1e-4
    assert sps.chisquare(np.bincount(full[np.arange(n), x, y, 2], minlength=4)).pvalue > 1e-4
    assert np.all(np.count_nonzero(full[:, :, :, 0] == 6, axis=(1, 2)) == nob)
