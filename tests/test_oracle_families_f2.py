"""Pins of the oracle's further Table 9 families (row f2):
Empty-Random-SxS and DistShift1/2 (Table 9; MiniGrid's EmptyEnv with
agent_start_pos=None and DistShiftEnv; R#33, R#34).

DistShift: the layout the MiniGrid source fixes (goal (W-2, 1), lava strips
x = 3..W-4 on rows 1 and 2 (DistShift1) or 5 (DistShift2), agent (1,1) east)
and two hand-walked trajectories whose outcome differs between the two
variants.  Empty-Random: the start state is uniform over the (W-2)(H-2)-1
empty interior cells and the 4 directions (chi-square), never the goal.
"""
import numpy as np
import pytest
from scipy import stats as sps

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
    from inputgen import record_from_map
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
