"""P7: invariants checked at every step of random oracle rollouts.

From the rules (Table 9 caption P:974):
the agent never stands on an impassable object; the border stays walls; keys
are conserved (grid + pocket); a locked door opens only through toggle with a
same-colour key; reward != 0 implies terminated; lava implies terminated with
0 (minigrid mode); truncation happens exactly at step_count == T without an
event; the call after a terminal step returns step_count 0 with reward 0;
observation values lie in the legal set; the stats identity
sum_len == sum of terminal step counts.
"""
import numpy as np
import pytest

from inputgen import BALL, DOOR, EMPTY, GOAL, KEY, LAVA, LOCKED, OPEN, WALL, random_actions
from oracle import OracleEnv

ENVS = ["Empty-5x5-v0", "Empty-8x8-v0", "DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0",
        "KeyCorridorS3R3-v0", "LavaGapS7-v0", "DoorKey-5x5-v0", "KeyCorridorS3R1-v0",
        "DoorKey-16x16-v0", "Dynamic-Obstacles-16x16-v0", "KeyCorridorS4R3-v0", "KeyCorridorS6R3-v0",
        "Empty-Random-8x8-v0", "DistShift1-v0", "DistShift2-v0", "SimpleCrossingS11N5-v0", "GoToDoor-8x8-v0",
        "FourRooms-v0", "Dynamic-Obstacles-Random-6x6"]


@pytest.mark.parametrize("env_id", ENVS)
def test_invariants_random_rollout(env_id):
    n, K = 48, 400
    env = OracleEnv(env_id, n, seed=123)
    s = env.spec
    H, W, T = s.height, s.width, s.max_steps
    env.reset()
    # exercise pickup/drop/toggle densely: half the lanes avoid 'left'/'right'
    acts = random_actions(99, K, n, s.n_actions)
    if s.n_actions == 7:
        bias = random_actions(98, K, n, 0, high=5) + 2
        acts[:, : n // 2] = bias[:, : n // 2]
    p = 3 * H * W
    prev = env.export()
    ep_len_sum = 0
    for t in range(K):
        obs, r, te, tr = env.step(acts[t])
        rec = env.export()
        cells = rec[:, :p].reshape(n, H, W, 3)
        for e in range(n):
            c = cells[e]
            ty = c[:, :, 0]
            ax, ay, ad = (int(v) for v in rec[e, p: p + 3])
            carry = (int(rec[e, p + 3]), int(rec[e, p + 4]))
            sc = int(rec[e, p + 5]) | (int(rec[e, p + 6]) << 8)
            was_done = prev[e, p + 11] == 1
            under = c[ay, ax]
            assert under[0] in (EMPTY, GOAL, LAVA) or (under[0] == DOOR and under[2] == OPEN), (t, e)
            border = np.ones((H, W), bool)
            border[1:-1, 1:-1] = False
            if s.family != 8:  # GoToDoor's room may be smaller than its grid (R#37)
                assert np.all(ty[border] == WALL)
            if was_done:
                assert sc == 0 and r[e] == 0 and te[e] == 0 and tr[e] == 0
                continue
            pc = prev[e, :p].reshape(H, W, 3)
            n_keys = np.count_nonzero(ty == KEY) + (carry[0] == KEY)
            n_keys0 = np.count_nonzero(pc[:, :, 0] == KEY) + (prev[e, p + 3] == KEY)
            assert n_keys == n_keys0
            # balls are conserved too in DynObs, where they move (grid + pocket)
            n_b = np.count_nonzero(ty == BALL) + (carry[0] == BALL)
            assert n_b == np.count_nonzero(pc[:, :, 0] == BALL) + (prev[e, p + 3] == BALL)
            unlocked = (pc[:, :, 0] == DOOR) & (pc[:, :, 2] == LOCKED) & ~((ty == DOOR) & (c[:, :, 2] == LOCKED))
            if unlocked.any():
                assert acts[t, e] == 5 and prev[e, p + 3] == KEY
                (uy, ux), = np.argwhere(unlocked)
                assert pc[uy, ux, 1] == prev[e, p + 4]
            if r[e] != 0:
                assert te[e] == 1
            if s.family == 8 and acts[t, e] in (5, 6):  # GoToDoor: toggle / done end the episode
                assert te[e] == 1
            if te[e] == 0 and tr[e] == 0:
                assert sc < T
            if tr[e]:
                assert sc == T and te[e] == 0
            if under[0] == LAVA:
                assert te[e] == 1 and r[e] == 0
            if te[e] or tr[e]:
                ep_len_sum += sc
        o = obs
        assert np.all(o[:, :, :, 0] <= 9) and np.all(o[:, :, :, 1] <= 5) and np.all(o[:, :, :, 2] <= 2)
        assert np.all(o[:, :, :, 0][o[:, :, :, 2] > 0] == DOOR)
        prev = rec
    st = env.stats()
    assert st[1] == ep_len_sum
    assert st[0] == st[2] + st[4] + st[5] + st[6]  # every episode ends one way
    assert st[7] == 0
