"""Pins of the Dynamic-Obstacles transition system mu (the oracle's
`Env::step`, oracle/minigrid.cpp, the DynObs block) against what the paper,
SPEC and MiniGrid fix, on imported states whose outcome holds for EVERY
Philox draw.

Sources: the transition mu "updates the state of the entities according to
the MDP state transitions" (App. A); R_3 "-1 when the agent is
hit by a flying object" and "All environments terminate when the reward is
not 0" (Table 9 caption); SPEC's forced move "ball with one
free neighbor -> ball at that neighbor" and stay-if-none;
MiniGrid's DynamicObstaclesEnv.step (R#4, R#5): the front cell is read BEFORE
the balls move, each ball in creation order is `place_obj`-ed inside the 3x3
box around it (clipped to the grid), never on an object or the agent, and
stays when no cell is free.

(a) a ball with exactly one admissible cell moves there, its old cell empties;
(b) a ball with none stays;
(c) the agent's cell and the goal are never chosen;
(d) two balls competing for one cell: creation order decides, both ways;
    a vacated cell is free for the later balls of the same step;
(e) a ball that moves into the agent's front cell blocks `forward`:
    no collision, reward 0 (not_clear is read before the motion);
(f) a ball in front that moves away still gives the -1 collision, and the
    agent moves into the vacated cell (the intervention reads after);
    a wall front gives the collision whatever the balls do; the goal in
    front is a success, not a collision;
(g) ball conservation and grid <-> record consistency at every step of a
    random rollout, each move inside the 3x3 box, never onto the agent;
(h) chi-square: destinations uniform over the admissible cells, balls
    independent of each other (distinct Philox words), and the draw is
    word i of block (env, episode, 1<<16 | step_count, 0) (R#20-R#22).
"""
import numpy as np
import pytest
from scipy.stats import chi2

from inputgen import BALL, EMPTY, GOAL, decode_record, random_actions, record_from_map
from oracle import OracleEnv
from oracle.binding import philox4x32_10

ID = "Dynamic-Obstacles-8x8-v0"
N = 256  # envs per fixture: 256 different Philox streams (global index)


def run_fixture(rows, agent_dir, balls, action, *, n=N, seed=0, step_count=5, episode=3, env_id=ID):
    env = OracleEnv(env_id, n, seed=seed)
    env.reset()
    rec = record_from_map(rows, agent_dir, balls=balls, step_count=step_count, episode=episode)
    env.import_(np.tile(rec, (n, 1)))
    _, r, te, tr = env.step(np.full(n, action, np.uint8))
    H, W = len(rows), len(rows[0])
    ds = [decode_record(x, H, W, len(balls)) for x in env.export()]
    return ds, r, te, tr, env


# ball 0 at (1,1): its box is x 0..2, y 0..2; (2,1) wall, agent (2,2): only (1,2)
FORCED = ["########",
          "#B#....#",
          "#.A....#",
          "#......#",
          "#...B..#",
          "#....B.#",
          "#...B.G#",
          "########"]
OTHER = [(4, 4), (5, 5), (4, 6)]


def test_a_forced_move_and_old_cell_cleared():
    for action in (0, 1):  # left / right: no interaction with the front cell
        ds, r, te, tr, _ = run_fixture(FORCED, 0, [(1, 1)] + OTHER, action)
        for d in ds:
            assert d["balls"][0] == (1, 2)
            assert d["cells"][2, 1, 0] == BALL and d["cells"][1, 1, 0] == EMPTY
            assert d["agent"][:2] == (2, 2)
        assert not te.any() and not tr.any() and not r.any()


def test_b_no_admissible_cell_stays():
    rows = [r for r in FORCED]
    rows[2] = "##A....#"  # (1,2) wall too: the box holds walls and the agent only
    ds, r, te, *_ = run_fixture(rows, 0, [(1, 1)] + OTHER, 1)
    for d in ds:
        assert d["balls"][0] == (1, 1) and d["cells"][1, 1, 0] == BALL
    assert not te.any()


def test_c_agent_and_goal_never_chosen():
    # ball 0 at (5,5): its box holds walls, the agent (6,5) and the goal (6,6)
    rows = ["########",
            "#B.B...#",
            "#......#",
            "#B.....#",
            "#...####",
            "#...#BA#",
            "#...##G#",
            "########"]
    balls = [(5, 5), (1, 1), (3, 1), (1, 3)]
    ds, r, te, *_ = run_fixture(rows, 2, balls, 1)
    for d in ds:
        assert d["balls"][0] == (5, 5), "only the goal and the agent were free: the ball must stay"
        assert d["cells"][6, 6, 0] == GOAL
    # open (5,6): now it is the only admissible cell
    rows[6] = "#...#.G#"
    ds, *_ = run_fixture(rows, 2, balls, 1)
    for d in ds:
        assert d["balls"][0] == (5, 6) and d["cells"][5, 5, 0] == EMPTY


# ball at (1,1) and ball at (1,3) both have (1,2) as their only admissible cell
CONTEST = ["########",
           "#B#....#",
           "#.A....#",
           "#B#....#",
           "###....#",
           "#......#",
           "#..B.B.#",
           "########"]


def test_d_creation_order_decides():
    far = [(3, 6), (5, 6)]
    ds, *_ = run_fixture(CONTEST, 0, [(1, 1), (1, 3)] + far, 1)
    for d in ds:
        assert d["balls"][:2] == [(1, 2), (1, 3)]
    ds, *_ = run_fixture(CONTEST, 0, [(1, 3), (1, 1)] + far, 1)
    for d in ds:
        assert d["balls"][:2] == [(1, 2), (1, 1)]


def test_d_vacated_cell_is_free_for_later_balls():
    # ball 0 at (1,2) can only go to (1,1); ball 1 at (1,3) can only go to
    # the cell ball 0 just left
    rows = ["########",
            "#.#....#",
            "#B#....#",
            "#B##A..#",
            "###....#",
            "#......#",
            "#..B.B.#",
            "########"]
    ds, *_ = run_fixture(rows, 0, [(1, 2), (1, 3), (3, 6), (5, 6)], 1)
    for d in ds:
        assert d["balls"][:2] == [(1, 1), (1, 2)]
        assert d["cells"][3, 1, 0] == EMPTY


def test_e_ball_into_front_cell_blocks_forward_without_collision():
    # agent (2,2) facing east, front (3,2) empty; ball 0 at (3,1) whose only
    # admissible cell is (3,2)
    rows = ["########",
            "#.#B#..#",
            "#.A.#..#",
            "#......#",
            "#......#",
            "#...B..#",
            "#...B.B#",
            "########"]
    ds, r, te, tr, env = run_fixture(rows, 0, [(3, 1), (4, 5), (4, 6), (6, 6)], 2)
    for d in ds:
        assert d["balls"][0] == (3, 2)
        assert d["agent"][:2] == (2, 2)  # blocked by the ball that moved in
    assert not te.any() and not r.any() and not tr.any()
    assert env.stats()[5] == 0


def test_f_ball_leaving_front_cell_still_collides():
    # agent (2,2) east, ball 0 in front at (3,2); its only admissible cell is (3,1)
    rows = ["########",
            "#.#.#..#",
            "#.AB#..#",
            "#.###..#",
            "#......#",
            "#...B..#",
            "#...B.B#",
            "########"]
    ds, r, te, tr, env = run_fixture(rows, 0, [(3, 2), (4, 5), (4, 6), (6, 6)], 2)
    for d in ds:
        assert d["balls"][0] == (3, 1)
        assert d["agent"][:2] == (3, 2)  # the intervention reads the front after the motion
    assert te.all() and np.all(r == -1.0) and not tr.any()
    assert env.stats()[5] == N  # n_failure counts the collisions


def test_f_wall_front_collides_goal_front_succeeds():
    rows = ["########",
            "#A.....#",
            "#......#",
            "#......#",
            "#..B...#",
            "#...B..#",
            "#..B..B#",
            "########"]
    # facing north at (1,1): wall in front
    ds, r, te, *_ = run_fixture(rows, 3, [(3, 4), (4, 5), (3, 6), (6, 6)], 2)
    assert te.all() and np.all(r == -1.0)
    assert all(d["agent"][:2] == (1, 1) for d in ds)
    # facing east into the goal: the success reward (Eq. 1, sc = 10), not the collision
    rows2 = ["########",
             "#......#",
             "#.B....#",
             "#......#",
             "#..B...#",
             "#...B..#",
             "#..B.AG#",
             "########"]
    ds, r, te, *_ = run_fixture(rows2, 0, [(2, 2), (3, 4), (4, 5), (3, 6)], 2, step_count=9)
    want = np.float32(1.0 - 0.9 * (10 / 256))
    assert te.all() and np.all(r == want)
    assert all(d["agent"][:2] == (6, 6) for d in ds)


@pytest.mark.parametrize("env_id", [ID, "Dynamic-Obstacles-16x16-v0", "Dynamic-Obstacles-5x5-v0",
                                    "Dynamic-Obstacles-Random-6x6-v0"])
def test_g_conservation_and_box_moves(env_id):
    n, K = 64, 300
    env = OracleEnv(env_id, n, seed=7)
    s = env.spec
    H, W, nb = s.height, s.width, s.n_obstacles
    env.reset()
    acts = random_actions(5, K, n, s.n_actions)
    prev = [decode_record(x, H, W, nb) for x in env.export()]
    for t in range(K):
        env.step(acts[t])
        cur = [decode_record(x, H, W, nb) for x in env.export()]
        for e in range(n):
            d, p = cur[e], prev[e]
            cells = d["cells"][:, :, 0]
            # grid <-> record: the listed balls are exactly the ball cells, distinct
            assert sorted(d["balls"]) == sorted((int(x), int(y)) for y, x in np.argwhere(cells == BALL))
            assert len(set(d["balls"])) == nb
            assert (d["agent"][0], d["agent"][1]) not in d["balls"]
            if p["prev_done"]:
                continue  # regenerated level
            for (bx, by), (ox, oy) in zip(d["balls"], p["balls"]):
                assert max(abs(bx - ox), abs(by - oy)) <= 1  # inside the 3x3 box
                assert 1 <= bx <= W - 2 and 1 <= by <= H - 2
        prev = cur


def _chi2_ok(counts):
    counts = np.asarray(counts, float)
    exp = counts.sum() / counts.size
    stat = float(((counts - exp) ** 2 / exp).sum())
    return chi2.sf(stat, counts.size - 1) > 1e-4, stat


# ball 0 at (2,2): box x 1..3, y 1..3; (1,1) and (3,3) walls, agent (3,1):
# admissible (2,1), (1,2), (3,2), (1,3), (2,3) -> 5 cells
# ball 1 at (5,5): box x 4..6, y 4..6; goal (6,6), (4,4) wall: admissible
# (5,4), (6,4), (4,5), (6,5), (4,6), (5,6) -> 6 cells
CHI_ROWS = ["########",
            "##.A...#",
            "#.B....#",
            "#..#...#",
            "#...#..#",
            "#B...B.#",
            "#B....G#",
            "########"]
CHI_BALLS = [(2, 2), (5, 5), (1, 5), (1, 6)]
ADM0 = [(2, 1), (1, 2), (3, 2), (1, 3), (2, 3)]
ADM1 = [(5, 4), (6, 4), (4, 5), (6, 5), (4, 6), (5, 6)]


def test_h_uniform_independent_and_draw_discipline():
    n = 12000
    seed, ep, sc = 0x1234_5678_9ABC, 11, 17
    ds, *_ = run_fixture(CHI_ROWS, 1, CHI_BALLS, 1, n=n, seed=seed, step_count=sc, episode=ep)
    b0 = [ADM0.index(d["balls"][0]) for d in ds]
    b1 = [ADM1.index(d["balls"][1]) for d in ds]
    ok, stat = _chi2_ok(np.bincount(b0, minlength=5))
    assert ok, stat
    ok, stat = _chi2_ok(np.bincount(b1, minlength=6))
    assert ok, stat
    # independence of ball 0 and ball 1: uniform over the 30 pairs
    ok, stat = _chi2_ok(np.bincount(np.array(b0) * 6 + np.array(b1), minlength=30))
    assert ok, stat
    # draw discipline (R#20-R#22): ball i takes word i of the Philox block
    # (env, episode, 1<<16 | step_count, 0) keyed by the seed, mapped by
    # bounded(u, |C|) onto the admissible cells enumerated row-major
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for e in range(0, n, 97):
        w = philox4x32_10([e, ep, (1 << 16) | sc, 0], key)
        assert ds[e]["balls"][0] == ADM0[(int(w[0]) * 5) >> 32]
        assert ds[e]["balls"][1] == ADM1[(int(w[1]) * 6) >> 32]
