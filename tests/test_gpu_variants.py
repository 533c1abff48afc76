"""GPU <-> oracle parity of the f3/f4 variants: reward costs composed with
the event rewards (step and rollout paths) and the full-grid observation."""
import zlib

import numpy as np
import pytest
import torch

from inputgen import random_actions, random_records
from oracle import OracleEnv

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("env_id,mode", [("DoorKey-8x8-v0", 0), ("LavaGapS7-v0", 1),
                                         ("Dynamic-Obstacles-8x8-v0", 0), ("KeyCorridorS3R3-v0", 1),
                                         ("GoToDoor-6x6-v0", 1), ("GoToDoor-6x6-v0", 0)])
def test_reward_costs_parity(env_id, mode):
    from paper_2407_19396_b200 import NavixEnv
    n, K = 700, 150
    g = NavixEnv(env_id, n, seed=2, reward_mode=mode)
    r = NavixEnv(env_id, n, seed=2, reward_mode=mode)
    o = OracleEnv(env_id, n, seed=2, reward_mode=mode)
    g.set_reward_costs(0.0125, 0.003)
    r.set_reward_costs(0.0125, 0.003)
    o.set_reward_costs(0.0125, 0.003)
    g.reset()
    r.reset()
    o.reset()
    acts = random_actions(9, K, n, 0, high=8)
    ro, rr, rte, rtr = r.rollout(torch.from_numpy(acts).cuda())
    for t in range(K):
        go, gr, gte, gtr = g.step(torch.from_numpy(acts[t]).cuda())
        oo, orw, ote, otr = o.step(acts[t])
        assert np.array_equal(gr.cpu().numpy().view(np.uint32), orw.view(np.uint32)), t
        assert np.array_equal(rr[t].cpu().numpy().view(np.uint32), orw.view(np.uint32)), t
        assert np.array_equal(gte.cpu().numpy(), ote) and np.array_equal(go.cpu().numpy(), oo)


@pytest.mark.parametrize("env_id,nob", [("DoorKey-8x8-v0", 0), ("KeyCorridorS3R3-v0", 0),
                                        ("Dynamic-Obstacles-8x8-v0", 4), ("Empty-5x5-v0", 0),
                                        ("KeyCorridorS3R1-v0", 0), ("LavaGapS6-v0", 0),
                                        ("DoorKey-16x16-v0", 0), ("Dynamic-Obstacles-16x16-v0", 8),
                                        ("FourRooms-v0", 0)])
def test_full_obs_parity(env_id, nob):
    from paper_2407_19396_b200 import NavixEnv
    n = 1500
    g = NavixEnv(env_id, n, seed=4)
    o = OracleEnv(env_id, n, seed=4)
    g.reset()
    o.reset()
    np.testing.assert_array_equal(g.observe_full().cpu().numpy(), o.observe_full())
    s = g.spec
    recs = random_records(zlib.crc32(env_id.encode()) % 997, n, s.height, s.width, s.max_steps, nob)
    g.import_state(recs)
    o.import_(recs)
    np.testing.assert_array_equal(g.observe_full().cpu().numpy(), o.observe_full())
    acts = random_actions(1, 20, n, 0, high=8)
    for t in range(20):
        g.step(torch.from_numpy(acts[t]).cuda())
        o.step(acts[t])
    np.testing.assert_array_equal(g.observe_full().cpu().numpy(), o.observe_full())


@pytest.mark.parametrize("env_id,mode,rev,tev", [("DoorKey-8x8-v0", 0, 0, 7), ("Empty-5x5-v0", 0, 7, 0),
                                                 ("LavaGapS7-v0", 1, 5, 3), ("Dynamic-Obstacles-8x8-v0", 0, 7, 3),
                                                 ("GoToDoor-8x8-v0", 0, 7, 1), ("KeyCorridorS3R3-v0", 1, 1, 6),
                                                 ("Dynamic-Obstacles-8x8-v0", 1, 0, 0)])
def test_event_functions_parity(env_id, mode, rev, tev):
    # Table 6 / 7 selection incl. `free` (R#42), step and rollout paths, with costs composed
    from paper_2407_19396_b200 import NavixEnv
    n, K = 600, 300
    g = NavixEnv(env_id, n, seed=3, reward_mode=mode)
    r = NavixEnv(env_id, n, seed=3, reward_mode=mode)
    o = OracleEnv(env_id, n, seed=3, reward_mode=mode)
    for e in (g, r, o):
        e.set_event_functions(rev, tev)
        e.set_reward_costs(0.01, 0.0)
        e.reset()
    acts = random_actions(12, K, n, 0, high=8)
    ro, rr, rte, rtr = r.rollout(torch.from_numpy(acts).cuda())
    for t in range(K):
        go, gr, gte, gtr = g.step(torch.from_numpy(acts[t]).cuda())
        oo, orw, ote, otr = o.step(acts[t])
        assert np.array_equal(gr.cpu().numpy().view(np.uint32), orw.view(np.uint32)), t
        assert np.array_equal(rr[t].cpu().numpy().view(np.uint32), orw.view(np.uint32)), t
        assert np.array_equal(gte.cpu().numpy(), ote) and np.array_equal(gtr.cpu().numpy(), otr), t
        assert np.array_equal(go.cpu().numpy(), oo), t
    np.testing.assert_array_equal(g.stats().cpu().numpy(), o.stats())
    np.testing.assert_array_equal(g.export_state(), o.export())


def test_setter_validation():
    from paper_2407_19396_b200 import NavixEnv, NavixError
    g = NavixEnv("DoorKey-8x8-v0", 10)
    with pytest.raises(NavixError):
        g.set_event_functions(8, 7)
    with pytest.raises(NavixError):
        g.set_reward_costs(-1.0, 0.0)
    assert g.lib.navix_set_observation(g.h, 2) == 2
    with pytest.raises(ValueError):
        NavixEnv("DoorKey-8x8-v0", 10, observation="rgb")


def test_every_accepted_id_has_a_kernel():
    # every id navix_spec_of accepts launches (reset, steps, observe, rollout,
    # full observation) in both observation kinds
    from paper_2407_19396_b200 import NavixEnv, NavixError, spec_of
    fams = ["Empty-{s}x{s}", "Empty-Random-{s}x{s}", "DoorKey-{s}x{s}", "DoorKey-Random-{s}x{s}",
            "Dynamic-Obstacles-{s}x{s}", "Dynamic-Obstacles-Random-{s}x{s}", "LavaGapS{s}", "GoToDoor-{s}x{s}",
            "KeyCorridorS{s}R1", "KeyCorridorS{s}R2", "KeyCorridorS{s}R3", "SimpleCrossingS{s}N1",
            "SimpleCrossingS{s}N2", "SimpleCrossingS{s}N3", "SimpleCrossingS{s}N5"]
    ids = [f.format(s=s) for f in fams for s in range(2, 19)] + ["FourRooms", "DistShift1", "DistShift2"]
    n_ok = 0
    for env_id in ids:
        try:
            spec_of(env_id)
        except NavixError:
            continue
        for obs in ("symbolic", "categorical"):
            g = NavixEnv(env_id, 130, seed=1, observation=obs)
            g.reset()
            for t in range(3):
                g.step(g.sample_actions(2, t, 1)[0])
            g.rollout_random(3, 3, 2)
            g.observe()
            g.observe_full()
            torch.cuda.synchronize()
            g.close()
        n_ok += 1
    assert n_ok == 43


def test_gotodoor_mission_matches_the_oracle_target():
    # the mission colour = the colour of the oracle's target door (its record's
    # last two bytes give the target (x, y)), across auto-resets
    from paper_2407_19396_b200 import NavixEnv, NavixError
    for S in (5, 6, 8):
        env_id = f"GoToDoor-{S}x{S}-v0"
        n = 700
        g = NavixEnv(env_id, n, seed=7)
        o = OracleEnv(env_id, n, seed=7)
        g.reset()
        o.reset()
        acts = random_actions(4, 30, n, 7)
        for t in range(30):
            g.step(torch.from_numpy(acts[t]).cuda())
            o.step(acts[t])
            rec = o.export()
            tx, ty = rec[:, -2].astype(int), rec[:, -1].astype(int)
            cells = rec[:, :3 * S * S].reshape(n, S, S, 3)
            want = cells[np.arange(n), ty, tx, 1]
            assert np.all(cells[np.arange(n), ty, tx, 0] == 4)  # the target is a door
            np.testing.assert_array_equal(g.observe_mission().cpu().numpy(), want, err_msg=f"{env_id} t={t}")
    with pytest.raises(NavixError):
        NavixEnv("DoorKey-8x8-v0", 10).observe_mission()
