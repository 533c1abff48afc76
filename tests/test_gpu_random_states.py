"""GPU <-> oracle parity on random imported states (observation and step rules
in configurations the generators never produce: doors of every state and
colour, keys/balls/boxes/lava/goals anywhere, every carried object, every
pose), plus export/import round trips.  Bit-exact."""
import zlib

import numpy as np
import pytest
import torch

from inputgen import random_actions, random_records
from oracle import OracleEnv

pytestmark = pytest.mark.gpu

CASES = [("DoorKey-8x8-v0", 0), ("Empty-5x5-v0", 0), ("LavaGapS7-v0", 0), ("KeyCorridorS3R3-v0", 0),
         ("Dynamic-Obstacles-8x8-v0", 4), ("KeyCorridorS3R1-v0", 0), ("DoorKey-6x6-v0", 0),
         ("Dynamic-Obstacles-5x5-v0", 2), ("DoorKey-16x16-v0", 0), ("Dynamic-Obstacles-16x16-v0", 8),
         ("KeyCorridorS5R3-v0", 0), ("DistShift2-v0", 0), ("Empty-Random-6x6-v0", 0),
         ("SimpleCrossingS11N5-v0", 0), ("GoToDoor-5x5-v0", 0), ("GoToDoor-8x8-v0", 0),
         ("FourRooms-v0", 0)]


@pytest.mark.parametrize("env_id,nob", CASES)
def test_random_states_observe_and_step(env_id, nob):
    from paper_2407_19396_b200 import NavixEnv
    n = 3000
    g = NavixEnv(env_id, n, seed=21)
    s = g.spec
    o = OracleEnv(env_id, n, seed=21)
    recs = random_records(zlib.crc32(env_id.encode()) % 1000, n, s.height, s.width, s.max_steps, nob, p_prev_done=0.05,
                          open_edge=env_id.startswith("GoToDoor"))  # R#37: open grid edge, target bytes
    g.import_state(recs)
    o.import_(recs)
    np.testing.assert_array_equal(g.export_state(), recs)  # import/export round trip
    np.testing.assert_array_equal(g.observe().cpu().numpy(), o.observe())
    acts = random_actions(5, 12, n, 0, high=8)
    for t in range(12):
        go, gr, gte, gtr = g.step(torch.from_numpy(acts[t]).cuda())
        oo, orw, ote, otr = o.step(acts[t])
        np.testing.assert_array_equal(go.cpu().numpy(), oo, err_msg=f"obs step {t}")
        np.testing.assert_array_equal(gr.cpu().numpy().view(np.uint32), orw.view(np.uint32))
        np.testing.assert_array_equal(gte.cpu().numpy(), ote)
        np.testing.assert_array_equal(gtr.cpu().numpy(), otr)
        np.testing.assert_array_equal(g.export_state(), o.export(), err_msg=f"state step {t}")
    np.testing.assert_array_equal(g.stats().cpu().numpy(), o.stats())


def test_import_rejects_illegal_records():
    from paper_2407_19396_b200 import NavixEnv, NavixError
    g = NavixEnv("DoorKey-8x8-v0", 2)
    s = g.spec
    good = random_records(1, 2, 8, 8, s.max_steps)
    g.import_state(good)
    bad = good.copy()
    bad[0, 0:3] = (1, 0, 0)  # border cell not a wall
    with pytest.raises(NavixError):
        g.import_state(bad)
    bad = good.copy()
    bad[1, 3 * 64] = 0  # agent on the border
    with pytest.raises(NavixError):
        g.import_state(bad)
    bad = good.copy()
    bad[0, 3 * 9] = 42  # unknown object type
    with pytest.raises(NavixError):
        g.import_state(bad)
    with pytest.raises(NavixError):
        g.import_state(good[:1])
    np.testing.assert_array_equal(g.export_state(), good)  # rejected imports change nothing


@pytest.mark.parametrize("env_id", ["KeyCorridorS3R3-v0", "KeyCorridorS3R1-v0", "KeyCorridorS4R3-v0",
                                    "KeyCorridorS6R3-v0"])
@pytest.mark.parametrize("p_prev_done", [0.03, 0.15])
def test_keycorridor_sparse_resets_warp_generator(env_id, p_prev_done):
    # random step counts desynchronise the episodes, so most steps reset a few
    # lanes per warp: the warp-cooperative connect_all (<= 4 resetting lanes)
    # and the one-lane-per-level path (more) both run, on the persistent
    # (S3R*) and one-tile (S4R3, S6R3) kernels
    from paper_2407_19396_b200 import NavixEnv
    n = 2000
    g = NavixEnv(env_id, n, seed=5)
    s = g.spec
    o = OracleEnv(env_id, n, seed=5)
    recs = random_records(77, n, s.height, s.width, s.max_steps, 0, p_prev_done=p_prev_done)
    g.import_state(recs)
    o.import_(recs)
    steps = 300 if s.height <= 7 else 60
    acts = random_actions(9, steps, n, 0, high=8)
    for t in range(steps):
        go, gr, gte, gtr = g.step(torch.from_numpy(acts[t]).cuda())
        oo, orw, ote, otr = o.step(acts[t])
        np.testing.assert_array_equal(go.cpu().numpy(), oo, err_msg=f"obs step {t}")
        np.testing.assert_array_equal(gr.cpu().numpy().view(np.uint32), orw.view(np.uint32))
        np.testing.assert_array_equal(gte.cpu().numpy(), ote)
        np.testing.assert_array_equal(gtr.cpu().numpy(), otr)
        if t % 50 == 49:
            np.testing.assert_array_equal(g.export_state(), o.export(), err_msg=f"state step {t}")
    np.testing.assert_array_equal(g.stats().cpu().numpy(), o.stats())
