"""f1: navix_rollout — K steps in one launch with the state kept
on chip — must be bit-identical to K navix_step calls (every output of every
step, the final canonical state, the statistics), and to the oracle."""
import numpy as np
import pytest
import torch

from inputgen import random_actions
from oracle import OracleEnv

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("env_id,n,K", [
    ("DoorKey-8x8-v0", 4096, 96), ("Dynamic-Obstacles-8x8-v0", 1000, 80), ("KeyCorridorS3R3-v0", 777, 300),
    ("LavaGapS7-v0", 513, 120), ("Empty-5x5-v0", 16, 250), ("DoorKey-5x5-v0", 129, 64),
    ("KeyCorridorS3R1-v0", 200, 290), ("DoorKey-16x16-v0", 300, 100), ("Dynamic-Obstacles-16x16-v0", 260, 60),
    ("Empty-Random-6x6-v0", 300, 150), ("DistShift1-v0", 300, 120),
    ("SimpleCrossingS9N3-v0", 300, 150), ("GoToDoor-8x8-v0", 300, 100),
    ("FourRooms-v0", 300, 130)])
@pytest.mark.parametrize("small_batch_kernels", [True, False])
def test_rollout_equals_sequential_steps(env_id, n, K, small_batch_kernels):
    # small_batch_kernels=False: the one-tile-per-CTA rollout and the
    # persistent step at every size (navix_set_small_batch_threshold(0))
    from paper_2407_19396_b200 import NavixEnv
    a = NavixEnv(env_id, n, seed=8)
    b = NavixEnv(env_id, n, seed=8)
    if not small_batch_kernels:
        a.set_small_batch_threshold(0)
        b.set_small_batch_threshold(0)
    a.reset()
    b.reset()
    acts = torch.from_numpy(random_actions(6, 2 * K, n, 0, high=8)).cuda()
    for half in range(2):  # two consecutive rollouts: state carried over between launches
        ro, rr, rte, rtr = a.rollout(acts[half * K:(half + 1) * K].contiguous())
        for t in range(K):
            o, r, te, tr = b.step(acts[half * K + t])
            assert torch.equal(ro[t], o), (half, t)
            assert torch.equal(rr[t].view(torch.int32), r.view(torch.int32))
            assert torch.equal(rte[t], te) and torch.equal(rtr[t], tr)
        assert np.array_equal(a.export_state(), b.export_state())
    assert torch.equal(a.stats(), b.stats())


def test_rollout_matches_oracle():
    from paper_2407_19396_b200 import NavixEnv
    n, K = 2048, 200
    g = NavixEnv("DoorKey-8x8-v0", n, seed=3)
    o = OracleEnv("DoorKey-8x8-v0", n, seed=3)
    g.reset()
    o.reset()
    acts = random_actions(2, K, n, 7)
    ro, rr, rte, rtr = g.rollout(torch.from_numpy(acts).cuda())
    for t in range(K):
        oo, orw, ote, otr = o.step(acts[t])
        assert np.array_equal(ro[t].cpu().numpy(), oo), t
        assert np.array_equal(rr[t].cpu().numpy().view(np.uint32), orw.view(np.uint32))
        assert np.array_equal(rte[t].cpu().numpy(), ote) and np.array_equal(rtr[t].cpu().numpy(), otr)
    assert np.array_equal(g.export_state(), o.export())
    assert np.array_equal(g.stats().cpu().numpy(), o.stats())


@pytest.mark.parametrize("env_id,n,K,t0", [("DoorKey-8x8-v0", 1000, 50, 0), ("Dynamic-Obstacles-8x8-v0", 513, 40, 7),
                                          ("KeyCorridorS3R3-v0", 300, 30, 123), ("FourRooms-v0", 200, 30, 5)])
def test_rollout_random_policy_in_kernel(env_id, n, K, t0):
    # row f1: the in-kernel random policy equals rollout() on sample_actions()'s stream
    from paper_2407_19396_b200 import NavixEnv
    a = NavixEnv(env_id, n, seed=4)
    b = NavixEnv(env_id, n, seed=4)
    a.reset()
    b.reset()
    ra = a.rollout_random(77, t0, K)
    rb = b.rollout(b.sample_actions(77, t0, K))
    for x, y in zip(ra, rb):
        assert torch.equal(x, y)
    np.testing.assert_array_equal(a.export_state(), b.export_state())


@pytest.mark.parametrize("env_id", ["DoorKey-8x8-v0", "KeyCorridorS3R3-v0", "LavaGapS7-v0", "Empty-5x5-v0",
                                    "GoToDoor-8x8-v0"])
def test_rollout_dense_random_states_vs_oracle(env_id):
    # imported random states (keys, balls, boxes, doors of every state near the
    # agent): pickups, drops and toggles change the grid mid-rollout, so the
    # rollout's cached transposed lines (odd directions) must be refreshed
    # exactly when the grid changes
    from paper_2407_19396_b200 import NavixEnv
    from inputgen import random_records
    n, K = 1500, 60
    g = NavixEnv(env_id, n, seed=12)
    o = OracleEnv(env_id, n, seed=12)
    s = g.spec
    recs = random_records(31, n, s.height, s.width, s.max_steps, 0, p_prev_done=0.02,
                          open_edge=env_id.startswith("GoToDoor"))
    g.import_state(recs)
    o.import_(recs)
    acts = random_actions(13, K, n, 0, high=7)
    ro, rr, rte, rtr = g.rollout(torch.from_numpy(acts).cuda())
    for t in range(K):
        oo, orw, ote, otr = o.step(acts[t])
        assert np.array_equal(ro[t].cpu().numpy(), oo), t
        assert np.array_equal(rr[t].cpu().numpy().view(np.uint32), orw.view(np.uint32))
        assert np.array_equal(rte[t].cpu().numpy(), ote) and np.array_equal(rtr[t].cpu().numpy(), otr)
    assert np.array_equal(g.export_state(), o.export())
