"""Direct GPU <-> oracle parity for the paths earlier compared GPU-vs-GPU only
(VERDICT r1 "chain of equality"): the in-kernel random policy of
navix_rollout_random against the ORACLE stepping the oracle's own,
independently written action stream (oracle.sample_actions, R#20 domain 2),
and the categorical rollout / step_host against the oracle's type channel —
one env of every family group (inst_*.cu)."""
import numpy as np
import pytest
import torch

from oracle import OracleEnv
from oracle import sample_actions as oracle_sample_actions

pytestmark = pytest.mark.gpu

GROUPS = [("Empty-Random-8x8", 300, 80, 0), ("DoorKey-8x8-v0", 1000, 60, 11), ("DoorKey-16x16-v0", 200, 40, 3),
          ("Dynamic-Obstacles-8x8-v0", 513, 60, 7), ("Dynamic-Obstacles-16x16-v0", 200, 40, 0),
          ("KeyCorridorS3R3-v0", 300, 60, 123), ("KeyCorridorS5R3-v0", 150, 30, 9), ("LavaGapS7-v0", 400, 60, 2),
          ("Crossings-S9N2-v0", 300, 50, 4), ("DistShift2-v0", 300, 50, 1), ("GoToDoor-6x6-v0", 300, 50, 5),
          ("FourRooms-v0", 200, 40, 5)]


@pytest.mark.parametrize("env_id,n,K,t0", GROUPS)
def test_rollout_random_vs_oracle(env_id, n, K, t0):
    from paper_2407_19396_b200 import NavixEnv
    seed, aseed, begin, total = 4, 77, 1000, 100000
    g = NavixEnv(env_id, n, seed=seed, env_begin=begin, num_envs_total=total)
    o = OracleEnv(env_id, n, seed=seed, env_begin=begin, num_envs_total=total)
    g.reset()
    o.reset()
    ro, rr, rte, rtr = g.rollout_random(aseed, t0, K)
    acts = oracle_sample_actions(aseed, begin, n, t0, K, o.spec.n_actions)  # the oracle's own stream
    for t in range(K):
        oo, orw, ote, otr = o.step(acts[t])
        np.testing.assert_array_equal(ro[t].cpu().numpy(), oo, err_msg=f"obs step {t}")
        np.testing.assert_array_equal(rr[t].cpu().numpy().view(np.uint32), orw.view(np.uint32))
        np.testing.assert_array_equal(rte[t].cpu().numpy(), ote)
        np.testing.assert_array_equal(rtr[t].cpu().numpy(), otr)
    np.testing.assert_array_equal(g.export_state(), o.export())
    np.testing.assert_array_equal(g.stats().cpu().numpy(), o.stats())


@pytest.mark.parametrize("env_id", ["DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0", "KeyCorridorS3R3-v0",
                                    "DoorKey-16x16-v0", "FourRooms-v0", "GoToDoor-8x8-v0"])
def test_categorical_rollout_and_step_host_vs_oracle(env_id):
    from paper_2407_19396_b200 import NavixEnv
    n, K = 333, 30
    a = NavixEnv(env_id, n, seed=8, observation="categorical")
    c = NavixEnv(env_id, n, seed=8, observation="categorical")
    o = OracleEnv(env_id, n, seed=8)
    a.reset()
    c.reset()
    o.reset()
    acts = oracle_sample_actions(5, 0, n, 0, K, o.spec.n_actions)
    ro, rr, rte, rtr = a.rollout(torch.from_numpy(acts).cuda())
    h_obs = torch.empty((n, 7, 7), dtype=torch.uint8).pin_memory()
    h_rew = torch.empty(n, dtype=torch.float32).pin_memory()
    h_te = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_tr = torch.empty(n, dtype=torch.uint8).pin_memory()
    for t in range(K):
        oo, orw, ote, otr = o.step(acts[t])
        np.testing.assert_array_equal(ro[t].cpu().numpy(), oo[..., 0], err_msg=f"rollout step {t}")
        np.testing.assert_array_equal(rr[t].cpu().numpy().view(np.uint32), orw.view(np.uint32))
        np.testing.assert_array_equal(rte[t].cpu().numpy(), ote)
        c.step_host(torch.from_numpy(acts[t]), h_obs, h_rew, h_te, h_tr)
        np.testing.assert_array_equal(h_obs.numpy(), oo[..., 0], err_msg=f"step_host step {t}")
        np.testing.assert_array_equal(h_rew.numpy().view(np.uint32), orw.view(np.uint32))
        np.testing.assert_array_equal(h_te.numpy(), ote)
        np.testing.assert_array_equal(h_tr.numpy(), otr)
    np.testing.assert_array_equal(a.export_state(), o.export())
    np.testing.assert_array_equal(c.export_state(), o.export())
