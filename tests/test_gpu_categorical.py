"""GPU <-> oracle parity of the categorical observations (row f3; Table 5
`categorical` / `categorical_first_person`; R#41): the
49-byte first-person record and the W x H full grid are the entity-type
channel of the oracle's symbolic observations, byte for byte, on every path
that emits observations (reset, step incl. auto-reset, observe, rollout,
step_host, observe_full)."""
import numpy as np
import pytest
import torch

from inputgen import random_actions
from oracle import OracleEnv

pytestmark = pytest.mark.gpu

ENVS = ["DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0", "KeyCorridorS3R3-v0", "LavaGapS7-v0", "Empty-5x5-v0",
        "GoToDoor-8x8-v0", "Empty-16x16-v0", "DistShift2-v0", "FourRooms-v0", "SimpleCrossingS11N5-v0"]


@pytest.mark.parametrize("env_id", ENVS)
@pytest.mark.parametrize("n", [333, 1024])
def test_categorical_step_parity(env_id, n):
    from paper_2407_19396_b200 import NavixEnv
    g = NavixEnv(env_id, n, seed=6, observation="categorical")
    o = OracleEnv(env_id, n, seed=6)
    assert g.reset().shape == (n, 7, 7)
    np.testing.assert_array_equal(g.obs.cpu().numpy(), o.reset()[..., 0])
    acts = random_actions(3, 200, n, 0, high=8)
    for t in range(200):
        go, gr, gte, gtr = g.step(torch.from_numpy(acts[t]).cuda())
        oo, orw, ote, otr = o.step(acts[t])
        np.testing.assert_array_equal(go.cpu().numpy(), oo[..., 0], err_msg=f"step {t}")
        np.testing.assert_array_equal(gr.cpu().numpy().view(np.uint32), orw.view(np.uint32))
        np.testing.assert_array_equal(gte.cpu().numpy(), ote)
        np.testing.assert_array_equal(gtr.cpu().numpy(), otr)
    np.testing.assert_array_equal(g.observe().cpu().numpy(), o.observe()[..., 0])
    full = g.observe_full().cpu().numpy()
    s = g.spec
    assert full.shape == (n, s.width, s.height)
    np.testing.assert_array_equal(full, o.observe_full()[..., 0])
    np.testing.assert_array_equal(g.export_state(), o.export())


@pytest.mark.parametrize("env_id", ["DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0", "DoorKey-16x16-v0", "FourRooms-v0"])
def test_categorical_rollout_and_step_host(env_id):
    from paper_2407_19396_b200 import NavixEnv
    n, K = 700, 40
    a = NavixEnv(env_id, n, seed=8, observation="categorical")
    b = NavixEnv(env_id, n, seed=8, observation="categorical")
    c = NavixEnv(env_id, n, seed=8, observation="categorical")
    a.reset()
    b.reset()
    c.reset()
    acts = torch.from_numpy(random_actions(4, K, n, 0, high=8)).cuda()
    ro, rr, rte, rtr = a.rollout(acts)
    assert ro.shape == (K, n, 7, 7)
    h_obs = torch.empty((n, 7, 7), dtype=torch.uint8).pin_memory()
    h_rew = torch.empty(n, dtype=torch.float32).pin_memory()
    h_te = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_tr = torch.empty(n, dtype=torch.uint8).pin_memory()
    for t in range(K):
        go, gr, gte, gtr = b.step(acts[t])
        assert torch.equal(ro[t], go) and torch.equal(rr[t], gr) and torch.equal(rte[t], gte)
        c.step_host(acts[t].cpu().contiguous(), h_obs, h_rew, h_te, h_tr)
        assert torch.equal(h_obs, go.cpu()) and torch.equal(h_rew, gr.cpu())
    np.testing.assert_array_equal(a.export_state(), b.export_state())


def test_switching_kind_keeps_the_state():
    from paper_2407_19396_b200 import NavixEnv
    n = 300
    g = NavixEnv("KeyCorridorS3R3-v0", n, seed=1)
    o = OracleEnv("KeyCorridorS3R3-v0", n, seed=1)
    g.reset()
    o.reset()
    acts = random_actions(2, 30, n, 7)
    for t in range(30):
        g.step(torch.from_numpy(acts[t]).cuda())
        o.step(acts[t])
    cat = torch.empty((n, 7, 7), dtype=torch.uint8, device="cuda")
    g.lib.navix_set_observation(g.h, 1)
    g.obs_shape = (7, 7)
    g.observe(out=cat)
    np.testing.assert_array_equal(cat.cpu().numpy(), o.observe()[..., 0])
