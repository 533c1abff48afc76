"""The small-batch kernel (navix_step_wide): 8 lanes per env,
observation split by view column.  Bit-exact against the oracle and against
the one-thread-per-env persistent kernel on the same handle state, for every
family it serves, ragged env counts (a CTA holds 16 envs), both observation
kinds, unaligned outputs (the byte-copy path), dense random imported states
(doors, keys, boxes, pickups / drops / toggles mid-batch) and auto-resets
(Dynamic-Obstacles' in-loop level generation and -Random's generator call)."""
import zlib

import numpy as np
import pytest
import torch

from inputgen import random_actions, random_records
from oracle import OracleEnv

pytestmark = pytest.mark.gpu

IDS = ["Empty-5x5-v0", "Empty-8x8-v0", "DoorKey-8x8-v0", "DoorKey-5x5-v0", "Dynamic-Obstacles-8x8-v0",
       "Dynamic-Obstacles-5x5-v0", "Dynamic-Obstacles-Random-6x6", "KeyCorridorS3R3-v0", "KeyCorridorS3R1-v0",
       "LavaGapS7-v0", "Empty-Random-8x8"]


def _step_all(g, o, acts, *, obs_off=0, cat=False):
    n = g.n
    per = 49 if cat else 147
    buf = torch.zeros(obs_off + n * per, dtype=torch.uint8, device="cuda")
    obs = buf[obs_off:].view(n, 7, 7) if cat else buf[obs_off:].view(n, 7, 7, 3)
    rew = torch.empty(n, dtype=torch.float32, device="cuda")
    te = torch.empty(n, dtype=torch.uint8, device="cuda")
    tr = torch.empty(n, dtype=torch.uint8, device="cuda")
    for t in range(acts.shape[0]):
        g.step(torch.from_numpy(acts[t]).cuda(), out=(obs, rew, te, tr))
        oo, orw, ote, otr = o.step(acts[t])
        np.testing.assert_array_equal(obs.cpu().numpy(), oo[..., 0] if cat else oo, err_msg=f"obs step {t}")
        np.testing.assert_array_equal(rew.cpu().numpy().view(np.uint32), orw.view(np.uint32), err_msg=f"rew {t}")
        np.testing.assert_array_equal(te.cpu().numpy(), ote)
        np.testing.assert_array_equal(tr.cpu().numpy(), otr)


@pytest.mark.parametrize("env_id", IDS)
@pytest.mark.parametrize("n", [1, 17, 333])
def test_wide_kernel_vs_oracle(env_id, n):
    from paper_2407_19396_b200 import NavixEnv
    g = NavixEnv(env_id, n, seed=31)
    g.set_small_batch_threshold(1 << 30)  # force the small-batch kernel
    o = OracleEnv(env_id, n, seed=31)
    g.reset()
    o.reset()
    _step_all(g, o, random_actions(4, 300, n, 0, high=8))
    np.testing.assert_array_equal(g.export_state(), o.export())
    np.testing.assert_array_equal(g.stats().cpu().numpy(), o.stats())


@pytest.mark.parametrize("env_id", ["DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0", "KeyCorridorS3R3-v0"])
def test_wide_kernel_categorical_and_unaligned(env_id):
    from paper_2407_19396_b200 import NavixEnv
    n = 129
    for cat, off in ((True, 0), (False, 1), (True, 3)):
        g = NavixEnv(env_id, n, seed=5, observation="categorical" if cat else "symbolic")
        g.set_small_batch_threshold(1 << 30)
        o = OracleEnv(env_id, n, seed=5)
        g.reset()
        o.reset()
        _step_all(g, o, random_actions(6, 120, n, 0, high=8), obs_off=off, cat=cat)


@pytest.mark.parametrize("env_id,nob", [("DoorKey-8x8-v0", 0), ("KeyCorridorS3R3-v0", 0), ("LavaGapS7-v0", 0),
                                        ("Dynamic-Obstacles-8x8-v0", 4), ("Empty-5x5-v0", 0)])
def test_wide_kernel_random_states(env_id, nob):
    from paper_2407_19396_b200 import NavixEnv
    n = 1000
    g = NavixEnv(env_id, n, seed=21)
    g.set_small_batch_threshold(1 << 30)
    o = OracleEnv(env_id, n, seed=21)
    s = g.spec
    recs = random_records(zlib.crc32(env_id.encode()) % 997, n, s.height, s.width, s.max_steps, nob,
                          p_prev_done=0.05)
    g.import_state(recs)
    o.import_(recs)
    _step_all(g, o, random_actions(7, 12, n, 0, high=8))
    np.testing.assert_array_equal(g.export_state(), o.export())


@pytest.mark.parametrize("env_id", ["DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0", "KeyCorridorS3R3-v0"])
def test_wide_and_persistent_kernels_interleave(env_id):
    # switching kernels between steps of one handle: the state layout is shared
    from paper_2407_19396_b200 import NavixEnv
    n = 2048
    g = NavixEnv(env_id, n, seed=2)
    o = OracleEnv(env_id, n, seed=2)
    g.reset()
    o.reset()
    acts = random_actions(8, 90, n, 0, high=8)
    for k in range(3):
        g.set_small_batch_threshold(1 << 30 if k % 2 == 0 else 0)
        _step_all(g, o, acts[30 * k:30 * (k + 1)])
    np.testing.assert_array_equal(g.export_state(), o.export())


@pytest.mark.parametrize("env_id", IDS)
@pytest.mark.parametrize("n,K", [(17, 120), (333, 60)])
def test_wide_rollout_vs_oracle(env_id, n, K):
    # navix_rollout_wide: the state stays in SMEM / registers across K steps
    from paper_2407_19396_b200 import NavixEnv
    g = NavixEnv(env_id, n, seed=13)
    g.set_small_batch_threshold(1 << 30)
    o = OracleEnv(env_id, n, seed=13)
    g.reset()
    o.reset()
    acts = random_actions(9, 2 * K, n, 0, high=8)
    for half in range(2):  # two launches: the state is carried over in HBM
        ro, rr, rte, rtr = g.rollout(torch.from_numpy(acts[half * K:(half + 1) * K]).cuda())
        for t in range(K):
            oo, orw, ote, otr = o.step(acts[half * K + t])
            np.testing.assert_array_equal(ro[t].cpu().numpy(), oo, err_msg=f"rollout obs {half} {t}")
            np.testing.assert_array_equal(rr[t].cpu().numpy().view(np.uint32), orw.view(np.uint32))
            np.testing.assert_array_equal(rte[t].cpu().numpy(), ote)
            np.testing.assert_array_equal(rtr[t].cpu().numpy(), otr)
        np.testing.assert_array_equal(g.export_state(), o.export())
    np.testing.assert_array_equal(g.stats().cpu().numpy(), o.stats())


@pytest.mark.parametrize("env_id", ["DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0", "KeyCorridorS3R3-v0"])
def test_wide_rollout_random_categorical_and_tile_kernel(env_id):
    # the in-kernel policy and categorical obs on the small-batch rollout, and
    # the one-tile-per-CTA rollout kernel forced at the same size: all equal
    from paper_2407_19396_b200 import NavixEnv
    from oracle import sample_actions as oracle_sample_actions
    n, K = 300, 50
    a = NavixEnv(env_id, n, seed=3, observation="categorical")
    b = NavixEnv(env_id, n, seed=3, observation="categorical")
    a.set_small_batch_threshold(1 << 30)
    b.set_small_batch_threshold(0)
    o = OracleEnv(env_id, n, seed=3)
    a.reset()
    b.reset()
    o.reset()
    ra = a.rollout_random(21, 4, K)
    rb = b.rollout_random(21, 4, K)
    for x, y in zip(ra, rb):
        assert torch.equal(x, y)
    acts = oracle_sample_actions(21, 0, n, 4, K, o.spec.n_actions)
    for t in range(K):
        oo, orw, ote, otr = o.step(acts[t])
        np.testing.assert_array_equal(ra[0][t].cpu().numpy(), oo[..., 0])
        np.testing.assert_array_equal(ra[1][t].cpu().numpy().view(np.uint32), orw.view(np.uint32))
    np.testing.assert_array_equal(a.export_state(), o.export())
    np.testing.assert_array_equal(b.export_state(), o.export())
