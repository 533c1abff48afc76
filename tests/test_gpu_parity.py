"""GPU <-> oracle parity through the C ABI (libnavix.so), bit-exact.

Every output of every step (observation bytes, reward bits, terminated,
truncated) and the canonical state export are compared with the CPU oracle
on identical seeded inputs (inputgen: numpy PCG64 actions, fed to both
sides).  Full-batch comparison for the small configs of BASELINE.json; for
the large configs the GPU runs the full batch in the bench's launch
configuration and the oracle recomputes contiguous blocks of envs spread over
the batch (head, middle, ragged tail), which it can afford one by one.
"""
import numpy as np
import pytest
import torch

from inputgen import random_actions
from oracle import OracleEnv, sample_actions as oracle_sample_actions

pytestmark = pytest.mark.gpu


def navix():
    from paper_2407_19396_b200 import NavixEnv
    return NavixEnv


def _blocks(n, block):
    if n <= 4 * block:
        return [(0, n)]
    mid = (n // 2) // 128 * 128 + 37
    return [(0, block), (mid, mid + block), (n - block, n)]


def run_parity(env_id, n, steps, seed=0, action_seed=1, block=128, reward_mode=0, export_every=50):
    NavixEnv = navix()
    g = NavixEnv(env_id, n, seed=seed, reward_mode=reward_mode)
    blocks = _blocks(n, block)
    oracles = [OracleEnv(env_id, e - b, seed=seed, env_begin=b, num_envs_total=n, reward_mode=reward_mode)
               for b, e in blocks]
    idx = torch.cat([torch.arange(b, e) for b, e in blocks]).cuda()
    obs = g.reset()
    o_obs = np.concatenate([o.reset() for o in oracles])
    np.testing.assert_array_equal(obs[idx].cpu().numpy(), o_obs)
    acts = random_actions(action_seed, steps, n, g.spec.n_actions, high=8)  # 8: includes out-of-range 7
    acts_dev = torch.from_numpy(acts).cuda()
    for t in range(steps):
        obs, rew, te, tr = g.step(acts_dev[t])
        outs = [o.step(acts[t, b:e]) for o, (b, e) in zip(oracles, blocks)]
        o_obs = np.concatenate([x[0] for x in outs])
        o_rew = np.concatenate([x[1] for x in outs])
        o_te = np.concatenate([x[2] for x in outs])
        o_tr = np.concatenate([x[3] for x in outs])
        got_obs = obs[idx].cpu().numpy()
        if not np.array_equal(got_obs, o_obs):
            bad = np.argwhere((got_obs != o_obs).reshape(len(o_obs), -1).any(1))[:, 0]
            raise AssertionError(f"{env_id} step {t}: obs differ for {len(bad)} envs, first local {bad[:5]}")
        np.testing.assert_array_equal(rew[idx].cpu().numpy().view(np.uint32), o_rew.view(np.uint32),
                                      err_msg=f"reward bits step {t}")
        np.testing.assert_array_equal(te[idx].cpu().numpy(), o_te, err_msg=f"terminated step {t}")
        np.testing.assert_array_equal(tr[idx].cpu().numpy(), o_tr, err_msg=f"truncated step {t}")
        if (t + 1) % export_every == 0 or t == steps - 1:
            rec = g.export_state()
            o_rec = np.concatenate([o.export() for o in oracles])
            np.testing.assert_array_equal(rec[idx.cpu().numpy()], o_rec, err_msg=f"state step {t}")
    if len(blocks) == 1 and blocks[0] == (0, n):
        np.testing.assert_array_equal(g.stats().cpu().numpy(), oracles[0].stats())
    return g


def test_parity_cfg1_empty5x5_16_envs_1000_steps():
    run_parity("Empty-5x5-v0", 16, 1000, export_every=1)


@pytest.mark.parametrize("env_id", ["Empty-8x8-v0", "DoorKey-8x8-v0"])
def test_parity_cfg2_2048_envs_1000_steps(env_id):
    run_parity(env_id, 2048, 1000, block=2048)


def test_parity_cfg3_dynobs_65536():
    run_parity("Dynamic-Obstacles-8x8-v0", 65536, 1000, block=128)


@pytest.mark.parametrize("env_id", ["KeyCorridorS3R3-v0", "LavaGapS7-v0"])
def test_parity_cfg4_262144(env_id):
    run_parity(env_id, 262144, 600, block=128)


def test_parity_cfg5_doorkey_1M_sampled():
    run_parity("DoorKey-8x8-v0", 1 << 20, 300, block=96, export_every=100)


@pytest.mark.parametrize("env_id", ["DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0"])
def test_parity_max_size_ragged_sampled(env_id):
    # [CFG 5]'s largest size, 2^23 envs per GPU, plus a ragged tail of 77:
    # head, middle and tail blocks against the oracle, the state at the end
    run_parity(env_id, (1 << 23) + 77, 40, block=96, export_every=1000)


@pytest.mark.parametrize("env_id", ["Empty-6x6-v0", "DoorKey-5x5-v0", "DoorKey-6x6-v0",
                                    "Dynamic-Obstacles-5x5-v0", "Dynamic-Obstacles-6x6-v0",
                                    "LavaGapS5-v0", "LavaGapS6-v0", "KeyCorridorS3R1-v0",
                                    "KeyCorridorS3R2-v0"])
def test_parity_other_sizes_ragged(env_id):
    # 333 envs: two full tiles and a ragged tail of 77 (plain-store path)
    run_parity(env_id, 333, 400, block=333, seed=5)


@pytest.mark.parametrize("env_id", ["Empty-16x16-v0", "DoorKey-16x16-v0", "Dynamic-Obstacles-16x16-v0",
                                    "KeyCorridorS4R3-v0", "KeyCorridorS5R3-v0", "KeyCorridorS6R3-v0"])
def test_parity_row_f2_wide_grids(env_id):
    # grids up to 16x16 (16-byte rows, one tile per CTA): 4 full tiles + a ragged tail
    run_parity(env_id, 555, 500, block=555, seed=12)


@pytest.mark.parametrize("env_id", ["DoorKey-8x8-v0", "LavaGapS7-v0", "Dynamic-Obstacles-8x8-v0",
                                    "GoToDoor-8x8-v0", "GoToDoor-5x5-v0"])
def test_parity_reward_mode_navix(env_id):
    run_parity(env_id, 512, 300, block=512, reward_mode=1, seed=9)


@pytest.mark.parametrize("n", [1, 7, 128, 129])
def test_parity_tiny_batches(n):
    run_parity("DoorKey-8x8-v0", n, 200, block=n, seed=2)


def test_sample_actions_matches_oracle():
    NavixEnv = navix()
    for env_id in ("DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0"):
        g = NavixEnv(env_id, 1000, env_begin=3000, num_envs_total=10000)
        a = g.sample_actions(12345, 77, 20).cpu().numpy()
        b = oracle_sample_actions(12345, 3000, 1000, 77, 20, g.spec.n_actions)
        np.testing.assert_array_equal(a, b)


def test_shard_invariance_and_determinism():
    NavixEnv = navix()
    n, steps, G = 1000, 300, 4
    env_id = "KeyCorridorS3R3-v0"
    full = NavixEnv(env_id, n, seed=11)
    full.reset()
    acts = torch.from_numpy(random_actions(3, steps, n, 7)).cuda()
    bounds = [(r * n // G, (r + 1) * n // G) for r in range(G)]
    shards = [NavixEnv(env_id, e - b, seed=11, env_begin=b, num_envs_total=n) for b, e in bounds]
    for s in shards:
        s.reset()
    again = NavixEnv(env_id, n, seed=11)
    again.reset()
    for t in range(steps):
        o, r, te, tr = [x.clone() for x in full.step(acts[t])]
        o2, r2, te2, tr2 = again.step(acts[t])
        assert torch.equal(o, o2) and torch.equal(r, r2) and torch.equal(te, te2) and torch.equal(tr, tr2)
        for s, (b, e) in zip(shards, bounds):
            so, sr, ste, str_ = s.step(acts[t, b:e].contiguous())
            assert torch.equal(so, o[b:e]) and torch.equal(sr, r[b:e])
            assert torch.equal(ste, te[b:e]) and torch.equal(str_, tr[b:e])
    tot = sum(s.stats().cpu() for s in shards)
    assert torch.equal(tot, full.stats().cpu())
    assert np.array_equal(np.concatenate([s.export_state() for s in shards]), full.export_state())


def test_step_host_matches_device_path():
    NavixEnv = navix()
    n = 300
    a = NavixEnv("DoorKey-8x8-v0", n, seed=4)
    b = NavixEnv("DoorKey-8x8-v0", n, seed=4)
    a.reset()
    b.reset()
    acts = random_actions(8, 50, n, 7)
    h_obs = torch.empty((n, 7, 7, 3), dtype=torch.uint8).pin_memory()
    h_rew = torch.empty(n, dtype=torch.float32).pin_memory()
    h_te = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_tr = torch.empty(n, dtype=torch.uint8).pin_memory()
    for t in range(50):
        ha = torch.from_numpy(acts[t]).pin_memory()
        a.step_host(ha, h_obs, h_rew, h_te, h_tr)
        o, r, te, tr = b.step(ha.cuda())
        assert torch.equal(h_obs, o.cpu()) and torch.equal(h_rew, r.cpu())
        assert torch.equal(h_te, te.cpu()) and torch.equal(h_tr, tr.cpu())


def test_unaligned_obs_buffer_uses_plain_stores():
    NavixEnv = navix()
    n = 256
    a = NavixEnv("LavaGapS7-v0", n, seed=6)
    b = NavixEnv("LavaGapS7-v0", n, seed=6)
    big = torch.empty(n * 147 + 1, dtype=torch.uint8, device="cuda")
    view = big[1:].view(n, 7, 7, 3)  # 1-byte offset: not 16-byte aligned
    a.reset(out=view)
    ref = b.reset()
    assert torch.equal(view, ref)
    acts = torch.from_numpy(random_actions(2, 30, n, 7)).cuda()
    for t in range(30):
        out = (view, torch.empty(n, device="cuda"), torch.empty(n, dtype=torch.uint8, device="cuda"),
               torch.empty(n, dtype=torch.uint8, device="cuda"))
        a.step(acts[t], out=out)
        ro = b.step(acts[t])[0]
        assert torch.equal(view, ro)


def test_cuda_graph_replay_matches_eager():
    """The bench times CUDA-graph replays of the persistent step kernel (its
    tile scheduler resets itself at the end of every launch)."""
    NavixEnv = navix()
    n, K = 5000, 40
    a = NavixEnv("DoorKey-8x8-v0", n, seed=3)
    b = NavixEnv("DoorKey-8x8-v0", n, seed=3)
    a.reset()
    b.reset()
    acts = a.sample_actions(1, 0, K)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for t in range(K):
            a.step(acts[t])
    for rep in range(3):  # capture does not execute; replay 3 times = 3*K steps
        graph.replay()
        for t in range(K):
            b.step(acts[t])
        torch.cuda.synchronize()
        assert np.array_equal(a.export_state(), b.export_state()), rep
    assert torch.equal(a.obs, b.obs) and torch.equal(a.reward, b.reward)
    assert torch.equal(a.stats(), b.stats())


@pytest.mark.parametrize("env_id", ["Empty-Random-5x5-v0", "Empty-Random-6x6-v0", "Empty-Random-8x8-v0",
                                    "Empty-Random-16x16-v0", "DistShift1-v0", "DistShift2-v0",
                                    "SimpleCrossingS9N1-v0", "SimpleCrossingS9N2-v0", "SimpleCrossingS9N3-v0",
                                    "SimpleCrossingS11N5-v0", "DoorKey-Random-8x8", "GoToDoor-5x5-v0",
                                    "GoToDoor-6x6-v0", "GoToDoor-8x8-v0", "FourRooms-v0",
                                    "Dynamic-Obstacles-Random-5x5", "Dynamic-Obstacles-Random-6x6",
                                    "Navix-Crossings-S9N1-v0", "Navix-Crossings-S9N2-v0", "Navix-Crossings-S9N3-v0",
                                    "Navix-Crossings-S11N5-v0", "Navix-LavaGap-S7-v0"])
def test_parity_row_f2_more_families(env_id):
    # Empty-Random (random start cell + direction per episode) and DistShift (9x7, lava strips)
    run_parity(env_id, 555, 600, block=555, seed=21)


def test_reset_seed_equals_fresh_handle():
    # reset(key) with a new key: same as a handle created with that seed
    NavixEnv = navix()
    n = 777
    a = NavixEnv("KeyCorridorS3R3-v0", n, seed=1)
    b = NavixEnv("KeyCorridorS3R3-v0", n, seed=99)
    o = OracleEnv("KeyCorridorS3R3-v0", n, seed=99)
    a.reset()
    a.step(torch.zeros(n, dtype=torch.uint8, device="cuda"))
    ga = a.reset_seed(99).clone()
    assert torch.equal(ga, b.reset())
    np.testing.assert_array_equal(ga.cpu().numpy(), o.reset())
    acts = random_actions(5, 300, n, 7)
    for t in range(300):
        oa = a.step(torch.from_numpy(acts[t]).cuda())[0].clone()
        ob = b.step(torch.from_numpy(acts[t]).cuda())[0]
        assert torch.equal(oa, ob), t
    np.testing.assert_array_equal(a.export_state(), b.export_state())
    assert torch.equal(a.stats(), b.stats())


def test_step_before_reset_is_an_error():
    from paper_2407_19396_b200 import NavixError
    NavixEnv = navix()
    g = NavixEnv("DoorKey-8x8-v0", 100)
    with pytest.raises(NavixError) as e:
        g.step(torch.zeros(100, dtype=torch.uint8, device="cuda"))
    assert "navix_reset" in str(e.value)
    g.reset()
    g.step(torch.zeros(100, dtype=torch.uint8, device="cuda"))


def test_caller_owned_state_buffer():
    # navix_create_shard(state_dev = a caller-owned torch buffer of navix_state_bytes)
    from paper_2407_19396_b200 import state_bytes
    NavixEnv = navix()
    n = 1000
    buf = torch.empty(state_bytes("DoorKey-8x8-v0", n), dtype=torch.uint8, device="cuda")
    a = NavixEnv("DoorKey-8x8-v0", n, seed=3, state=buf)
    b = NavixEnv("DoorKey-8x8-v0", n, seed=3)
    assert torch.equal(a.reset(), b.reset())
    acts = torch.from_numpy(random_actions(2, 50, n, 7)).cuda()
    for t in range(50):
        oa = a.step(acts[t])[0].clone()
        assert torch.equal(oa, b.step(acts[t])[0]), t
    np.testing.assert_array_equal(a.export_state(), b.export_state())
    a.close()
    assert buf.numel() == state_bytes("DoorKey-8x8-v0", n)  # still owned (not freed) by the caller


@pytest.mark.parametrize("env_id", ["KeyCorridorS3R3-v0", "Dynamic-Obstacles-8x8-v0", "GoToDoor-8x8-v0",
                                    "DistShift1-v0", "SimpleCrossingS11N5-v0", "LavaGapS7-v0"])
def test_parity_dynamic_scheduler_sampled(env_id):
    # > 4 tiles per CTA: the atomic tile scheduler (and, for KeyCorridor, the
    # reset-first tile lists) at full scale, 300 steps (KeyCorridor truncates
    # everyone at 270), sampled blocks against the oracle
    run_parity(env_id, (1 << 20) + 77, 300, block=96, export_every=100, seed=2)


@pytest.mark.parametrize("env_id", ["KeyCorridorS3R3-v0", "DoorKey-8x8-v0"])
def test_cuda_graph_replay_dynamic_scheduler(env_id):
    # graph replays of the persistent kernel in its dynamic-scheduler regime
    # (epoch-stamped reset-first lists for KeyCorridor) equal eager launches
    NavixEnv = navix()
    n, K = (1 << 19) + 1000, 100
    a = NavixEnv(env_id, n, seed=5)
    b = NavixEnv(env_id, n, seed=5)
    a.reset()
    b.reset()
    acts = a.sample_actions(1, 0, K)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for t in range(K):
            a.step(acts[t])
    for rep in range(3):  # 300 steps: includes KeyCorridor's truncation at 270
        graph.replay()
        for t in range(K):
            b.step(acts[t])
        torch.cuda.synchronize()
        assert torch.equal(a.obs, b.obs) and torch.equal(a.reward, b.reward), rep
    assert np.array_equal(a.export_state(), b.export_state())
    assert torch.equal(a.stats(), b.stats())


def test_side_stream_and_graph_on_side_stream():
    # every call enqueues on torch's current stream: a side stream gives the
    # same results as the default one
    NavixEnv = navix()
    n = 3000
    a = NavixEnv("LavaGapS7-v0", n, seed=8)
    b = NavixEnv("LavaGapS7-v0", n, seed=8)
    acts = torch.from_numpy(random_actions(6, 60, n, 7)).cuda()
    a.reset()
    for t in range(60):
        a.step(acts[t])
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        b.reset()
        for t in range(60):
            b.step(acts[t])
        ob = b.obs.clone()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    assert torch.equal(a.obs, ob)
    np.testing.assert_array_equal(a.export_state(), b.export_state())
