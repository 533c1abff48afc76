"""Memory-safety evidence in place of compute-sanitizer (closed on this pool;
SURVEY §4 item 6, SPEC's schedule-independence property).

Every output buffer lives inside a larger allocation whose guard bytes before
and after it are poisoned with 0xA5, and the output region itself is poisoned
again before EVERY call.  After each call: no guard byte changed (no
out-of-bounds write), and the output equals the oracle's (every byte was
written: 0xA5 is not a legal obs byte, flag or reward in these envs).  The
caller-owned state buffer gets guards too.  Cases: tiny batches, ragged tails,
unaligned obs bases (plain-store path), wide grids (one-tile kernel), the
persistent kernel, the fused rollout, categorical obs, observe_full."""
import numpy as np
import pytest
import torch

from inputgen import random_actions
from oracle import OracleEnv

pytestmark = pytest.mark.gpu
POISON = 0xA5
G = 4096  # guard bytes on each side


class Guarded:
    """A [G | region | G] uint8 allocation; `view` is the region (offset `off`)."""

    def __init__(self, nbytes, off=0, align=1):
        self.buf = torch.full((G + off + nbytes + G,), POISON, dtype=torch.uint8, device="cuda")
        self.lo, self.nbytes = G + off, nbytes
        assert (self.buf.data_ptr() + self.lo) % align == 0

    def region(self):
        return self.buf[self.lo:self.lo + self.nbytes]

    def poison(self):
        self.region().fill_(POISON)

    def guards_intact(self):
        b = self.buf
        return bool((b[:self.lo] == POISON).all()) and bool((b[self.lo + self.nbytes:] == POISON).all())


def _outputs(n, obs_per, off):
    obs = Guarded(n * obs_per, off)
    rew = Guarded(4 * n, 0, 4)
    te, tr = Guarded(n), Guarded(n)
    views = (obs.region().view(n, *((7, 7, 3) if obs_per == 147 else (7, 7))),
             rew.region().view(torch.float32), te.region(), tr.region())
    return [obs, rew, te, tr], views


CASES = [("DoorKey-8x8-v0", 1, 0), ("DoorKey-8x8-v0", 7, 1), ("DoorKey-8x8-v0", 129, 3),
         ("DoorKey-8x8-v0", 333, 16), ("DoorKey-8x8-v0", 1280, 0), ("Dynamic-Obstacles-8x8-v0", 333, 2),
         ("KeyCorridorS3R3-v0", 260, 0), ("DoorKey-16x16-v0", 200, 5), ("FourRooms-v0", 131, 0),
         ("KeyCorridorS6R3-v0", 129, 0), ("GoToDoor-8x8-v0", 200, 1), ("DistShift1-v0", 257, 0)]


@pytest.mark.parametrize("env_id,n,off", CASES)
def test_step_writes_exactly_its_outputs(env_id, n, off):
    from paper_2407_19396_b200 import NavixEnv, state_bytes
    sb = state_bytes(env_id, n)
    state = Guarded(sb, 0, 256)
    g = NavixEnv(env_id, n, seed=3, state=state.region())
    o = OracleEnv(env_id, n, seed=3)
    bufs, (obs, rew, te, tr) = _outputs(n, 147, off)
    bufs[0].poison()
    g.reset(out=obs)
    np.testing.assert_array_equal(obs.cpu().numpy(), o.reset())
    acts = random_actions(8, 60, n, o.spec.n_actions)
    for t in range(60):
        for b in bufs:
            b.poison()
        g.step(torch.from_numpy(acts[t]).cuda(), out=(obs, rew, te, tr))
        oo, orw, ote, otr = o.step(acts[t])
        torch.cuda.synchronize()
        assert all(b.guards_intact() for b in bufs), f"guard byte overwritten at step {t}"
        assert state.guards_intact(), f"state guard overwritten at step {t}"
        np.testing.assert_array_equal(obs.cpu().numpy(), oo, err_msg=f"obs step {t}")
        np.testing.assert_array_equal(rew.cpu().numpy().view(np.uint32), orw.view(np.uint32))
        np.testing.assert_array_equal(te.cpu().numpy(), ote)
        np.testing.assert_array_equal(tr.cpu().numpy(), otr)
    # observe and the full-grid obs write exactly their records too
    ob = Guarded(n * 147, off)
    g.observe(out=ob.region().view(n, 7, 7, 3))
    torch.cuda.synchronize()
    assert ob.guards_intact()
    np.testing.assert_array_equal(ob.region().view(n, 7, 7, 3).cpu().numpy(), o.observe())
    s = g.spec
    fb = Guarded(n * s.width * s.height * 3, off)
    g.observe_full(out=fb.region().view(n, s.width, s.height, 3))
    torch.cuda.synchronize()
    assert fb.guards_intact()
    np.testing.assert_array_equal(fb.region().view(n, s.width, s.height, 3).cpu().numpy(), o.observe_full())


@pytest.mark.parametrize("env_id,n,off", [("DoorKey-8x8-v0", 333, 0), ("DoorKey-8x8-v0", 129, 7),
                                          ("Dynamic-Obstacles-8x8-v0", 256, 0), ("KeyCorridorS4R3-v0", 150, 2)])
def test_rollout_writes_exactly_its_outputs(env_id, n, off):
    from paper_2407_19396_b200 import NavixEnv
    K = 6
    g = NavixEnv(env_id, n, seed=5)
    o = OracleEnv(env_id, n, seed=5)
    g.reset()
    o.reset()
    acts = random_actions(2, K, n, o.spec.n_actions)
    obs = Guarded(K * n * 147, off)
    rew, te, tr = Guarded(4 * K * n, 0, 4), Guarded(K * n), Guarded(K * n)
    out = (obs.region().view(K, n, 7, 7, 3), rew.region().view(torch.float32).view(K, n),
           te.region().view(K, n), tr.region().view(K, n))
    g.rollout(torch.from_numpy(acts).cuda(), out=out)
    torch.cuda.synchronize()
    assert all(b.guards_intact() for b in (obs, rew, te, tr))
    for t in range(K):
        oo, orw, ote, otr = o.step(acts[t])
        np.testing.assert_array_equal(out[0][t].cpu().numpy(), oo, err_msg=f"rollout obs {t}")
        np.testing.assert_array_equal(out[1][t].cpu().numpy().view(np.uint32), orw.view(np.uint32))
        np.testing.assert_array_equal(out[2][t].cpu().numpy(), ote)
        np.testing.assert_array_equal(out[3][t].cpu().numpy(), otr)
    np.testing.assert_array_equal(g.export_state(), o.export())


@pytest.mark.parametrize("n,off", [(333, 1), (128, 0)])
def test_categorical_step_writes_exactly_its_outputs(n, off):
    from paper_2407_19396_b200 import NavixEnv
    g = NavixEnv("DoorKey-8x8-v0", n, seed=6, observation="categorical")
    o = OracleEnv("DoorKey-8x8-v0", n, seed=6)
    bufs, (obs, rew, te, tr) = _outputs(n, 49, off)
    g.reset(out=obs)
    o.reset()
    acts = random_actions(9, 20, n, 7)
    for t in range(20):
        for b in bufs:
            b.poison()
        g.step(torch.from_numpy(acts[t]).cuda(), out=(obs, rew, te, tr))
        oo, *_ = o.step(acts[t])
        torch.cuda.synchronize()
        assert all(b.guards_intact() for b in bufs)
        np.testing.assert_array_equal(obs.cpu().numpy(), oo[:, :, :, 0])


@pytest.mark.parametrize("env_id", ["DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0", "KeyCorridorS3R3-v0",
                                    "LavaGapS7-v0", "GoToDoor-8x8-v0", "DoorKey-16x16-v0", "FourRooms-v0"])
@pytest.mark.parametrize("n", [200, 3000])
def test_garbage_in_padding_slots(env_id, n):
    # a caller-owned state buffer starts as random bytes: the padding slots of
    # the last tile (never written) must not steer any kernel out of bounds
    from paper_2407_19396_b200 import NavixEnv, state_bytes
    sb = state_bytes(env_id, n)
    state = Guarded(sb, 0, 256)
    state.region().copy_(torch.randint(0, 256, (sb,), dtype=torch.uint8, device="cuda"))
    g = NavixEnv(env_id, n, seed=9, state=state.region())
    o = OracleEnv(env_id, n, seed=9)
    np.testing.assert_array_equal(g.reset().cpu().numpy(), o.reset())
    acts = random_actions(3, 30, n, o.spec.n_actions)
    for t in range(20):
        go, *_ = g.step(torch.from_numpy(acts[t]).cuda())
        oo, *_ = o.step(acts[t])
        np.testing.assert_array_equal(go.cpu().numpy(), oo, err_msg=f"step {t}")
    np.testing.assert_array_equal(g.observe().cpu().numpy(), o.observe())
    np.testing.assert_array_equal(g.observe_full().cpu().numpy(), o.observe_full())
    ro = g.rollout(torch.from_numpy(acts[20:30]).cuda())[0]
    for t in range(10):
        np.testing.assert_array_equal(ro[t].cpu().numpy(), o.step(acts[20 + t])[0])
    torch.cuda.synchronize()
    assert state.guards_intact()
