"""P3 on the GPU: every length-8 action sequence on Empty-5x5, one lane each
(7^8 = 5,764,801 lanes through the C ABI in one batch).

Pins: the number of lanes terminating at step L equals count(L) * 7^(8-L),
count(L) from the independent 36-state DP (test_oracle_bruteforce.py /
tests/golden/p3_*.json); every terminating lane's reward is the pinned
Eq. (1) value for L; no lane terminates twice; and a strided sample of lanes
matches the oracle's full outputs byte for byte at every step.
"""
import numpy as np
import pytest
import torch

from oracle import OracleEnv, success_reward
from test_oracle_bruteforce import dp_first_goal_counts

pytestmark = pytest.mark.gpu


def test_gpu_bruteforce_empty5_all_length8_sequences():
    from paper_2407_19396_b200 import NavixEnv
    L_MAX = 8
    n = 7 ** L_MAX
    g = NavixEnv("Empty-5x5-v0", n)
    g.reset()
    lanes = torch.arange(n, device="cuda", dtype=torch.int64)
    sample = np.arange(0, n, 9973)
    o = OracleEnv("Empty-5x5-v0", len(sample))
    o.reset()
    dp = dp_first_goal_counts(L_MAX)
    total = torch.zeros(n, dtype=torch.int32, device="cuda")
    for t in range(L_MAX):
        a = ((lanes // 7 ** (L_MAX - 1 - t)) % 7).to(torch.uint8)
        obs, r, te, tr = g.step(a)
        L = t + 1
        assert int(te.sum()) == dp[L] * 7 ** (L_MAX - L), L
        assert int(tr.sum()) == 0
        if dp[L]:
            want = np.float32(success_reward(0, L, 100))
            rr = r[te == 1].cpu().numpy()
            assert np.all(rr.view(np.uint32) == want.view(np.uint32))
        assert int((r[te == 0] != 0).sum()) == 0
        total += te.to(torch.int32)
        oo, orw, ote, otr = o.step(a.cpu().numpy()[sample])
        idx = torch.from_numpy(sample).cuda()
        assert np.array_equal(obs[idx].cpu().numpy(), oo)
        assert np.array_equal(r[idx].cpu().numpy().view(np.uint32), orw.view(np.uint32))
        assert np.array_equal(te[idx].cpu().numpy(), ote)
    assert int(total.max()) <= 1
