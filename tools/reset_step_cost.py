#!/usr/bin/env python
"""Device time of ONE step as a function of how many envs auto-reset in it:
canonical states from a fresh reset, with prev_done set on a random fraction
p of the envs (imported), then one timed step (CUDA events), median of R.

usage: python tools/reset_step_cost.py [num_envs] [env_id ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19396_b200 import NavixEnv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
ids = sys.argv[2:] or ["DoorKey-8x8-v0", "LavaGapS7-v0", "KeyCorridorS3R3-v0", "KeyCorridorS4R3-v0"]
R = 15
for env_id in ids:
    env = NavixEnv(env_id, n, seed=0)
    env.reset()
    s = env.spec
    base = env.export_state()
    off = 3 * s.height * s.width + 11  # prev_done byte of the canonical record
    acts = torch.full((n,), 2, dtype=torch.uint8, device="cuda")  # forward: no grid writes
    row = []
    for p in (0.0, 0.001, 0.004, 0.02, 0.1):
        rng = np.random.default_rng(1)
        ts = []
        for r in range(R):
            rec = base.copy()
            rec[:, off] = rng.random(n) < p
            env.import_state(rec)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            env.step(acts)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        row.append(f"p={p}: {sorted(ts)[R // 2]:6.1f}")
    print(f"{env_id:24s} n={n}  one step (us): " + "  ".join(row))
    env.close()
