#!/usr/bin/env python
"""Small run of every kernel (reset, persistent step, one-tile step, rollout,
observe, full obs, sample actions, stats) for compute-sanitizer:
  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_run.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19396_b200 import NavixEnv  # noqa: E402

for env_id in ("DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0", "KeyCorridorS3R3-v0", "DoorKey-16x16-v0",
               "Dynamic-Obstacles-16x16-v0", "Empty-5x5-v0"):
    n = 300
    env = NavixEnv(env_id, n, seed=1)
    env.reset()
    acts = env.sample_actions(1, 0, 12)
    for t in range(6):
        env.step(acts[t])
    env.rollout(acts[6:12].contiguous())
    env.observe()
    env.observe_full()
    env.stats()
    torch.cuda.synchronize()
    env.close()
print("sanitize run ok")
