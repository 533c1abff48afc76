#!/usr/bin/env python
"""Device latency of level generation: 100 graph-captured navix_reset calls
(memset + one MODE_RESET launch) on 1 env (one lane's serial generator) and
on 32 envs (one warp, divergent lanes), per family.

usage: python tools/gen_latency.py [env_id ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19396_b200 import NavixEnv  # noqa: E402

ids = sys.argv[1:] or ["Empty-8x8-v0", "DoorKey-8x8-v0", "KeyCorridorS3R3-v0", "KeyCorridorS6R3-v0",
                       "FourRooms-v0", "Dynamic-Obstacles-8x8-v0", "GoToDoor-8x8-v0"]
R = 100
for env_id in ids:
    row = []
    for n in (1, 32):
        env = NavixEnv(env_id, n, seed=0)
        env.reset()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for r in range(R):
                env.reset_seed(r)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        row.append(e0.elapsed_time(e1) * 1e3 / R)
        env.close()
    print(f"{env_id:28s} reset (memset + kernel): 1 env {row[0]:6.2f} us, 32 envs {row[1]:6.2f} us")
