#!/usr/bin/env python
"""Per-step device time of the step kernel over a long run (one CUDA-graph
replay per step, events between steps), to locate reset spikes.

usage: python tools/step_times.py [env_id] [num_envs] [steps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19396_b200 import NavixEnv  # noqa: E402

env_id = sys.argv[1] if len(sys.argv) > 1 else "KeyCorridorS3R3-v0"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 600
env = NavixEnv(env_id, n, seed=0)
env.reset()
acts = env.sample_actions(1, 0, steps)
slot = torch.empty(n, dtype=torch.uint8, device="cuda")
g = torch.cuda.CUDAGraph()
slot.copy_(acts[0])
torch.cuda.synchronize()
with torch.cuda.graph(g):
    env.step(slot)
torch.cuda.synchronize()
env.reset()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
for t in range(steps):
    slot.copy_(acts[t])
    ev[2 * t].record()
    g.replay()
    ev[2 * t + 1].record()
torch.cuda.synchronize()
ts = [ev[2 * t].elapsed_time(ev[2 * t + 1]) * 1e3 for t in range(steps)]
srt = sorted(ts)
print(f"{env_id} n={n}: median {srt[steps // 2]:.1f} us, mean {sum(ts) / steps:.1f} us, max {srt[-1]:.0f} us")
print("slowest steps (us, t):", sorted(((round(x), t) for t, x in enumerate(ts)), reverse=True)[:8])
w = max(1, steps // 10)
print("mean per window of", w, "steps:", [round(sum(ts[i:i + w]) / len(ts[i:i + w]), 1) for i in range(0, steps, w)])
