#!/usr/bin/env python
"""A short steady-state run for profiling: N envs of one id, step counts
desynchronised through the public state API (tools/sweep.py desynchronise),
then S plain (non-graph) steps of the random policy.  Run it once plainly,
then under ncu, e.g.
  ncu --set full -k regex:navix_step_persistent -s 10 -c 1 python tools/steady_steps.py KeyCorridorS3R3-v0 65536
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_2407_19396_b200 import NavixEnv  # noqa: E402
from sweep import desynchronise  # noqa: E402


def main():
    env_id = sys.argv[1] if len(sys.argv) > 1 else "KeyCorridorS3R3-v0"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    env = NavixEnv(env_id, n, seed=0)
    env.reset()
    desynchronise(env)
    acts = env.sample_actions(1, 0, steps)
    for t in range(steps):
        env.step(acts[t])
    torch.cuda.synchronize()
    print("ok", env_id, n, steps, env.stats().cpu().tolist())


if __name__ == "__main__":
    main()
