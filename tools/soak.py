#!/usr/bin/env python
"""Soak check: 2000 CUDA-graph-replayed steps (a 500-step graph replayed 4x)
at 2^20 + 77 envs (dynamic tile scheduler, KeyCorridor's reset-first lists,
PDL launches), then three 96-env blocks compared byte for byte with the CPU
oracle replaying the same action stream.

usage: PYTHONPATH=. python tools/soak.py [env_id ...]
"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2407_19396_b200 import NavixEnv
from oracle import OracleEnv
ENVS = sys.argv[1:] or ["KeyCorridorS3R3-v0", "Dynamic-Obstacles-8x8-v0", "DoorKey-8x8-v0", "GoToDoor-8x8-v0",
                        "Dynamic-Obstacles-16x16-v0"]
fail = False
for env_id in ENVS:
    n = (1 << 20) + 77
    g = NavixEnv(env_id, n, seed=11)
    g.reset()
    K = 500
    acts = g.sample_actions(3, 0, K)
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph):
        for t in range(K):
            g.step(acts[t])
    for rep in range(4):
        graph.replay()
    torch.cuda.synchronize()
    rec = g.export_state()
    # oracle: 3 blocks replaying the same 4 x 500 action stream
    ok = True
    for b in (0, n // 2, n - 96):
        o = OracleEnv(env_id, 96, seed=11, env_begin=b, num_envs_total=n)
        o.reset()
        a = acts[:, b:b + 96].cpu().numpy()
        for rep in range(4):
            for t in range(K):
                o.step(a[t])
        ok &= np.array_equal(o.export(), rec[b:b + 96])
    print(env_id, "2000 graph-replayed steps, sampled blocks equal oracle:", ok, flush=True)
    fail |= not ok
    del g, graph, acts
    torch.cuda.empty_cache()
sys.exit(1 if fail else 0)
