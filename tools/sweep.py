#!/usr/bin/env python
"""Batch-size sweep of the step kernel over the five headline environments
(SURVEY §8d): env-steps/s, us/step and the HBM roofline fraction per point,
device-timed over K CUDA-graph-replayed steps after warm-up (random policy
from the device Philox stream, actions resident in HBM).

usage: python tools/sweep.py [--steps 200] [--out profiles/r01/sweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import algorithmic_bytes, measured_peaks  # noqa: E402
from paper_2407_19396_b200 import NavixEnv  # noqa: E402

CONFIGS = [  # (env id, largest N) per BASELINE.json configs
    ("Empty-5x5-v0", 1 << 20),
    ("Empty-8x8-v0", 1 << 20),
    ("DoorKey-8x8-v0", 1 << 23),
    ("Dynamic-Obstacles-8x8-v0", 1 << 20),
    ("KeyCorridorS3R3-v0", 1 << 20),
    ("LavaGapS7-v0", 1 << 20),
    ("Empty-16x16-v0", 1 << 20),
    ("DoorKey-16x16-v0", 1 << 20),
    ("Dynamic-Obstacles-16x16-v0", 1 << 20),
    ("KeyCorridorS6R3-v0", 1 << 20),
    ("Empty-Random-8x8", 1 << 20),
    ("DistShift1-v0", 1 << 20),
    ("SimpleCrossingS9N3-v0", 1 << 20),
    ("SimpleCrossingS11N5-v0", 1 << 20),
    ("GoToDoor-8x8-v0", 1 << 20),
    ("FourRooms-v0", 1 << 20),
    ("Dynamic-Obstacles-Random-6x6", 1 << 20),
]
SIZES = [1, 8, 1 << 10, 1 << 11, 1 << 14, 1 << 16, 1 << 18, 1 << 20, 1 << 21, 1 << 22, 1 << 23]


def time_point(env_id: str, n: int, steps: int, warmup: int = 10):
    env = NavixEnv(env_id, n, seed=0)
    env.reset()
    ring = min(steps, 256)
    acts = env.sample_actions(1, 0, ring)
    for t in range(warmup):
        env.step(acts[t % ring])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for t in range(ring):
            env.step(acts[t])
    g.replay()
    torch.cuda.synchronize()
    reps = max(1, steps // ring)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / (reps * ring)
    B = algorithmic_bytes(env.spec)
    peak, _ = measured_peaks()
    st = env.stats().cpu().tolist()
    env.close()
    return {"env": env_id, "n": n, "us_per_step": t * 1e6, "env_steps_per_s": n / t,
            "GBps": B * n / t / 1e9, "frac_of_measured_hbm": B * n / t / 1e9 / peak, "bytes_per_env_step": B,
            "episodes": st[0]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "sweep.json"))
    ap.add_argument("--sizes", default="", help="comma-separated batch sizes (default: the full list)")
    ap.add_argument("--envs", default="", help="comma-separated env ids (default: all)")
    a = ap.parse_args()
    rows = []
    sizes = [int(x) for x in a.sizes.split(",") if x] or SIZES
    envs = set(x for x in a.envs.split(",") if x)
    for env_id, nmax in CONFIGS:
        if envs and env_id not in envs:
            continue
        for n in sizes:
            if n > nmax:
                continue
            r = time_point(env_id, n, a.steps)
            rows.append(r)
            print(f"{env_id:28s} N={n:>8d}  {r['us_per_step']:9.2f} us/step  {r['env_steps_per_s'] / 1e9:8.3f} G/s  "
                  f"{r['GBps']:7.0f} GB/s  {100 * r['frac_of_measured_hbm']:5.1f}%", flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump({"gpu": torch.cuda.get_device_name(), "steps": a.steps, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
