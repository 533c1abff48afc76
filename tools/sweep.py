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

import numpy as np
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
    ("Crossings-S9N3-v0", 1 << 20),
    ("Crossings-S11N5-v0", 1 << 20),
    ("GoToDoor-8x8-v0", 1 << 20),
    ("FourRooms-v0", 1 << 20),
    ("Dynamic-Obstacles-Random-6x6", 1 << 20),
]
SIZES = [1, 8, 1 << 10, 1 << 11, 1 << 14, 1 << 16, 1 << 18, 1 << 20, 1 << 21, 1 << 22, 1 << 23]
# every Table 9 id at the paper's batch (2048), 2^16 and 2^20 envs
CATALOG = ["Empty-5x5-v0", "Empty-6x6-v0", "Empty-8x8-v0", "Empty-16x16-v0", "Empty-Random-5x5", "Empty-Random-6x6",
           "Empty-Random-8x8", "Empty-Random-16x16", "DoorKey-5x5-v0", "DoorKey-6x6-v0", "DoorKey-8x8-v0",
           "DoorKey-16x16-v0", "DoorKey-Random-5x5", "DoorKey-Random-6x6", "DoorKey-Random-8x8",
           "DoorKey-Random-16x16", "FourRooms-v0", "KeyCorridorS3R1-v0", "KeyCorridorS3R2-v0", "KeyCorridorS3R3-v0",
           "KeyCorridorS4R3-v0", "KeyCorridorS5R3-v0", "KeyCorridorS6R3-v0", "LavaGapS5-v0", "LavaGapS6-v0",
           "LavaGapS7-v0", "SimpleCrossingS9N1-v0", "SimpleCrossingS9N2-v0", "SimpleCrossingS9N3-v0",
           "SimpleCrossingS11N5-v0", "Crossings-S9N1-v0", "Crossings-S9N2-v0", "Crossings-S9N3-v0",
           "Crossings-S11N5-v0", "Dynamic-Obstacles-5x5", "Dynamic-Obstacles-6x6", "Dynamic-Obstacles-8x8",
           "Dynamic-Obstacles-16x16", "DistShift1-v0", "DistShift2-v0", "GoToDoor-5x5-v0", "GoToDoor-6x6-v0",
           "GoToDoor-8x8-v0"]
CATALOG_SIZES = [1 << 11, 1 << 16, 1 << 20]


def desynchronise(env, seed: int = 1234):
    """Steady state: step counts uniform over [0, T) through the public state
    API, so the episodes no longer all truncate on the same step."""
    rec = env.export_state()
    s = env.spec
    p = 3 * s.height * s.width
    sc = np.random.default_rng(seed).integers(0, s.max_steps, size=env.n).astype(np.uint16)
    rec[:, p + 5] = (sc & 0xFF).astype(np.uint8)
    rec[:, p + 6] = (sc >> 8).astype(np.uint8)
    env.import_state(rec)


def time_point(env_id: str, n: int, steps: int, warmup: int = 10, runs: int = 5, desync: bool = False):
    env = NavixEnv(env_id, n, seed=0)
    env.reset()
    if desync:
        desynchronise(env)
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
    times = []
    for _ in range(runs):  # each point five times, 5/50/95 percentiles
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3 / (reps * ring))
    t = float(np.percentile(times, 50))
    B = algorithmic_bytes(env.spec)
    s_ = env.spec
    Bp = B - s_.height * s_.width + s_.height * 8 * ((s_.width + 7) // 8)
    peak, _ = measured_peaks()
    st = env.stats().cpu().tolist()
    env.close()
    rates = sorted(n / x for x in times)
    return {"env": env_id, "n": n, "us_per_step": t * 1e6, "env_steps_per_s": n / t,
            "env_steps_per_s_p5_p50_p95": [float(np.percentile(rates, q)) for q in (5, 50, 95)], "runs": runs,
            "GBps": B * n / t / 1e9, "frac_of_measured_hbm": B * n / t / 1e9 / peak, "bytes_per_env_step": B,
            # the layout's bytes: grid rows padded to 8-byte planes (layout.h)
            "padded_bytes_per_env_step": Bp, "frac_of_measured_hbm_padded": Bp * n / t / 1e9 / peak,
            "episodes": st[0], "desync": desync}


def time_rollout(env_id: str, n: int, K: int, runs: int = 5):
    """Row f1: K steps per launch (navix_rollout_random), per-step time."""
    env = NavixEnv(env_id, n, seed=0)
    env.reset()
    out = env.rollout_random(1, 0, K)  # warm-up, allocates the [K, n] outputs
    torch.cuda.synchronize()
    times = []
    for r in range(runs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        env.rollout_random(1, (r + 1) * K, K, out=out)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3 / K)
    t = float(np.percentile(times, 50))
    B = 1 + 147 + 4 + 2
    peak, _ = measured_peaks()
    env.close()
    rates = sorted(n / x for x in times)
    return {"env": env_id, "n": n, "rollout_k": K, "us_per_step": t * 1e6, "env_steps_per_s": n / t,
            "env_steps_per_s_p5_p50_p95": [float(np.percentile(rates, q)) for q in (5, 50, 95)], "runs": runs,
            "GBps": B * n / t / 1e9, "frac_of_measured_hbm": B * n / t / 1e9 / peak, "bytes_per_env_step": B}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "sweep.json"))
    ap.add_argument("--sizes", default="", help="comma-separated batch sizes (default: the full list)")
    ap.add_argument("--envs", default="", help="comma-separated env ids (default: all)")
    ap.add_argument("--runs", type=int, default=5, help="timed repetitions per point (percentiles)")
    ap.add_argument("--catalog", action="store_true", help="every Table 9 id at 2^11 / 2^16 / 2^20 envs")
    ap.add_argument("--rollout-k", type=int, default=0, help="time navix_rollout_random with K steps per launch")
    ap.add_argument("--desync", action="store_true",
                    help="steady state: desynchronise the episodes' step counts before timing")
    a = ap.parse_args()
    rows = []
    sizes = [int(x) for x in a.sizes.split(",") if x] or SIZES
    envs = set(x for x in a.envs.split(",") if x)
    configs = [(e, 1 << 20) for e in CATALOG] if a.catalog else CONFIGS
    if a.catalog and not a.sizes:
        sizes = CATALOG_SIZES
    if envs:  # the ids asked for, in the order given (ids outside CONFIGS up to 2^20 envs)
        known = dict(configs)
        configs = [(e, known.get(e, 1 << 20)) for e in a.envs.split(",") if e]
    for env_id, nmax in configs:
        for n in sizes:
            if n > nmax:
                continue
            if a.rollout_k:
                if n * a.rollout_k * 147 > (24 << 30):
                    continue
                r = time_rollout(env_id, n, a.rollout_k, runs=a.runs)
            else:
                r = time_point(env_id, n, a.steps, runs=a.runs, desync=a.desync)
            rows.append(r)
            pad = r.get("frac_of_measured_hbm_padded")
            print(f"{env_id:28s} N={n:>8d}  {r['us_per_step']:9.2f} us/step  {r['env_steps_per_s'] / 1e9:8.3f} G/s  "
                  f"{r['GBps']:7.0f} GB/s  {100 * r['frac_of_measured_hbm']:5.1f}%"
                  + (f"  (padded rows {100 * pad:5.1f}%)" if pad is not None else ""), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump({"gpu": torch.cuda.get_device_name(), "steps": a.steps, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
