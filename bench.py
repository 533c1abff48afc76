#!/usr/bin/env python
"""Benchmark of the batched MiniGrid step (BASELINE.json metric).

`python bench.py --gpus N --steps K --warmup W` (N > 1 under torchrun, one rank
per GPU) prints ONE JSON line on rank 0:
  env-steps/s of DoorKey-8x8 (device-timed, whole box, weak scaling at
  --envs-per-gpu envs per GPU), the HBM roofline fraction of the step kernel,
  an end-to-end number through the host-buffer C-ABI call, the CPU oracle
  timed on this host (cpu_baseline), clocks sampled during the timed region.
`--global-envs N` splits a fixed total of N envs over the ranks instead
(strong scaling, [CFG 5]'s 2^10..2^23 sweep); the line carries every rank's
step time.  A steady-state (desynchronised) number is measured beside the
synchronised one: step counts drawn uniformly over [0, T) are imported
before a second timed region, so truncations no longer coincide.
`--impl reference` times the CPU oracle (the reference arm of this tier) on
rank 0 and prints its line; other ranks exit 0.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import subprocess
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "env-steps/sec (device-timed, whole box) DoorKey-8x8 at 1/2/4/8 B200; % HBM roofline"
UNIT = "env-steps/s"


def algorithmic_bytes(spec) -> int:
    """1 action + H*W grid + 8 + 8 agent record r/w + 147 obs + 4 reward
    + 2 flags (+ 8 Dynamic-Obstacles ball positions r/w) per env-step."""
    b = 1 + spec.height * spec.width + 8 + 8 + 147 + 4 + 2
    if spec.family == 2:
        b += 8
    return b


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def step_kernel_name(env, env_id):
    """The step kernel launch_fhwk (csrc/step_kernel.cuh) picks: the persistent
    kernel for grids of at most 16 row planes (height x ceil(width / 8)), the
    one-tile kernel above that (or when NAVIX_STEP_KERNEL selects it)."""
    s = env.spec
    planes = s.height * ((s.width + 7) // 8)
    onetile = os.environ.get("NAVIX_STEP_KERNEL", "").startswith("o") or planes > 16
    return f"navix_kernel<{env_id}, STEP>" if onetile else f"navix_step_persistent<{env_id}>"


def committed_traffic(env_id: str):
    """dram bytes per env-step of the step kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(env_id)


# Sampler process: NVML SM clock + clock-event reasons every ~1 ms, one line
# "t_monotonic mhz reasons_mask" per sample, until stdin closes.  A separate
# process keeps sampling while the main thread sits in a blocking graph launch.
_SAMPLER = r"""
import os, select, sys, time
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("max", nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM), flush=True)
log = open(sys.argv[2], "w")  # a file, not the pipe: the parent reads it only at the end
while True:
    r, _, _ = select.select([sys.stdin], [], [], 0.0005)
    if r and not os.read(sys.stdin.fileno(), 64):
        break
    try:
        m = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        q = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        log.write("%r %d %d\n" % (time.monotonic(), m, q))
    except Exception:
        pass
log.close()
"""

_REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80}


class ClockSampler:
    """SM clocks and throttle reasons sampled by a separate process during the
    timed region (`start()` early, `mark()` around the region, `summary()`)."""

    def __init__(self, index: int):
        self.index, self.proc, self.max_mhz = index, None, None
        self.t0 = self.t1 = None

    def start(self):
        try:
            import tempfile
            fd, self.path = tempfile.mkstemp(prefix="navix_clocks_", suffix=".txt")
            os.close(fd)
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(self.index), self.path],
                                         stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            first = self.proc.stdout.readline().split()  # blocks until NVML is up
            self.max_mhz = int(first[1]) if first and first[0] == "max" else None
        except Exception:  # pragma: no cover - no NVML / sampler
            self.proc = None
        return self

    def mark_begin(self):
        self.t0 = time.monotonic()

    def mark_end(self):
        self.t1 = time.monotonic()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        try:
            self.proc.communicate(input="", timeout=30)
            with open(self.path) as f:
                out = f.read()
            os.remove(self.path)
        except Exception:  # pragma: no cover
            self.proc.kill()
            out = ""
        rows = []
        for line in out.splitlines():
            f = line.split()
            if len(f) == 3:
                rows.append((float(f[0]), int(f[1]), int(f[2])))
        window = [r for r in rows if self.t0 is not None and self.t0 <= r[0] <= self.t1]
        if not window and rows:  # region shorter than one sample: the nearest ones
            window = sorted(rows, key=lambda r: abs(r[0] - (self.t1 or r[0])))[:3]
        mhz = sorted(r[1] for r in window)
        reasons = sorted({k for r in window for k, bit in _REASONS.items() if r[2] & bit})
        return {"sm_mhz": mhz[len(mhz) // 2] if mhz else None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(window)}


def cpu_info():
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count()


def time_oracle(env_id: str, n_envs: int, steps: int, warmup: int, env_begin: int = 0, n_total=None):
    """Time the CPU oracle (single thread) on `n_envs` envs: returns env-steps/s."""
    from oracle import OracleEnv, sample_actions
    o = OracleEnv(env_id, n_envs, seed=0, env_begin=env_begin, num_envs_total=n_total)
    o.reset()
    acts = sample_actions(1, env_begin, n_envs, 0, warmup + steps, o.spec.n_actions)
    for t in range(warmup):
        o.step(acts[t])
    t0 = time.perf_counter()
    for t in range(warmup, warmup + steps):
        o.step(acts[t])
    dt = time.perf_counter() - t0
    return n_envs * steps / dt, dt


def calibrate_oracle(env_id: str) -> float:
    rate, _ = time_oracle(env_id, 256, 40, 2)
    return rate


def run_reference(args, rank):
    if rank != 0:
        return
    model, ncpu = cpu_info()
    rate = calibrate_oracle(args.env)
    # bounded sample per step: the whole (warmup + steps) run within ~budget seconds
    budget = args.ref_budget_s
    n_ref = int(max(16, min(total_envs(args, args.gpus), rate * budget / max(1, args.warmup + args.steps))))
    value, dt = time_oracle(args.env, n_ref, args.steps, args.warmup)
    sample = (f"{n_ref} envs (global indices 0..{n_ref - 1}) of the {args.env} workload per step, "
              f"{args.steps} timed steps after {args.warmup} warm-up, single-threaded C++ oracle, {model}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.global_envs > 0 else "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic", "config": workload_config(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "host": {"cpu_model": model, "nproc": ncpu},
    }
    print(json.dumps(line), flush=True)


def total_envs(args, world):
    """Whole-job env count: --global-envs (strong scaling) or envs-per-GPU x ranks (weak)."""
    return args.global_envs if args.global_envs > 0 else args.envs_per_gpu * world


def workload_config(args, world):
    n_total = total_envs(args, world)
    per = (f"{args.envs_per_gpu} envs per GPU ({n_total} total)" if args.global_envs <= 0 else
           f"{n_total} envs in total split over {world} GPU(s) (~{n_total // world} per GPU)")
    return {
        "workload": f"{args.env}, {per}, "
                    f"uniform random policy (Philox action stream), auto-reset, symbolic 7x7x3 obs",
        "env_id": args.env, "envs_per_gpu": n_total // world if args.global_envs > 0 else args.envs_per_gpu,
        "global_envs": n_total,
        "parallelism": f"env-sharded x{world} (NCCL all-reduce of int64[8] episode stats only)",
        "l2": "inputs larger than L2: per step per GPU ~230 MB (state 76 MB read+write, obs 154 MB) vs 126 MB L2",
        "graph": "CUDA graph of the timed steps (one step kernel launch per step)",
    }


def run_navix(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2407_19396_b200 import NavixEnv
    from paper_2407_19396_b200.distributed import (all_reduce_stats, gather_over_ranks, init_process_group,
                                                   max_over_ranks, mean_legacy_return, shard_for)

    gpu = local_rank
    if args.backend == "gloo":  # functional test of the multi-rank path on fewer GPUs (timings meaningless)
        gpu = local_rank % torch.cuda.device_count()
    clk = ClockSampler(gpu).start()  # up and sampling before the timed region
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    dist = None
    if world > 1:
        import torch.distributed as dist
        init_process_group(args.backend, dev)
    n_total = total_envs(args, world)
    if n_total < world:
        raise SystemExit("--global-envs must give every rank at least one env")
    sh = shard_for(n_total, rank, world)
    begin, end, n = sh.begin, sh.end, sh.n
    env = NavixEnv(args.env, n, seed=0, env_begin=begin, num_envs_total=n_total, device=dev)
    spec = env.spec
    B = algorithmic_bytes(spec)
    env.reset()
    ring = min(args.steps, args.action_ring)
    acts = env.sample_actions(1, 0, ring)  # random policy, inputs resident in HBM
    s = torch.cuda.current_stream(dev)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for t in range(args.warmup):
        env.step(acts[t % ring])
    barrier()

    # capture the timed steps as CUDA graphs (chunks of `ring` steps)
    graphs = []
    remaining = args.steps
    if not args.no_graph:
        torch.cuda.synchronize(dev)
        while remaining > 0:
            k = min(ring, remaining)
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph):
                for t in range(k):
                    env.step(acts[t])
            graphs.append(gph)
            remaining -= k
        # graph capture does not execute; warm the graphs once (untimed)
        for gph in graphs:
            gph.replay()
    barrier()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    clk.mark_begin()  # the sampler process covers the whole timed region
    ev0.record(s)
    if graphs:
        for gph in graphs:
            gph.replay()
    else:
        for t in range(args.steps):
            env.step(acts[t % ring])
    ev1.record(s)
    torch.cuda.synchronize(dev)
    clk.mark_end()
    t_local = ev0.elapsed_time(ev1) / 1e3
    t_max = max_over_ranks(t_local, dev)
    t_ranks = gather_over_ranks(t_local, dev)
    value = n_total * args.steps / t_max

    # episode statistics: the one collective of the path (NCCL all-reduce of int64[8])
    st = all_reduce_stats(env.stats()).cpu().numpy()
    # its cost (once per report interval): stats reduction kernel +
    # all-reduce, device-timed, against 100 steps
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(s)
    for _ in range(10):
        all_reduce_stats(env.stats())
    s1.record(s)
    torch.cuda.synchronize(dev)
    t_stats = max_over_ranks(s0.elapsed_time(s1) / 1e3 / 10, dev)

    # f1: fused K-step rollout (navix_rollout), same envs and random policy
    rollout = None
    if args.rollout_steps > 0:
        Kr = args.rollout_steps
        r_acts = acts[:Kr] if Kr <= ring else env.sample_actions(1, 0, Kr)
        outs = (torch.empty((Kr, n, 7, 7, 3), dtype=torch.uint8, device=dev),
                torch.empty((Kr, n), dtype=torch.float32, device=dev),
                torch.empty((Kr, n), dtype=torch.uint8, device=dev),
                torch.empty((Kr, n), dtype=torch.uint8, device=dev))
        env.rollout(r_acts, out=outs)  # warm-up
        barrier()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        r0.record(s)
        for _ in range(reps):
            env.rollout(r_acts, out=outs)
        r1.record(s)
        torch.cuda.synchronize(dev)
        t_r = max_over_ranks(r0.elapsed_time(r1) / 1e3 / reps, dev)
        # the same K steps with the random policy drawn inside the kernel (no action reads)
        env.rollout_random(1, 0, Kr, out=outs)
        barrier()
        r0.record(s)
        for _ in range(reps):
            env.rollout_random(1, 0, Kr, out=outs)
        r1.record(s)
        torch.cuda.synchronize(dev)
        t_rr = max_over_ranks(r0.elapsed_time(r1) / 1e3 / reps, dev)
        Br = 1 + 147 + 4 + 2
        rollout = {"steps_per_launch": Kr, "value": n_total * Kr / t_r, "unit": UNIT,
                   "ms_per_launch": 1e3 * t_r, "algorithmic_bytes_per_env_step": Br,
                   "achieved_GBps_per_gpu": Br * n * Kr / t_r / 1e9,
                   "frac_of_measured_hbm": Br * n * Kr / t_r / 1e9 / measured_peaks()[0],
                   "api": "navix_rollout (state on chip across the K steps; row f1)",
                   "in_kernel_policy": {"value": n_total * Kr / t_rr, "unit": UNIT, "ms_per_launch": 1e3 * t_rr,
                                        "api": "navix_rollout_random (Philox policy inside the kernel)"}}
        del outs

    # f3: the same step emitting Table 5 `categorical_first_person` (49 B records)
    categorical = None
    if args.categorical_steps > 0:
        Kc = min(args.categorical_steps, ring)
        cenv = NavixEnv(args.env, n, seed=0, env_begin=begin, num_envs_total=n_total, device=dev,
                        observation="categorical")
        cenv.reset()
        for t in range(args.warmup):
            cenv.step(acts[t % ring])
        torch.cuda.synchronize(dev)
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph):
            for t in range(Kc):
                cenv.step(acts[t])
        gph.replay()
        barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(s)
        gph.replay()
        c1.record(s)
        torch.cuda.synchronize(dev)
        t_c = max_over_ranks(c0.elapsed_time(c1) / 1e3 / Kc, dev)
        Bc = B - 147 + 49
        categorical = {"steps": Kc, "value": n_total / t_c, "unit": UNIT, "ms_per_step": 1e3 * t_c,
                       "algorithmic_bytes_per_env_step": Bc, "achieved_GBps_per_gpu": Bc * n / t_c / 1e9,
                       "frac_of_measured_hbm": Bc * n / t_c / 1e9 / measured_peaks()[0],
                       "api": "navix_step with navix_set_observation(CATEGORICAL) (row f3)"}
        del gph, cenv

    # steady state: the timed region above starts right after reset, so every
    # env's truncation falls on the same step (all episodes start together).
    # Desynchronise them through the public state API (step counts uniform
    # over [0, T), the parity suite's imported states), then time again.
    steady = None
    if args.steady_steps > 0:
        rec = env.export_state()
        p = 3 * spec.height * spec.width
        rng = np.random.default_rng(1234 + rank)
        sc = rng.integers(0, spec.max_steps, size=n).astype(np.uint16)
        rec[:, p + 5] = (sc & 0xFF).astype(np.uint8)
        rec[:, p + 6] = (sc >> 8).astype(np.uint8)
        env.import_state(rec)
        del rec
        Ks = min(args.steady_steps, ring)
        for t in range(args.warmup):
            env.step(acts[t % ring])
        torch.cuda.synchronize(dev)
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph):
            for t in range(Ks):
                env.step(acts[t])
        gph.replay()
        barrier()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(s)
        gph.replay()
        q1.record(s)
        torch.cuda.synchronize(dev)
        t_q = max_over_ranks(q0.elapsed_time(q1) / 1e3 / Ks, dev)
        steady = {"steps": Ks, "value": n_total / t_q, "unit": UNIT, "ms_per_step": 1e3 * t_q,
                  "frac_of_measured_hbm": B * n / t_q / 1e9 / measured_peaks()[0],
                  "desync": "step counts uniform over [0, T) imported before timing (navix_state_import); "
                            "episodes end on different steps, the steady-state auto-reset mix"}
        del gph

    # end to end through the host-buffer C-ABI call (H2D actions, D2H outputs)
    h_act = torch.from_numpy(np.ascontiguousarray(acts[: args.e2e_steps].cpu().numpy())).pin_memory()
    h_obs = torch.empty((n, 7, 7, 3), dtype=torch.uint8).pin_memory()
    h_rew = torch.empty(n, dtype=torch.float32).pin_memory()
    h_te = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_tr = torch.empty(n, dtype=torch.uint8).pin_memory()
    env.step_host(h_act[0], h_obs, h_rew, h_te, h_tr)  # allocates staging (untimed)
    barrier()
    t0 = time.perf_counter()
    for t in range(args.e2e_steps):
        env.step_host(h_act[t], h_obs, h_rew, h_te, h_tr)
    t_e2e = max_over_ranks(time.perf_counter() - t0, dev)
    e2e_value = n_total * args.e2e_steps / t_e2e

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peaks()
    per_launch_s = t_local / args.steps
    achieved = B * n / per_launch_s / 1e9
    traffic = committed_traffic(args.env)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": None if traffic is None else traffic * n,
            "algorithmic_bytes_per_env_step": B, "envs_per_launch": n, "kernel": step_kernel_name(env, args.env),
            "peak_source": peak_src}
    model, ncpu = cpu_info()
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        n_cpu = args.cpu_envs
        v, dt = time_oracle(args.env, n_cpu, args.cpu_steps, 2)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{n_cpu} envs x {args.cpu_steps} steps of {args.env} (global indices 0..{n_cpu - 1}, "
                         f"same seeds and Philox action stream), single-threaded C++ oracle, {dt:.1f} s, {model}"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * t_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.global_envs > 0 else "weak",
        "rank_ms_per_step": [1000 * t / args.steps for t in t_ranks], "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(args, world),
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n_total,
                "d2h_bytes_per_step": n_total * (147 + 4 + 1 + 1), "steps": args.e2e_steps,
                "api": "navix_step_host (pinned host buffers)"},
        "gpu_launches": args.steps,
        "rollout": rollout,
        "categorical": categorical,
        "steady_state": steady,
        "clocks": clk.summary(),
        "stats_allreduce": {"us_per_call": 1e6 * t_stats,
                            "frac_of_100_steps": t_stats / (100 * t_max / args.steps),
                            "api": "navix_stats + torch.distributed all_reduce (NCCL for N > 1)"},
        "episode_stats": {k: int(v) for k, v in zip(
            ("episodes", "sum_len", "n_success", "sum_success_step", "n_lava", "n_failure", "n_truncated",
             "gen_failures"), st)},
        "mean_episode_return_minigrid": mean_legacy_return(st, spec.max_steps),
        "host": {"cpu_model": model, "nproc": ncpu},
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="navix", choices=["navix", "reference"])
    ap.add_argument("--env", default="DoorKey-8x8-v0")
    ap.add_argument("--envs-per-gpu", type=int, default=1 << 20)
    ap.add_argument("--global-envs", type=int, default=0,
                    help="fixed total env count split over the ranks (strong scaling); 0: --envs-per-gpu per rank")
    ap.add_argument("--steady-steps", type=int, default=200,
                    help="steps of the desynchronised steady-state measurement (0: skip)")
    ap.add_argument("--action-ring", type=int, default=1000)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--rollout-steps", type=int, default=64)
    ap.add_argument("--categorical-steps", type=int, default=200)
    ap.add_argument("--cpu-envs", type=int, default=4096)
    ap.add_argument("--cpu-steps", type=int, default=1000)
    ap.add_argument("--ref-budget-s", type=float, default=60.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: functional tests only)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    run_navix(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
