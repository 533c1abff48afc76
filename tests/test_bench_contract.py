"""bench.py's JSON-line contract (the driver parses it): the reference arm on
the CPU oracle (no GPU) and the navix arm on a small workload (GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches"}


def _free_port() -> str:
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        return str(sock.getsockname()[1])


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "3", "--warmup", "3", "--envs-per-gpu", "512",
              "--ref-budget-s", "3"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("DoorKey-8x8-v0")


@pytest.mark.gpu
def test_navix_arm_line():
    d = _run(["--steps", "5", "--warmup", "3", "--envs-per-gpu", "8192", "--cpu-envs", "64", "--cpu-steps", "5",
              "--rollout-steps", "4", "--categorical-steps", "4", "--e2e-steps", "2"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["scaling"] == "weak"
    assert d["value"] > 0 and d["unit"] == "env-steps/s" and d["dtype"] == "u8" and d["vs_baseline"] is None
    roof = d["roofline"]
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s" and 0 < roof["frac"] < 1.5
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 8192 and d["e2e"]["d2h_bytes_per_step"] == 8192 * 153
    assert d["gpu_launches"] == 5
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["rollout"]["value"] > 0 and d["categorical"]["value"] > 0
    assert len(d["rank_ms_per_step"]) == 1 and abs(d["rank_ms_per_step"][0] - d["ms_per_step"]) < 1e-6
    assert d["steady_state"]["value"] > 0 and "uniform over [0, T)" in d["steady_state"]["desync"]


@pytest.mark.gpu
def test_navix_arm_strong_scaling_split():
    # [CFG 5]: a fixed global env count split over the ranks (here one rank)
    d = _run(["--steps", "4", "--warmup", "3", "--global-envs", "3000", "--no-cpu-baseline", "--rollout-steps", "0",
              "--categorical-steps", "0", "--e2e-steps", "1", "--steady-steps", "4"])
    assert d["scaling"] == "strong" and d["config"]["global_envs"] == 3000 and d["config"]["envs_per_gpu"] == 3000
    assert "3000 envs in total" in d["config"]["workload"]
    assert d["e2e"]["h2d_bytes_per_step"] == 3000 and d["roofline"]["envs_per_launch"] == 3000


@pytest.mark.gpu
def test_navix_arm_multirank_path_gloo():
    # the torchrun path (2 ranks, barriers, max over ranks, stats all-reduce,
    # one line from rank 0) on whatever GPUs exist; gloo so that two ranks may
    # share one GPU — a functional check, the timings are meaningless
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", _free_port(), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "4", "--warmup", "3", "--envs-per-gpu", "4096", "--rollout-steps", "2",
           "--categorical-steps", "2", "--e2e-steps", "1", "--backend", "gloo"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_envs"] == 8192 and d["value"] > 0
    assert d["cpu_baseline"] is None  # rank 0 at N = 1 only
    assert len(d["rank_ms_per_step"]) == 2 and abs(max(d["rank_ms_per_step"]) - d["ms_per_step"]) < 1e-6
    st = d["episode_stats"]
    assert st["episodes"] >= 0 and st["gen_failures"] == 0


def _torchrun_bench(nproc, extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", _free_port(), os.path.join(ROOT, "bench.py"),
           "--gpus", str(nproc), *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_navix_arm_multirank_strong_split_gloo():
    # --global-envs under torchrun: 5001 envs split 2500 / 2501, strong scaling
    d = _torchrun_bench(2, ["--steps", "3", "--warmup", "3", "--global-envs", "5001", "--rollout-steps", "0",
                            "--categorical-steps", "0", "--e2e-steps", "1", "--steady-steps", "3",
                            "--backend", "gloo"])
    assert d["scaling"] == "strong" and d["config"]["global_envs"] == 5001 and len(d["rank_ms_per_step"]) == 2


@pytest.mark.gpu
def test_navix_arm_two_gpus_nccl():
    # the NCCL path (device_id-bound process group, stats SUM and time MAX
    # all-reduces on the device) with the CUDA kernels on two real GPUs
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (this pool gives one per call; the driver's scaling run covers it)")
    d = _torchrun_bench(2, ["--steps", "5", "--warmup", "3", "--envs-per-gpu", "65536", "--rollout-steps", "2",
                            "--categorical-steps", "2", "--e2e-steps", "1", "--steady-steps", "5"])
    assert d["n_gpus"] == 2 and d["value"] > 0 and len(d["rank_ms_per_step"]) == 2
    assert d["episode_stats"]["gen_failures"] == 0


def test_reference_arm_under_torchrun_prints_once():
    # N > 1: rank 0 alone times the oracle and prints; the other ranks exit 0 without work
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", _free_port(), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "3", "--warmup", "3", "--envs-per-gpu", "256",
           "--ref-budget-s", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
