"""Several devices in ONE process (the C ABI's `device` argument): each handle
runs on its own device with that device's launch state (dynamic-SMEM opt-in,
SM count, occupancy are per device, step_kernel.cuh device_launch_info).
Families whose kernels need > 48 KB of dynamic SMEM (16x16 grids, FourRooms,
DistShift) are the ones a per-process cache broke.  Skips with fewer than two
GPUs (this pool gives one per call)."""
import numpy as np
import pytest
import torch

from inputgen import random_actions
from oracle import OracleEnv

pytestmark = pytest.mark.gpu

IDS = ["DoorKey-16x16-v0", "FourRooms-v0", "DistShift1-v0", "DoorKey-8x8-v0", "Dynamic-Obstacles-8x8-v0"]


@pytest.mark.parametrize("env_id", IDS)
def test_two_devices_one_process(env_id):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_2407_19396_b200 import NavixEnv
    n, steps = 300, 40
    envs = []
    for dev in (1, 0):  # device 1 first: its launch state must not come from device 0
        with torch.cuda.device(dev):
            envs.append(NavixEnv(env_id, n, seed=4, device=f"cuda:{dev}"))
    o = OracleEnv(env_id, n, seed=4)
    first = o.reset()
    for g in envs:
        with torch.cuda.device(g.device):
            np.testing.assert_array_equal(g.reset().cpu().numpy(), first)
    acts = random_actions(3, steps, n, o.spec.n_actions)
    for t in range(steps):
        oo, orw, ote, otr = o.step(acts[t])
        for g in envs:
            with torch.cuda.device(g.device):
                go, gr, gte, gtr = g.step(torch.from_numpy(acts[t]).to(g.device))
                np.testing.assert_array_equal(go.cpu().numpy(), oo)
                np.testing.assert_array_equal(gr.cpu().numpy().view(np.uint32), orw.view(np.uint32))
    for g in envs:
        np.testing.assert_array_equal(g.export_state(), o.export())
