import sys, torch
sys.path.insert(0, '.')
from paper_2407_19396_b200 import NavixEnv
for env_id in ["DoorKey-8x8-v0", "KeyCorridorS3R3-v0", "KeyCorridorS6R3-v0", "FourRooms-v0", "GoToDoor-8x8-v0", "Dynamic-Obstacles-8x8-v0", "Empty-8x8-v0"]:
    ts = []
    for seed in range(40):
        env = NavixEnv(env_id, 1, seed=seed)
        env.reset()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); env.reset_seed(seed + 1000); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
        env.close()
    ts.sort()
    print(f"{env_id:28s} reset of 1 env: median {ts[20]:.1f} us, max {ts[-1]:.1f} us")
