import torch, sys
sys.path.insert(0, '.')
from paper_2407_19396_b200 import NavixEnv
env_id = sys.argv[1] if len(sys.argv) > 1 else "KeyCorridorS3R3-v0"
n = 1 << 20
env = NavixEnv(env_id, n, seed=0)
env.reset()
acts = env.sample_actions(1, 0, 600)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(601)]
ev[0].record()
for t in range(600):
    env.step(acts[t])
    ev[t + 1].record()
torch.cuda.synchronize()
ts = [ev[t].elapsed_time(ev[t + 1]) * 1e3 for t in range(600)]
srt = sorted(ts)
print(env_id, "median us", srt[300], "max", srt[-5:], "mean", sum(ts) / 600)
big = [(t, round(x)) for t, x in enumerate(ts) if x > 3 * srt[300]]
print("slow steps", big[:20])
