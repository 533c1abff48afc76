import numpy as np, torch
from inputgen import random_actions
from oracle import OracleEnv
from paper_2407_19396_b200 import NavixEnv
env_id, n = "GoToDoor-6x6-v0", 555
g = NavixEnv(env_id, n, seed=21); o = OracleEnv(env_id, n, seed=21)
g.reset(); o.reset()
acts = random_actions(1, 3, n, 7, high=8)
for t in range(3):
    pre = o.export()
    go, *_ = g.step(torch.from_numpy(acts[t]).cuda()); oo, *_ = o.step(acts[t])
go = go.cpu().numpy()
bad = np.argwhere((go != oo).reshape(n, -1).any(1))[:, 0]
for e in bad[:2]:
    H = W = 6
    rec = pre[e]; print("env", e, "action", acts[2, e], "agent", rec[108:111], "target", rec[-2:])
    c = rec[:108].reshape(6, 6, 3)
    for y in range(6): print(" ".join(f"{c[y,x,0]}{c[y,x,1]}{c[y,x,2]}" for x in range(6)))
    print("oracle obs type/col/state\n", oo[e].transpose(1, 0, 2).reshape(7, 21))
    print("gpu obs\n", go[e].transpose(1, 0, 2).reshape(7, 21))
