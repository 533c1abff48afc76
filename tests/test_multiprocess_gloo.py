"""The N>1 path on CPU: world_size 2 over gloo (127.0.0.1).

Each rank takes its contiguous shard of the global env range
(paper_2407_19396_b200.distributed), steps it (here with the CPU oracle,
standing in for the GPU kernel, which needs no communication), and the
int64[8] statistics are all-reduced; the slowest rank's time is taken with a
MAX all-reduce.  The reduced statistics and the gathered per-rank states must
equal the single-process run bit-for-bit (shard invariance).
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from inputgen import random_actions

ENV_ID, N_TOTAL, STEPS = "KeyCorridorS3R3-v0", 301, 120


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from oracle import OracleEnv
    from paper_2407_19396_b200.distributed import (all_reduce_stats, init_process_group, max_over_ranks,
                                                   shard_for)
    init_process_group("gloo")
    sh = shard_for(N_TOTAL, rank, world)
    env = OracleEnv(ENV_ID, sh.n, seed=17, env_begin=sh.begin, num_envs_total=N_TOTAL)
    env.reset()
    acts = random_actions(4, STEPS, N_TOTAL, 7)
    for t in range(STEPS):
        env.step(acts[t, sh.begin:sh.end])
    stats = all_reduce_stats(torch.from_numpy(env.stats()))
    slowest = max_over_ranks(float(rank + 1))
    gathered = [None] * world
    dist.all_gather_object(gathered, (sh.begin, sh.end, env.export()))
    if rank == 0:
        q.put((stats.numpy(), slowest, gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_equals_single_process():
    from oracle import OracleEnv
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    stats, slowest, gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = OracleEnv(ENV_ID, N_TOTAL, seed=17)
    ref.reset()
    acts = random_actions(4, STEPS, N_TOTAL, 7)
    for t in range(STEPS):
        ref.step(acts[t])
    assert np.array_equal(stats, ref.stats())
    assert slowest == 2.0
    gathered.sort(key=lambda g: g[0])
    assert [(b, e) for b, e, _ in gathered] == [(0, 150), (150, 301)]
    assert np.array_equal(np.concatenate([g[2] for g in gathered]), ref.export())


def test_mean_legacy_return_is_order_free():
    from paper_2407_19396_b200.distributed import mean_legacy_return
    s = np.array([10, 900, 3, 120, 0, 1, 6, 0])
    want = (3 - 0.9 * 120 / 640 - 1) / 10
    assert mean_legacy_return(s, 640) == want
    assert mean_legacy_return(np.zeros(8), 640) == 0.0
