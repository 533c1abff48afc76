#!/usr/bin/env python
"""Summarise an ncu report of the step kernel: key metrics, stall reasons,
dynamic opcode mix and the hottest source lines (SASS <-> -lineinfo join).

usage: python tools/analyze_ncu.py gpurun_out/prof_TAG.ncu-rep [--so path] [--kernel substr] [--json out]
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
import tempfile
from collections import Counter

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'smsp__inst_executed.sum',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__sass_branch_targets_threads_divergent.sum',
        'sm__cycles_elapsed.avg.per_second', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__grid_size', 'launch__block_size', 'launch__shared_mem_per_block_static']


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--so", default="paper_2407_19396_b200/libnavix.so")
    ap.add_argument("--kernel", default="navix_step_persistentILi1ELi8ELi8ELi0E")  # the rollout / full-obs kernels share the template args
    ap.add_argument("--envs", type=int, default=1 << 20)
    ap.add_argument("--json")
    ap.add_argument("--lines", type=int, default=30)
    a = ap.parse_args()
    raw = list(csv.reader(io.StringIO(run(["ncu", "-i", a.rep, "--page", "raw", "--csv"]))))
    h, u, v = raw[0], raw[1], raw[2]
    metrics = {k: (v[h.index(k)], u[h.index(k)]) for k in KEYS if k in h}
    stalls = {}
    for i, n in enumerate(h):
        if n.startswith('smsp__pcsamp_warps_issue_stalled_') and not n.endswith('not_issued'):
            try:
                stalls[n.replace('smsp__pcsamp_warps_issue_stalled_', '')] = float(v[i].replace(',', ''))
            except ValueError:
                pass
    for k, (val, unit) in metrics.items():
        print(f"{k:62s} {val:>18s} {unit}")
    tot = sum(stalls.values()) or 1
    print("stall samples:", ", ".join(f"{k} {100 * s / tot:.0f}%" for k, s in sorted(stalls.items(), key=lambda x: -x[1])[:8]))
    sass = list(csv.reader(io.StringIO(run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    hh = sass[1]
    ie, src = hh.index('Instructions Executed'), hh.index('Source')
    prof = [(r[src].strip(), int(r[ie])) for r in sass[2:] if len(r) > ie and r[ie].isdigit()]
    ops = Counter()
    for ins, n in prof:
        t = ins.split()
        o = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
        ops[o] += n
    total = sum(ops.values())
    per_env = 32 / a.envs
    print(f"dynamic warp instructions {total}, thread-instr/env ~{total * per_env:.0f}")
    print("opcodes/env:", ", ".join(f"{o} {n * per_env:.0f}" for o, n in ops.most_common(14)))
    lines = []
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(a.so)], cwd=d, capture_output=True)
        dis, st = [], []
        for cub in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):  # the TU holding the kernel
            dis = run(["nvdisasm", "-g", "-c", os.path.join(d, cub)]).split("\n")
            st = [i for i, l in enumerate(dis) if l.startswith('//----') and a.kernel in l]
            if st:
                break
        if st:
            if st:
                en = [i for i, l in enumerate(dis[st[0] + 1:], st[0] + 1) if l.startswith('//----')]
                seq, cur = [], None
                for l in dis[st[0]: en[0] if en else len(dis)]:
                    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
                    if m:
                        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
                        continue
                    if re.match(r'\s+/\*[0-9a-f]{4,}\*/', l):
                        seq.append(cur)
                if len(seq) == len(prof):
                    by = Counter()
                    for key, (_, n) in zip(seq, prof):
                        by[key] += n
                    lines = [(k, n * per_env) for k, n in by.most_common(a.lines)]
                    print("hottest lines (thread-instr/env):")
                    for k, n in lines:
                        print(f"  {n:7.1f}  {k}")
                else:
                    print(f"(sass/lineinfo length mismatch {len(seq)} vs {len(prof)}: rebuild matches the profiled .so?)")
    if a.json:
        json.dump({"report": os.path.basename(a.rep), "metrics": metrics, "stall_samples": stalls,
                   "thread_instr_per_env": total * per_env,
                   "opcodes_per_env": {o: n * per_env for o, n in ops.most_common(30)},
                   "hottest_lines": lines}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
