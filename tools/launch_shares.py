#!/usr/bin/env python
"""Per-kernel launch count, mean duration and share of the GPU time from an
ncu launch list (`--metrics gpu__time_duration.sum --csv --log-file`).

usage: python tools/launch_shares.py gpurun_out/launches_TAG.csv [--out profiles/.../launch_shares.json]
"""
import argparse
import csv
import json
import re
from collections import OrderedDict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 14 and r[0].isdigit()]
    agg = OrderedDict()
    for r in rows:
        name = re.sub(r"\(.*$", "", r[4]).strip()
        ns = float(r[14].replace(",", ""))
        d = agg.setdefault(name, [0, 0.0])
        d[0] += 1
        d[1] += ns
    total = sum(v[1] for v in agg.values()) or 1.0
    out = {k: {"launches": n, "avg_ns": t / n, "share": t / total} for k, (n, t) in agg.items()}
    for k, v in out.items():
        print(f"{v['launches']:5d} x {v['avg_ns'] / 1e3:9.2f} us  {100 * v['share']:5.1f}%  {k}")
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
