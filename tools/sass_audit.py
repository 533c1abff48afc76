#!/usr/bin/env python
"""SASS audit of libnavix.so (no GPU needed): for every kernel, the count of
TMA bulk copies (UBLKCP.S.G global->shared, UBLKCP.G.S shared->global),
mbarrier ops (SYNCS.*), local-memory traffic (LDL / STL = spills or indexed
locals) and ptxas' own spill report; plus an excerpt of the headline kernel's
SASS around its bulk copies.

usage: python tools/sass_audit.py [--so paper_2407_19396_b200/libnavix.so] [--out profiles/r02/sass_audit.txt]
"""
import argparse
import glob
import os
import re
import subprocess
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADLINE = "_ZN5navix21navix_step_persistentILi1ELi8ELi8ELi0EEEvNS_10KernelArgsE"


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


def ptxas_spills():
    out = {}
    for f in glob.glob(os.path.join(ROOT, "build", "*.ptxas.txt")):
        cur = None
        for line in open(f):
            m = re.search(r"Function properties for (\S+)", line)
            if m:
                cur = m.group(1)
            m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
            if m and cur:
                out[cur] = (int(m.group(1)), int(m.group(2)))
            m = re.search(r"Used (\d+) registers", line)
            if m and cur:
                out[cur] = out.get(cur, (0, 0)) + (int(m.group(1)),)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", default=os.path.join(ROOT, "paper_2407_19396_b200", "libnavix.so"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "sass_audit.txt"))
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.so], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    spills = ptxas_spills()
    rows = []
    for name, lines in funcs.items():
        c = Counter()
        for ln in lines:
            for op in ("UBLKCP.S.G", "UBLKCP.G.S", "LDL", "STL"):
                if re.search(r"\b" + re.escape(op) + r"\b", ln):
                    c[op] += 1
            if "SYNCS." in ln:
                c["SYNCS"] += 1
        rows.append((name, c, spills.get(name)))
    dem = demangle([r[0] for r in rows])
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        f.write(f"SASS audit of {os.path.relpath(a.so, ROOT)} ({len(rows)} kernels)\n")
        f.write("static instruction counts: UBLKCP.S.G (TMA bulk global->shared), UBLKCP.G.S (shared->global),\n"
                "SYNCS (mbarrier), LDL/STL (local memory); ptxas: spill store/load bytes, registers\n\n")
        f.write(f"{'kernel':90s} {'S.G':>4s} {'G.S':>4s} {'SYNCS':>5s} {'LDL':>4s} {'STL':>4s}  ptxas(spill st, ld, regs)\n")
        n_local = []
        for (name, c, sp), d in sorted(zip(rows, dem), key=lambda x: x[1]):
            f.write(f"{d[:90]:90s} {c['UBLKCP.S.G']:4d} {c['UBLKCP.G.S']:4d} {c['SYNCS']:5d} {c['LDL']:4d} "
                    f"{c['STL']:4d}  {sp}\n")
            if c["LDL"] or c["STL"]:
                n_local.append(d)
        f.write(f"\nkernels with local-memory instructions: {len(n_local)}\n")
        for d in n_local:
            f.write(f"  {d}\n")
        f.write(f"\n---- excerpt: {HEADLINE} (DoorKey-8x8 persistent step), lines with bulk copies / mbarriers\n")
        lines = funcs.get(HEADLINE, [])
        for i, ln in enumerate(lines):
            if "UBLKCP" in ln or "SYNCS" in ln or "ELECT" in ln:
                f.write(ln.rstrip() + "\n")
    print(open(a.out).read()[:3000])


if __name__ == "__main__":
    main()
