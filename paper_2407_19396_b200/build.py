"""Build libnavix.so in-tree with nvcc for sm_100a (no JIT cache, no CPU path)."""
from __future__ import annotations

import glob
import hashlib
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libnavix.so")
# every translation unit: the C ABI, the dispatcher and one file of kernel
# instantiations per family group (compiled in parallel)
SOURCES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(CSRC, "*.cu")))
HEADERS = ["layout.h", "philox.cuh", "levelgen.cuh", "obs.cuh", "step_kernel.cuh",
           os.path.join("..", "..", "include", "navix.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    *os.environ.get("NAVIX_EXTRA_NVCC_FLAGS", "").split(),  # A/B experiments only
]


def source_hash() -> str:
    """16 hex digits of SHA-256 over every source / header this library is
    built from and the compiler flags: the build id compiled into libnavix.so
    (navix_build_id) and compared with the tree by the tests."""
    h = hashlib.sha256()
    for name in SOURCES + HEADERS:
        h.update(name.encode() + b"\0")
        with open(os.path.join(CSRC, name), "rb") as f:
            h.update(f.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()[:16]


def embedded_build_id(path: str = SO) -> str | None:
    """The build id inside a built .so, read from its bytes (without loading it)."""
    if not os.path.exists(path):
        return None
    with open(path, "rb") as f:
        m = re.search(rb"NAVIX_BUILD_ID=([0-9a-f]{16})", f.read())
    return m.group(1).decode() if m else None


def _stale() -> bool:
    # content-addressed, not by mtime: a prebuilt .so from another tree (or a
    # checkout that reset mtimes) is rebuilt unless its id matches this tree
    return embedded_build_id() != source_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return SO
    os.makedirs(os.path.join(HERE, "..", "build"), exist_ok=True)

    bid = source_hash()

    def compile_one(src):
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, f'-DNAVIX_BUILD_ID="{bid}"', "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(os.path.join(HERE, "..", "build", src.replace(".cu", ".ptxas.txt")), "w") as f:
            f.write(r.stderr)
        return src, obj, r

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs = []
    for src, obj, r in results:
        if verbose or r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    # default static cudart: the .so carries its own runtime, shares the
    # primary context (and stream handles) with torch's.
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", SO]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    for o in objs:
        os.remove(o)
    if embedded_build_id() != bid:
        raise RuntimeError("libnavix.so does not carry the build id it was compiled with")
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
