"""Build libhks.so in-tree with nvcc for sm_100a (B200).  No JIT cache: the .so ships with the repo
snapshot to the GPU box.  Usage: python -m paper_2507_04775_b200.build [--force]"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libhks.so")
OBJ = os.path.join(HERE, "build")
SOURCES = ["ctx.cu", "ntt.cu", "ntt_tc.cu", "kernels.cu", "capi.cu", "prof.cu", "shard.cu"]
HEADERS = ["internal.h", "modarith.cuh", "tc.cuh", os.path.join("..", "..", "include", "hks.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps)


def _compile(src: str, force: bool) -> str:
    s = os.path.join(CSRC, src)
    o = os.path.join(OBJ, src.replace(".cu", ".o"))
    if force or _stale(o, s):
        log = o + ".log"
        with open(log, "w") as f:
            subprocess.check_call([NVCC, *FLAGS, "-c", s, "-o", o], stdout=f, stderr=subprocess.STDOUT)
    return o


def build(force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), SOURCES))
    if force or not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        tmp = OUT + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs])
        os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
