"""Build libesp.so (all CUDA sources, sm_100a) in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, no fast-math and
-fmad=false (fp32 results must match the oracle bit for bit, SURVEY.md 7 hard
part 5), linked against the same libnccl.so.2 that torch loads.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libesp.so")
OBJ = os.path.join(HERE, "build")
SOURCES = ["world.cu", "ctx.cu", "plan.cu", "hier.cu", "mcast.cu", "k_dgc.cu", "k_sign.cu", "k_randomk.cu", "k_h2.cu",
           "k_push.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl headers (nvidia-nccl wheel) not found")


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def _flags(nd):
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
                   "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(nd, "include"),
                   "-I", os.path.join(ROOT, "include"), "-diag-suppress", "186"]


def _fingerprint(flags) -> str:
    """sha256 over every source and header byte and the compiler flags: the
    library is rebuilt whenever any of them differs from what built it
    (file timestamps do not survive copies, so they are not trusted)."""
    import hashlib
    h = hashlib.sha256()
    files = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)) + [os.path.join(ROOT, "include", "esp.h")]
    for f in files:
        h.update(os.path.basename(f).encode() + b"\0")
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(flags).encode())
    return h.hexdigest()


STAMP = LIB + ".sha256"


def build(force: bool = False, verbose: bool = False) -> str:
    nd = nccl_dir()
    os.makedirs(OBJ, exist_ok=True)
    flags = _flags(nd)
    fp = _fingerprint(flags)
    if not force and os.path.exists(LIB) and os.path.exists(STAMP):
        with open(STAMP) as fh:
            if fh.read().strip() == fp:
                return LIB
    print(f"[libesp] compiling {len(SOURCES)} sources for sm_100a -> {LIB}", file=sys.stderr)

    def compile_one(src):
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        cmd = [_nvcc(), *flags, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    libdir = os.path.join(nd, "lib")
    cmd = [_nvcc(), *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-L", libdir, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath={libdir}", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    with open(STAMP, "w") as fh:
        fh.write(fp + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
