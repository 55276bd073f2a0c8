"""Build libmaple.so in-tree: nvcc for sm_100a (tcgen05 needs the 'a' target), g++ for the host lattice.

    python -m paper_2412_13576_b200.build      # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmaple.so")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v"] + ARCH
CU_SOURCES = ["capi.cu", "k_descent_simt.cu", "k_descent_tc.cu", "k_descent_tcp.cu", "k_post.cu", "k_augment.cu", "k_feasible.cu"]
CPP_SOURCES = ["lattice.cpp", "sparse_ell.cpp"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r.stdout + r.stderr


def _stale(obj, srcs):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "maple.h"))
    jobs, objs = [], []
    for src in CU_SOURCES + CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            if src.endswith(".cu"):
                jobs.append([NVCC] + NVFLAGS + ["-c", s, "-o", o])
            else:
                jobs.append(["g++", "-std=c++17", "-O3", "-fPIC", "-pthread", "-c", s, "-o", o])
    logs = []
    with ThreadPoolExecutor(max_workers=max(1, min(8, len(jobs)))) as ex:
        logs = list(ex.map(_run, jobs))
    if jobs or force or _stale(OUT, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", OUT] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    if verbose:
        for lg in logs:
            sys.stdout.write(lg)
    if logs:
        with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
            f.write("".join(logs))
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
