"""Build libhgnn.so (C-ABI + sm_100a kernels) in-tree with nvcc.

Called by __graft_entry__.build() and, lazily, by the binding. Cross-compiles
without a GPU. Flags: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
INC = os.path.join(ROOT, "include")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libhgnn.so")
OBJDIR = os.path.join(HERE, "build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["kernels.cu", "agg.cu", "degsort.cu", "tcdirect.cu", "tcmn.cu", "p2p.cu", "ctx.cu"]
CPP_SOURCES = ["host.cpp", "container.cpp", "shm.cpp"]


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # torch's bundled NCCL (the one torch loads at run time)
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _sources():
    srcs = [os.path.join(CSRC, f) for f in CU_SOURCES + CPP_SOURCES]
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hdrs.append(os.path.join(INC, "hgnn.h"))
    return srcs, hdrs


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    srcs, hdrs = _sources()
    return any(os.path.getmtime(p) > t for p in srcs + hdrs + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    common = ["-O3", "-std=c++17", f"-I{INC}", f"-I{CSRC}", f"-I{nccl_inc}"]
    jobs = []
    for f in CU_SOURCES:
        obj = os.path.join(OBJDIR, f + ".o")
        cmd = [NVCC] + ARCH + ["-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"] + \
            common + ["-c", os.path.join(CSRC, f), "-o", obj]
        jobs.append((cmd, obj))
    for f in CPP_SOURCES:
        obj = os.path.join(OBJDIR, f + ".o")
        cmd = ["g++", "-fPIC", "-Wall", "-pthread", "-fopenmp", "-msse4.2", "-I/usr/local/cuda/include"] + common + \
            ["-c", os.path.join(CSRC, f), "-o", obj]
        jobs.append((cmd, obj))

    def run(job):
        cmd, obj = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("compile failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stderr

    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        logs = list(ex.map(run, jobs))
    if verbose:
        for l in logs:
            sys.stderr.write(l)
    with open(os.path.join(OBJDIR, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    tmp = LIB + f".tmp{os.getpid()}"
    link = [NVCC] + ARCH + ["-shared", "-cudart", "shared", "-o", tmp] + [o for _, o in jobs] + \
        [f"-L{nccl_lib}", "-lnccl", "-Xlinker", f"-rpath,{nccl_lib}", "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-Xlinker", "--no-undefined",
         "-lpthread", "-lgomp"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + " ".join(link) + "\n" + r.stdout + r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
