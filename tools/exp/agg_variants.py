"""Build libhgnn variants differing only in agg.cu compile-time knobs (experiments).

  python tools/exp/agg_variants.py NAME:-DX=1,-DY=2 ...      (agg.cu)
  python tools/exp/agg_variants.py NAME:tcmn.cu:-DX=1 ...     (another source)
writes paper_2207_11333_b200/lib/variants/libhgnn_NAME.so
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2207_11333_b200 import build as B  # noqa: E402

B.build()
vdir = os.path.join(B.LIBDIR, "variants")
os.makedirs(vdir, exist_ok=True)
nccl_inc, nccl_lib = B._nccl_dirs()
for spec in sys.argv[1:]:
    name, _, rest = spec.partition(":")
    src, _, flags = rest.partition(":") if (".cu" in rest or rest.startswith("all")) else ("agg.cu", "", rest)
    defs = [f for f in flags.split(",") if f]
    srcs = B.CU_SOURCES if src == "all" else [src]
    vobjs, spills = [], []
    for sf in srcs:
        obj = os.path.join(B.OBJDIR, f"{sf[:-3]}_{name}.o")
        cmd = [B.NVCC] + B.ARCH + ["-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
                                   "-O3", "-std=c++17", f"-I{B.INC}", f"-I{B.CSRC}", f"-I{nccl_inc}"] + defs + \
            ["-c", os.path.join(B.CSRC, sf), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr)
        spills += [l for l in r.stderr.splitlines() if "spill" in l or "Used" in l]
        vobjs.append(obj)
    objs = [os.path.join(B.OBJDIR, f + ".o") for f in B.CU_SOURCES + B.CPP_SOURCES if f not in srcs] + vobjs
    out = os.path.join(vdir, f"libhgnn_{name}.so")
    link = [B.NVCC] + B.ARCH + ["-shared", "-cudart", "shared", "-o", out] + objs + \
        [f"-L{nccl_lib}", "-lnccl", "-Xlinker", f"-rpath,{nccl_lib}", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
         "-lpthread", "-lgomp"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    print(name, defs, out)
    for l in spills[-16:]:
        print("   ", l.strip())
