"""I/O backend comparison (Fig. "Comparison of
different I/O methods"): time to load a PCQM-shaped dataset into the pinned Table-1
store from (a) the packed container with subfiles (ADIOS stand-in) and (b) one object
file per graph (the Pickle-style baseline). Prints one JSON line.

  python tools/bench_io.py [--graphs 100000] [--dir /tmp/hgio] [--threads 16]
Caches: files are written then evicted with posix_fadvise(DONTNEED) before each timed
load ("cold" where the filesystem honours it; tmpfs does not) -- reported as given.
"""
import argparse
import json
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import molgen  # noqa: E402
from paper_2207_11333_b200 import hgnn  # noqa: E402


def evict(d):
    n = 0
    for f in os.listdir(d):
        fd = os.open(os.path.join(d, f), os.O_RDONLY)
        try:
            os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
            n += 1
        finally:
            os.close(fd)
    return n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graphs", type=int, default=100000)
    ap.add_argument("--dir", default="/tmp/hgio")
    ap.add_argument("--threads", type=int, default=min(16, os.cpu_count() or 1))
    ap.add_argument("--subfiles", default="1,4,16,64")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    shutil.rmtree(a.dir, ignore_errors=True)
    os.makedirs(a.dir)
    data = molgen.generate("pcqm", a.graphs, 17)
    src = hgnn.Store(data)
    raw = sum(int(v.nbytes) for k, v in data.items() if hasattr(v, "nbytes"))
    out = {"metric": "dataset load time into the Table-1 store, packed container vs object files",
           "graphs": a.graphs, "threads": a.threads, "raw_bytes": raw, "dir": a.dir, "container": {}}

    def timed(fn, d):
        best = None
        for _ in range(a.reps):
            evict(d)
            t = time.perf_counter()
            s = fn()
            dt = time.perf_counter() - t
            del s
            best = dt if best is None else min(best, dt)
        return best

    for k in [int(v) for v in a.subfiles.split(",")]:
        d = os.path.join(a.dir, f"c{k}")
        t0 = time.perf_counter()
        src.write_container(d, k, a.threads)
        tw = time.perf_counter() - t0
        size = sum(os.path.getsize(os.path.join(d, f)) for f in os.listdir(d))
        tr = timed(lambda: hgnn.Store.from_container(d, a.threads), d)
        out["container"][k] = {"write_s": tw, "load_s": tr, "graphs_per_s": a.graphs / tr, "bytes": size}
    d = os.path.join(a.dir, "obj")
    t0 = time.perf_counter()
    src.write_objfiles(d, a.threads)
    tw = time.perf_counter() - t0
    size = sum(os.path.getsize(os.path.join(d, f)) for f in os.listdir(d))
    tr = timed(lambda: hgnn.Store.from_objfiles(d, a.graphs, a.threads), d)
    out["objfiles"] = {"write_s": tw, "load_s": tr, "graphs_per_s": a.graphs / tr, "bytes": size, "files": a.graphs}
    best = min(v["load_s"] for v in out["container"].values())
    out["speedup_container_vs_objfiles"] = out["objfiles"]["load_s"] / best
    out["note"] = ("load = read + validate into the store used by hg_pack; paper: ADIOS 4.2x faster than Pickle on "
                   "one Summit node (PAPER.md:346)")
    print(json.dumps(out))
    shutil.rmtree(a.dir, ignore_errors=True)


if __name__ == "__main__":
    main()
