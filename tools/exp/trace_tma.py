"""Per-CTA %globaltimer trace of the TMA GEMM kernels inside the captured step.

  python tools/exp/trace_tma.py [--graphs 20000]
Prints, per Op (0 update, 1 dA, 2 proj, 3 dX), the CTA-time breakdown of the
LAST launch of that kernel in one graph-replayed step.
"""
import argparse
import ctypes
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import molgen  # noqa: E402
from paper_2207_11333_b200 import hgnn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--graphs", type=int, default=20000)
ap.add_argument("--B", type=int, default=128)
args = ap.parse_args()

d = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
data = molgen.generate_to(d, "pcqm", args.graphs, 7)
store = hgnn.Store(data, copy=False)
st = store.stats()
delta = store.degree_stat()
B, H, L = args.B, 128, 6
max_nodes = B * st["max_nodes_per_graph"]
max_edges = B * int(np.diff(np.asarray(data["edge_offset"])).max())
cfg = hgnn.make_config(data["f_node"], 4, H, L, B, max_nodes, max_edges, delta, n_slots=1, max_degree=st["max_degree"])
ctx = hgnn.Context(cfg, device=0)
ctx.params_init(1234)
ctx.comm_init(0, 1)
hyper = dict(hgnn.DEFAULT_ADAMW)
ids = hgnn.hg_shard(13, 0, 0, 1, args.graphs)[:B]
ctx.upload(hgnn.hg_pack_host(store, ids, cfg), 0)
ctx.capture_step(0, **hyper)
for _ in range(5):
    ctx.train_step(0, graph=True, **hyper)
torch.cuda.synchronize()
lib = hgnn.load()
lib.hg_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
names = {0: "update", 1: "dA", 2: "proj", 3: "dX"}
for op in range(4):
    buf.zero_()
    assert lib.hg_debug_set_trace(buf.data_ptr(), op) == 0
    ctx.train_step(0, graph=True, **hyper)
    torch.cuda.synchronize()
    t = buf.view(-1, 8).cpu().numpy()
    t = t[t[:, 0] > 0]
    valid = t[t[:, 6] > 0]
    t0 = t[:, 0].min()
    span = t[:, 6].max() - t0 if len(valid) else 0
    print(f"\n== {names[op]}: {len(t)} CTAs launched, {len(valid)} with a tile; kernel span {span / 1e3:.2f} us")
    if len(valid):
        v = valid.astype(np.float64)
        cols = {
            "start skew": v[:, 0] - t0,
            "prologue+pdl": v[:, 1] - v[:, 0],
            "1st TMA->1st full": v[:, 3] - v[:, 2],
            "mainloop(MMA issue)": v[:, 4] - v[:, 3],
            "acc wait": v[:, 5] - v[:, 4],
            "epilogue": v[:, 6] - v[:, 5],
            "CTA total": v[:, 6] - v[:, 0],
        }
        for k, c in cols.items():
            print(f"  {k:22s} min {c.min() / 1e3:7.2f}  med {np.median(c) / 1e3:7.2f}  max {c.max() / 1e3:7.2f} us")
lib.hg_debug_set_trace(None, -1)
