"""Timeline of bench.py's end-to-end loop (hg_pack -> H2D + degree classes on the copy stream,
hg_train_step graph replay, loss read-back) under CUPTI (torch.profiler): gaps between steps.

  python tools/exp/e2e_timeline.py [--graphs 20000]
"""
import argparse
import json
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
ap.add_argument("--steps", type=int, default=12)
args = ap.parse_args()
d = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
data = molgen.generate_to(d, "pcqm", args.graphs, 7)
store = hgnn.Store(data, copy=False)
st = store.stats()
B = args.B
cfg = hgnn.make_config(data["f_node"], 4, 128, 6, B, B * st["max_nodes_per_graph"],
                       B * int(np.diff(np.asarray(data["edge_offset"])).max()), store.degree_stat(), n_slots=2,
                       max_degree=st["max_degree"])
ctx = hgnn.Context(cfg)
ctx.params_init(1234)
hyper = dict(hgnn.DEFAULT_ADAMW)
ids = hgnn.hg_shard(13, 0, 0, 1, args.graphs)
batches = [ids[k * B:(k + 1) * B] for k in range(len(ids) // B)]
for k in range(4):
    ctx.pack(store, batches[k], k % 2)
    ctx.train_step(k % 2, graph=True, **hyper)
    ctx.loss()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ctx.pack(store, batches[4], 0)
    for k in range(args.steps):
        ctx.train_step(k % 2, graph=True, **hyper)
        ctx.loss_enqueue(k % 4)
        if k + 1 < args.steps:
            ctx.pack(store, batches[5 + k], (k + 1) % 2)
        if k > 0:
            ctx.loss_fetch((k - 1) % 4)
    torch.cuda.synchronize()
path = "gpurun_out/e2e_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
# step boundaries: the first kernel after each OpProj start
starts = [e["ts"] for e in gpu if "OpProj" in e.get("name", "")]
ends = []
for i, s in enumerate(starts):
    nxt = starts[i + 1] if i + 1 < len(starts) else 1e30
    ends.append(max(e["ts"] + e["dur"] for e in gpu if s <= e["ts"] < nxt and e.get("cat") == "kernel"
                    and "degsort" not in e.get("name", "")))
print("step   start    span   gap-to-next")
for i, s in enumerate(starts):
    gap = (starts[i + 1] - ends[i]) if i + 1 < len(starts) else 0
    print(f"{i:3d} {s - t0:9.1f} {ends[i] - s:7.1f} {gap:7.1f}")
print("\ncopy-stream work (memcpy / degsort):")
for e in gpu:
    if e.get("cat") == "gpu_memcpy" or "degsort" in e.get("name", ""):
        print(f"  {e['ts'] - t0:9.1f} {e['dur']:7.1f} {e.get('name', '')[:60]}")
cpu = [e for e in ev if e.get("cat") in ("cpu_op", "user_annotation", "python_function") and "hg" in e.get("name", "")]
