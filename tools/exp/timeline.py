"""Kernel timeline of one graph-replayed training step (CUPTI via torch.profiler).

  python tools/exp/timeline.py [--graphs 20000] [--json out.json]
Prints every kernel of the last profiled step: start offset, duration, stream,
and the gap since the previous kernel on the same stream.
"""
import argparse
import json
import os
import re
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
ap.add_argument("--dataset", default="pcqm", choices=["pcqm", "aisd"])
ap.add_argument("--json", default="gpurun_out/timeline_trace.json")
ap.add_argument("--nosync", action="store_true", help="launch the profiled steps back to back")
args = ap.parse_args()

d = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
data = molgen.generate_to(d, args.dataset, args.graphs, 7)
store = hgnn.Store(data, copy=False)
st = store.stats()
B, H, L = args.B, 128, 6
cfg = hgnn.make_config(data["f_node"], 4, H, L, B, B * st["max_nodes_per_graph"],
                       B * int(np.diff(np.asarray(data["edge_offset"])).max()), store.degree_stat(), n_slots=1,
                       max_degree=st["max_degree"])
rank = int(os.environ.get("RANK", "0"))
world = int(os.environ.get("WORLD_SIZE", "1"))
torch.cuda.set_device(rank)
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
ctx = hgnn.Context(cfg, device=rank)
ctx.params_init(1234)
ctx.comm_init(rank, world)
hyper = dict(hgnn.DEFAULT_ADAMW)
ids = hgnn.hg_shard(13, 0, rank, world, args.graphs)[:B]
ctx.upload(hgnn.hg_pack_host(store, ids, cfg), 0)
ctx.capture_step(0, **hyper)
for _ in range(10):
    ctx.train_step(0, graph=True, **hyper)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

if world > 1:
    dist.barrier()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        ctx.train_step(0, graph=True, **hyper)
        if not args.nosync:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
if rank != 0:
    sys.exit(0)
os.makedirs(os.path.dirname(args.json) or ".", exist_ok=True)
prof.export_chrome_trace(args.json)
ev = json.load(open(args.json))["traceEvents"]
k = [e for e in ev if e.get("cat") == "kernel"]
k.sort(key=lambda e: e["ts"])
# split into steps at layer 0's projection (the first kernel of every step; the degree sort
# runs at upload time on the copy stream)
steps, cur = [], []
for e in k:
    if "OpProj" in e["name"] and cur:
        steps.append(cur)
        cur = []
    cur.append(e)
if cur:
    steps.append(cur)
s = steps[-1] if len(steps[-1]) > 10 else steps[-2]
t0 = s[0]["ts"]
t1 = max(e["ts"] + e["dur"] for e in s)
print(f"{len(steps)} steps profiled; last step: {len(s)} kernels, span {t1 - t0:.1f} us")


def short(n):
    n = re.sub(r"\(.*", "", n)
    n = n.replace("void ", "").replace("hg::", "")
    return n[:48]


last_end = {}
busy = 0.0
for e in s:
    stream = e["args"].get("stream")
    gap = e["ts"] - last_end.get(stream, e["ts"])
    last_end[stream] = e["ts"] + e["dur"]
    print(f"{e['ts'] - t0:8.1f} {e['dur']:7.1f} s{stream:<3} gap {gap:6.1f}  {short(e['name'])}")
agg = {}
for e in s:
    n = short(e["name"])
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += e["dur"]
print("\nper kernel (sum of durations, us):")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {t:8.1f} {c:4d}  {n}")
