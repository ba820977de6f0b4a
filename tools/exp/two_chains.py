"""Experiment: do two concurrent half-batch step graphs beat one full-batch graph?

Builds contexts with B=128 and two with B=64 (separate workspaces), captures their
step graphs and times (a) the B=128 graph alone, (b) the two B=64 graphs launched
on two streams concurrently, per iteration, with CUDA events.
"""
import os, sys, tempfile
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import molgen
from paper_2207_11333_b200 import hgnn

d = tempfile.mkdtemp(dir="/dev/shm")
data = molgen.generate_to(d, "pcqm", 40000, 7)
store = hgnn.Store(data, copy=False); st = store.stats()
H, L = 128, 6
emax = int(np.diff(np.asarray(data["edge_offset"])).max())
hyper = dict(hgnn.DEFAULT_ADAMW)
ids = hgnn.hg_shard(13, 0, 0, 1, 40000)


def make(B, off, stream):
    cfg = hgnn.make_config(data["f_node"], 4, H, L, B, B * st["max_nodes_per_graph"], B * emax, store.degree_stat(),
                           n_slots=1, max_degree=st["max_degree"])
    with torch.cuda.stream(stream):
        ctx = hgnn.Context(cfg, device=0)
        ctx.params_init(1234)
        ctx.comm_init(0, 1)
        ctx.upload(hgnn.hg_pack_host(store, ids[off:off + B], cfg), 0)
        ctx.capture_step(0, **hyper)
    return ctx


s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
full = make(128, 0, s0)
ha = make(64, 0, s0)
hb = make(64, 64, s1)
torch.cuda.synchronize()


def run(ctxs_streams, iters=50):
    for _ in range(5):
        for c, s in ctxs_streams:
            with torch.cuda.stream(s):
                c.train_step(0, graph=True, **hyper)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    e0.record(main)
    for _ in range(iters):
        evs = []
        for c, s in ctxs_streams:
            s.wait_stream(main)
            with torch.cuda.stream(s):
                c.train_step(0, graph=True, **hyper)
            ev = torch.cuda.Event()
            ev.record(s)
            evs.append(ev)
        for ev in evs:
            main.wait_event(ev)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


t_full = run([(full, s0)])
t_two = run([(ha, s0), (hb, s1)])
t_half = run([(ha, s0)])
print(f"B=128 one graph: {t_full * 1e3:.1f} us/step -> {128 / t_full * 1e3:.0f} graphs/s")
print(f"2 x B=64 concurrent: {t_two * 1e3:.1f} us/step -> {128 / t_two * 1e3:.0f} graphs/s")
print(f"B=64 alone: {t_half * 1e3:.1f} us/step")
