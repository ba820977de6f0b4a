"""Per-CTA timing of the fused dX -> dA kernel (trace op id 5)."""
import ctypes, os, sys, tempfile
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import molgen
from paper_2207_11333_b200 import hgnn
d = tempfile.mkdtemp(dir="/dev/shm")
data = molgen.generate_to(d, "pcqm", 20000, 7)
store = hgnn.Store(data, copy=False); st = store.stats()
B, H, L = 128, 128, 6
cfg = hgnn.make_config(data["f_node"], 4, H, L, B, B * st["max_nodes_per_graph"],
                       B * int(np.diff(np.asarray(data["edge_offset"])).max()), store.degree_stat(), n_slots=1,
                       max_degree=st["max_degree"])
ctx = hgnn.Context(cfg, device=0); ctx.params_init(1234); ctx.comm_init(0, 1)
hyper = dict(hgnn.DEFAULT_ADAMW)
ctx.upload(hgnn.hg_pack_host(store, hgnn.hg_shard(13, 0, 0, 1, 20000)[:B], cfg), 0)
ctx.capture_step(0, **hyper)
for _ in range(5): ctx.train_step(0, graph=True, **hyper)
torch.cuda.synchronize()
lib = hgnn.load(); lib.hg_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
assert lib.hg_debug_set_trace(buf.data_ptr(), 5) == 0
ctx.train_step(0, graph=True, **hyper); torch.cuda.synchronize()
t = buf.view(-1, 8).cpu().numpy(); t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
v = t[t[:, 7] == 1].astype(float)
print("CTAs", len(t), "valid", len(v), "span us", (t[:, 6].max() - t0) / 1e3)
for name, a, b in [("start", None, 0), ("prologue", 0, 1), ("->epi wait", 1, 2), ("stage1 (acc1)", 2, 3), ("epi1", 3, 4),
                   ("stage2 s0", 4, 5), ("epi2", 5, 6), ("total", 0, 6)]:
    c = v[:, b] - (t0 if a is None else v[:, a])
    print(f"{name:14s} min {c.min()/1e3:6.2f} med {np.median(c)/1e3:6.2f} max {c.max()/1e3:6.2f}")
lib.hg_debug_set_trace(None, -1)
