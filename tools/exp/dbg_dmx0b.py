import numpy as np, os, sys
sys.path.insert(0, "/root/repo")
import oracle as O
from tests import _parity as PT
from paper_2207_11333_b200 import hgnn
data = PT.generate("pcqm", 600, 21)
ctx, cfg, delta = PT.make_ctx(data, 128, 128, 6, seed=5)
ids = O.shard(23, 1, 0, 1, len(data["y"]))[:128]
ocfg = PT.oracle_cfg(cfg)
params = {k: np.asarray(v, np.float64) for k, v in hgnn.arena_to_dict(ctx.params_get(), ctx.layout).items()}
ctx.pack(ctx._store, ids, 0)
ctx.forward(0); ctx.backward(0)
g = hgnn.arena_to_dict(ctx.grads_get(), ctx.layout)
b = O.pack(data, ids)
loss, yhat, cache = O.forward(params, b, ocfg, delta)
og = O.backward(params, b, ocfg, cache)
for name in ["conv0.M_x", "conv0.b_M", "conv1.M_x"]:
    d = np.abs(np.asarray(g[name], np.float64) - og[name])
    print(name, "maxscaled", d.max() / np.abs(og[name]).max())
    if d.ndim == 2:
        print(" worst cols", np.argsort(-d.max(axis=0))[:6], "worst rows", np.argsort(-d.max(axis=1))[:6])
    else:
        print(" worst idx", np.argsort(-d)[:8])
print("N", int(b["rowptr"].shape[0] - 1))
import torch
H = 128
Nn = int(b["rowptr"].shape[0] - 1)
dP0 = ctx.view_f32(100, 0)[:Nn * H].cpu().numpy().reshape(Nn, H)
dPl0 = ctx.view_f32(101, 0)[:Nn * H].cpu().numpy().reshape(Nn, H)
lo_ref = dP0 - (dP0.view(np.uint32) & 0xFFFFE000).view(np.float32)
print("dP_lo_0 mismatch", np.abs(dPl0 - lo_ref).max(), "dP0 absmax", np.abs(dP0).max())
Fp = 36
xp = ctx.view_f32(102, 0)[:Nn * Fp].cpu().numpy().reshape(Nn, Fp)
x0 = np.asarray(b["x"], np.float32).reshape(Nn, -1)
print("xpad mismatch", np.abs(xp[:, :x0.shape[1]] - x0).max(), "pad cols max", np.abs(xp[:, x0.shape[1]:]).max())
bm_host = dP0.astype(np.float64).sum(0)
print("b_M from device dP0 vs gpu grad:", np.abs(bm_host - np.asarray(g["conv0.b_M"], np.float64)).max() / np.abs(bm_host).max())
print("b_M from device dP0 vs oracle:", np.abs(bm_host - og["conv0.b_M"]).max() / np.abs(bm_host).max())
