"""Which one-step parameter entries differ (GPU vs oracle) for a parity configuration.
  PYTHONPATH=. python tools/exp/param_diag.py preset B H L tensor"""
import sys

import numpy as np
import torch

import oracle as O
from tests import _parity as PT
from paper_2207_11333_b200 import hgnn

preset, B, H, L, name = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
data = PT.generate(preset, max(600, 4 * B), 21)
ctx, cfg, delta = PT.make_ctx(data, B, H, L, seed=5)
ids = O.shard(23, 1, 0, 1, len(data["y"]))[:B]
p0 = {k: np.asarray(v, np.float64) for k, v in hgnn.arena_to_dict(ctx.params_get(), ctx.layout).items()}
ctx.pack(ctx._store, ids, 0)
ctx.forward(0)
ctx.backward(0)
torch.cuda.synchronize()
gg = hgnn.arena_to_dict(ctx.grads_get(), ctx.layout)
b = O.pack(data, ids)
ocfg = PT.oracle_cfg(cfg)
loss, yhat, cache = O.forward(p0, b, ocfg, delta)
N = len(b["x"])
dec, counts = O.replay(cache, PT.gpu_decisions(ctx, N, H, L))
g = O.backward(p0, b, ocfg, cache, dec)
a, o = np.asarray(gg[name], np.float64).ravel(), g[name].ravel()
sa, so = a / (np.abs(a) + 1e-8), o / (np.abs(o) + 1e-8)  # Adam step-1 direction (eps = 1e-8)
d = np.abs(sa - so)
idx = np.argsort(-d)[:10]
print("step normwise", np.linalg.norm(sa - so) / np.linalg.norm(so), "n |g|<1e-6:", int((np.abs(o) < 1e-6).sum()))
print("max|g|", np.abs(o).max(), "normwise", np.linalg.norm(a - o) / np.linalg.norm(o))
for i in idx:
    print(i, "gpu", a[i], "oracle", o[i], "adam step ratio gpu/oracle",
          (a[i] / (abs(a[i]) + 1e-8)), (o[i] / (abs(o[i]) + 1e-8)))
