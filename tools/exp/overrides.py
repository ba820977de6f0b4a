"""Diagnose decision-replay overrides (tests/_parity.py) for one configuration:
for every argmax/argmin cell where the GPU's position differs from the oracle's,
report the oracle's float64 gap between the two candidates relative to |m|_inf
and whether the two candidate messages are exactly equal in float64.

  python tools/exp/overrides.py H L B
"""
import sys

import numpy as np
import torch

import oracle as O
from tests import _parity as PT

H, L, B = (int(a) for a in sys.argv[1:4])
data = PT.generate("pcqm", 800, 31)
ctx, cfg, delta = PT.make_ctx(data, B, H, L, seed=7)
ids = O.shard(17, 0, 0, 1, len(data["y"]))[:B]
params = {k: np.asarray(v, np.float64) for k, v in PT.hgnn.arena_to_dict(ctx.params_get(), ctx.layout).items()}
ctx.pack(ctx._store, ids, 0)
ctx.forward(0)
torch.cuda.synchronize()
b = O.pack(data, ids)
N = len(b["x"])
loss, yhat, cache = O.forward(params, b, PT.oracle_cfg(cfg), delta)
dec = PT.gpu_decisions(ctx, N, H, L)
for l, (c, g) in enumerate(zip(cache["layers"], dec)):
    msg, deg = c["msg"], c["deg"]
    ms = np.abs(msg).max()
    rowptr = np.concatenate([[0], np.cumsum(deg)])
    for k in ("argmax", "argmin"):
        own, gp = c[k], g[k]
        diff = (gp != own) & (deg > 0)[:, None]
        ii, cc = np.nonzero(diff)
        if len(ii) == 0:
            print(l, k, 0)
            continue
        mo = msg[rowptr[ii] + own[ii, cc], cc]
        mg = msg[rowptr[ii] + gp[ii, cc], cc]
        rel = np.abs(mo - mg) / ms
        exact = int((mo == mg).sum())
        degs = np.bincount(deg[ii], minlength=6)
        print(l, k, len(ii), "exact f64 ties", exact, "rel gap max", rel.max(), "median", np.median(rel),
              "gpu pos < own", int((gp[ii, cc] < own[ii, cc]).sum()), "deg hist", degs.tolist())
