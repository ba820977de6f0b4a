import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O
from tests import _parity as PT
from paper_2207_11333_b200 import hgnn
data = PT.generate("pcqm", 600, 51)
ids = O.shard(5, 0, 0, 1, 600)[:128]
for mode in (0, 5, 0):
    ctx, cfg, delta = PT.make_ctx(data, 128, 128, 6, seed=7)
    hgnn.load().hg_debug_set_tc_mode(mode)
    res = PT.run_step_parity(data, ids, ctx, cfg, delta, do_step=False)
    print("mode", mode, {k: (max(v.values()) if isinstance(v, dict) else v) for k, v in res.items() if k in ("yhat","X","grad_maxscaled","grad_normwise","out_of_band")})
    g = ctx.grads_get()
    if mode == 0: g0 = g
    else: print("bitwise equal to mode 0:", np.array_equal(g, g0), "max rel diff", float(np.abs(g-g0).max()/np.abs(g0).max()))
