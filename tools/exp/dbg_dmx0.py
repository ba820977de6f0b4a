import numpy as np, os, sys
sys.path.insert(0, "/root/repo")
import oracle as O
from tests import _parity as PT
from paper_2207_11333_b200 import hgnn
data = PT.generate("pcqm", 600, 51)
ids = O.shard(5, 0, 0, 1, 600)[:128]
L = int(os.environ.get("L", "2"))
ctx, cfg, delta = PT.make_ctx(data, 128, 128, L, seed=7)
res = PT.run_step_parity(data, ids, ctx, cfg, delta, do_step=False)
print(os.environ.get("HG_DMX0_SIMT"), {k: v for k, v in res["grad_maxscaled"].items() if "conv0" in k})
