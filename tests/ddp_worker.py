"""torchrun worker for tests/test_gpu_ddp.py: W ranks (one GPU each) run one
training step on disjoint equal sub-batches through the C-ABI with the NCCL
gradient mean (hg_allreduce_grads); rank 0 compares the
averaged gradient with the float64 oracle's gradient of the union batch
(SURVEY P8 on GPU) and every rank reports its parameters after AdamW."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import molgen  # noqa: E402
import oracle as O  # noqa: E402
from paper_2207_11333_b200 import hgnn  # noqa: E402
from tests._util import max_scaled, normwise  # noqa: E402


def main(out):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{lr}"))
    data = molgen.generate("pcqm", 800, 21)
    store = hgnn.Store(data)
    delta = O.degree_stat(data)
    Bg = 32 * world
    Bl = Bg // world
    nn = np.diff(data["node_offset"])
    ne = np.diff(data["edge_offset"])
    cfg = hgnn.make_config(data["f_node"], 4, 128, 3, Bl, int(np.sort(nn)[-Bl:].sum()), int(np.sort(ne)[-Bl:].sum()),
                           delta, max_degree=store.stats()["max_degree"])
    ctx = hgnn.Context(cfg, device=lr)
    ctx.params_init(5)
    ctx.comm_init(rank, world)
    batch = O.shard(9, 0, 0, 1, 800)[:Bg]
    mine = batch[rank * Bl:(rank + 1) * Bl]
    p0 = hgnn.arena_to_dict(ctx.params_get(), ctx.layout)
    ctx.pack(store, mine, 0)
    ctx.forward(0)
    ctx.backward(0)
    ctx.allreduce_grads()
    ctx.sync()
    g = hgnn.arena_to_dict(ctx.grads_get(), ctx.layout)
    ctx.step()
    ctx.sync()
    # one more step through the captured graph (allreduce inside the graph)
    ctx.pack(store, batch[(world + rank) * Bl % Bg:(world + rank) * Bl % Bg + Bl], 1)
    ctx.train_step(1, graph=True)
    ctx.sync()
    params = torch.from_numpy(ctx.params_get()).cuda()
    allp = [torch.zeros_like(params) for _ in range(world)]
    dist.all_gather(allp, params)
    same = all(torch.equal(allp[0], t) for t in allp)
    res = {"rank": rank, "params_identical": bool(same)}
    if rank == 0:
        ocfg = {"f_node": cfg.f_node, "f_edge": 4, "hidden": 128, "layers": 3, "fc_hidden": 128}
        pd = {k: np.asarray(v, np.float64) for k, v in p0.items()}
        b = O.pack(data, batch)
        _, _, cache = O.forward(pd, b, ocfg, delta)
        go = O.backward(pd, b, ocfg, cache)
        res["grad_maxscaled"] = max(max_scaled(g[k], go[k]) for k in go)
        res["grad_normwise"] = max(normwise(g[k], go[k]) for k in go)
        with open(out, "w") as f:
            json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()
    if not same:
        sys.exit(3)


if __name__ == "__main__":
    main(sys.argv[1])
