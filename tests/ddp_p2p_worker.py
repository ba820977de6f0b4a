"""torchrun worker for tests/test_gpu_ddp.py (peer-memory gradient exchange,
include/hgnn.h hg_p2p_open). Two contexts per rank start from
the same parameters: one takes K graph-replayed steps with the bucketed NCCL
allreduce + AdamW, the other the same K steps with the fused peer-memory
reduce -> sharded AdamW -> all-gather kernel. Reports: parameters bitwise
identical across ranks (both paths), the two paths' parameters per tensor
(normwise), and the P2P path's first-step parameters against the float64
oracle's full-batch AdamW step (DDP mean == union-batch gradient)."""
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
from tests._util import normwise  # noqa: E402

K = 4


def main(out):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{lr}"))
    data = molgen.generate("pcqm", 1200, 21)
    store = hgnn.Store(data)
    delta = O.degree_stat(data)
    Bl = 32
    Bg = Bl * world
    nn = np.diff(data["node_offset"])
    ne = np.diff(data["edge_offset"])
    cfg = hgnn.make_config(data["f_node"], 4, 128, 3, Bl, int(np.sort(nn)[-Bl:].sum()), int(np.sort(ne)[-Bl:].sum()),
                           delta, max_degree=store.stats()["max_degree"])
    order = O.shard(9, 0, 0, 1, 1200)
    batches = [order[k * Bg:(k + 1) * Bg] for k in range(K)]
    params = {}
    for mode in ("nccl", "p2p"):
        ctx = hgnn.Context(cfg, device=lr)
        ctx.params_init(5)
        ctx.comm_init(rank, world)
        if mode == "p2p":
            ctx.p2p_init(rank, world)
        p0 = hgnn.arena_to_dict(ctx.params_get(), ctx.layout)
        for k, bg in enumerate(batches):
            ctx.pack(store, bg[rank * Bl:(rank + 1) * Bl], k % 2)
            ctx.train_step(k % 2, graph=True)
            ctx.sync()
            if k == 0:
                params[mode + "_1"] = ctx.params_get()
        params[mode] = ctx.params_get()
        if mode == "p2p":
            # back to the NCCL exchange mid-run: the sharded moments are gathered,
            # then every rank must keep bitwise-identical parameters and moments
            ctx.p2p_close()
            for k in range(2):
                bg = order[(K + k) * Bg:(K + k + 1) * Bg]
                ctx.pack(store, bg[rank * Bl:(rank + 1) * Bl], k % 2)
                ctx.train_step(k % 2, graph=True)
                ctx.sync()
            m, v, _ = ctx.opt_state_get()
            params["switched"] = np.concatenate([ctx.params_get(), m, v])
        del ctx
    res = {"rank": rank}
    for mode in ("nccl", "p2p", "switched"):
        t = torch.from_numpy(params[mode]).cuda()
        allp = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allp, t)
        res[mode + "_identical"] = bool(all(torch.equal(allp[0], a) for a in allp))
    lay = hgnn.hg_param_layout(cfg)[0]
    a, b = hgnn.arena_to_dict(params["nccl"], lay), hgnn.arena_to_dict(params["p2p"], lay)
    res["p2p_vs_nccl_normwise"] = max(normwise(b[k], a[k]) for k in a)
    res["p2p_vs_nccl_bitwise"] = bool(np.array_equal(params["nccl"].view(np.uint32), params["p2p"].view(np.uint32)))
    if rank == 0:
        ocfg = {"f_node": cfg.f_node, "f_edge": 4, "hidden": 128, "layers": 3, "fc_hidden": 128}
        pd = {k: np.asarray(v, np.float64) for k, v in p0.items()}
        st = O.zero_state(pd)
        newp, _, _, _ = O.train_step(pd, st, data, batches[0], ocfg, delta, world=world)
        g1 = hgnn.arena_to_dict(params["p2p_1"], lay)
        n1 = hgnn.arena_to_dict(params["nccl_1"], lay)
        res["p2p_step1_vs_oracle_normwise"] = max(normwise(g1[k], newp[k]) for k in newp)
        res["nccl_step1_vs_oracle_normwise"] = max(normwise(n1[k], newp[k]) for k in newp)
        res["step1_p2p_vs_nccl"] = {k: normwise(g1[k], n1[k]) for k in newp}
        res["step1_bitwise"] = bool(np.array_equal(params["nccl_1"].view(np.uint32), params["p2p_1"].view(np.uint32)))
        with open(out, "w") as f:
            json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
