"""world_size-2 tests of the multi-rank host logic on CPU (gloo backend):
per-epoch sharding across ranks, the NCCL
unique-id rendezvous over torch.distributed, and the DDP gradient-mean
semantics with the oracle."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import molgen
    import oracle as O
    from paper_2207_11333_b200 import hgnn
    res = {}
    # (1) shards: disjoint, equal size, union = drop-last prefix of the permutation
    n = 1003
    ids = hgnn.hg_shard(17, 2, rank, world, n)
    np.testing.assert_array_equal(ids, O.shard(17, 2, rank, world, n))
    allids = [torch.zeros(len(ids), dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allids, torch.from_numpy(ids))
    u = torch.cat(allids).numpy()
    res["shard_ok"] = len(np.unique(u)) == world * (n // world)
    # (2) NCCL unique id broadcast: identical bytes on every rank
    uid = hgnn.nccl_unique_id_broadcast(rank, world)
    ids_all = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(ids_all, torch.from_numpy(uid))
    res["uid_ok"] = all(torch.equal(ids_all[0], t) for t in ids_all) and int(ids_all[0].sum()) > 0
    # (3) DDP mean: per-rank oracle gradients on equal sub-batches, averaged over
    # the process group, equal the single-process gradient of the union batch
    data = molgen.generate("tiny", 200, seed=4)
    cfg = {"f_node": data["f_node"], "f_edge": 4, "hidden": 8, "layers": 2, "fc_hidden": 8}
    p = O.init_params(cfg, 3)
    delta = O.degree_stat(data)
    batch = O.shard(5, 0, 0, 1, 200)[:16]
    mine = batch[rank * 8:(rank + 1) * 8]
    b = O.pack(data, mine)
    _, _, cache = O.forward(p, b, cfg, delta)
    g = O.backward(p, b, cfg, cache)
    worst = 0.0
    bf = O.pack(data, batch)
    _, _, cf = O.forward(p, bf, cfg, delta)
    gfull = O.backward(p, bf, cfg, cf)
    for k in sorted(g):
        t = torch.from_numpy(np.ascontiguousarray(g[k], np.float64))
        dist.all_reduce(t)
        t /= world
        worst = max(worst, float(np.abs(t.numpy() - gfull[k]).max() / max(np.abs(gfull[k]).max(), 1e-30)))
    res["ddp_worst"] = worst
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array([res["shard_ok"], res["uid_ok"], worst], np.float64))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_host_logic_gloo(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        shard_ok, uid_ok, worst = np.load(tmp_path / f"r{r}.npy")
        assert shard_ok == 1.0 and uid_ok == 1.0
        assert worst <= 1e-12
