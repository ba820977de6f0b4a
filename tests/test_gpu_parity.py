"""GPU parity: the CUDA path through the C-ABI vs the float64 oracle on the
same seeded inputs (bars: SURVEY §8(c) C19 / BASELINE north_star: forward
1e-4, gradients and one-step parameters 1e-3, packing bit-exact)."""
import numpy as np
import pytest

import oracle as O
from paper_2207_11333_b200 import hgnn
from tests import _parity as PT
from tests._util import make_store

pytestmark = pytest.mark.gpu


def test_device_pack_bit_exact(torch_cuda):
    data = PT.generate("pcqm", 2000, 11)
    ctx, cfg, delta = PT.make_ctx(data, 128, 128, 6)
    ids = O.shard(13, 0, 0, 1, 2000)[:128]
    ctx.pack(ctx._store, ids, 1)
    torch_cuda.cuda.synchronize()
    ref = O.pack(data, ids)
    off = hgnn.hg_batch_offsets(128, len(ref["x"]), len(ref["col"]), cfg.f_node, 4)
    blob = ctx.view(hgnn.VIEW_SLOT, 1)[:off["total"]].cpu().numpy()
    got = hgnn.unpack_blob(blob)
    for k in ("graph_ptr", "y", "rowptr", "col", "x", "eattr", "slot"):
        np.testing.assert_array_equal(np.asarray(got[k]).view(np.uint8), np.asarray(ref[k]).view(np.uint8), err_msg=k)
    got2 = ctx.batch_get(1)  # the same blob through hg_batch_get
    for k in ("graph_ptr", "y", "rowptr", "col", "x", "eattr", "slot"):
        np.testing.assert_array_equal(np.asarray(got2[k]).view(np.uint8), np.asarray(ref[k]).view(np.uint8), err_msg=k)


def test_config_a_every_step_of_an_epoch(torch_cuda):
    """BASELINE configs[0]: 1,000 molecules (<=20 atoms), L=2, H=32, batch 64, one
    epoch (15 steps, 40 dropped) with per-step re-sync (SURVEY §8(d) protocol)."""
    data = PT.generate("tiny", 1000, 1)
    ctx, cfg, delta = PT.make_ctx(data, 64, 32, 2, seed=2)
    ids = O.shard(3, 0, 0, 1, 1000)
    assert len(ids) // 64 == 15
    worst = {}
    for k in range(15):
        res = PT.run_step_parity(data, ids[k * 64:(k + 1) * 64], ctx, cfg, delta)
        PT.assert_parity(res)
        for key in ("yhat", "X"):
            worst[key] = max(worst.get(key, 0), res[key])
    print("config A worst", worst)


def test_config_a_free_running_epoch(torch_cuda):
    """Both sides run the 15-step epoch independently from identical init;
    final parameters normwise <= 1e-3 per tensor."""
    data = PT.generate("tiny", 1000, 1)
    ctx, cfg, delta = PT.make_ctx(data, 64, 32, 2, seed=2)
    ids = O.shard(3, 0, 0, 1, 1000)
    ocfg = PT.oracle_cfg(cfg)
    params = O.init_params(ocfg, 2)
    st = O.zero_state(params)
    for k in range(15):
        bi = ids[k * 64:(k + 1) * 64]
        ctx.pack(ctx._store, bi, k % 2)
        ctx.train_step(k % 2, graph=False)
        params, st, _, _ = O.train_step(params, st, data, bi, ocfg, delta)
    gp = hgnn.arena_to_dict(ctx.params_get(), ctx.layout)
    for name in params:
        assert PT.normwise(gp[name], params[name]) <= 1e-3, name


@pytest.mark.parametrize("preset,B,H,L", [
    ("pcqm", 128, 128, 6),   # BASELINE configs[1] workload: the bench's launch configuration
    ("aisd", 64, 128, 3),    # AISD-shaped molecules (F0 = 9)
    ("pcqm", 16, 256, 2),    # two 128-channel chunks per node
    ("tiny", 7, 64, 2),      # H not a multiple of 128 (one channel per lane), ragged batch
    ("tiny", 300, 128, 2),   # 128-row tiles with a ragged last tile, many tiny graphs
    ("aisd", 512, 128, 6),   # BASELINE configs[3] (D) at its full per-GPU size: N ~ 27 k, N=64 tiles
    ("aisd", 48, 256, 8),    # configs[4] shape (E, H=256, 8 layers), reduced batch: N=128 tiles
    ("aisd", 16, 512, 8),    # configs[4] shape (E, H=512, 8 layers), reduced batch
])
def test_one_step_parity(torch_cuda, preset, B, H, L):
    data = PT.generate(preset, max(600, 4 * B), 21)
    ctx, cfg, delta = PT.make_ctx(data, B, H, L, seed=5)
    ids = O.shard(23, 1, 0, 1, len(data["y"]))[:B]
    res = PT.run_step_parity(data, ids, ctx, cfg, delta)
    print(preset, B, H, L, {k: (max(v.values()) if isinstance(v, dict) else v) for k, v in res.items()})
    PT.assert_parity(res)


@pytest.mark.parametrize("max_degree", [None, 127])
def test_class_slot_capacities_agree(torch_cuda, max_degree):
    """The degree-class GEMMs with exactly the store's degree range (5 class slots) and with
    the full HG_MAX_DEGREE capacity (32 slots, class-indexed weights prepared per batch)
    compute the same step within the oracle bars (config B shape)."""
    data = PT.generate("pcqm", 600, 51)
    ids = O.shard(5, 0, 0, 1, 600)[:128]
    ctx, cfg, delta = PT.make_ctx(data, 128, 128, 6, seed=7, max_degree=max_degree)
    res = PT.run_step_parity(data, ids, ctx, cfg, delta, do_step=False)
    print(max_degree, {k: (max(v.values()) if isinstance(v, dict) else v) for k, v in res.items()})
    PT.assert_parity(res)


def _edge_case_store():
    rng = np.random.default_rng(0)
    F = 5
    graphs = [
        (rng.integers(0, 3, (1, F)).astype(np.float32), [], 1.0),                      # single isolated node
        (rng.integers(0, 3, (4, F)).astype(np.float32), [(0, 1, [1, 0, 0, 0])], 2.0),  # 2 isolated + 1 bond
        (rng.integers(0, 3, (128, F)).astype(np.float32),
         [(0, i, [0, 1, 0, 0]) for i in range(1, 128)], 3.0),                           # degree-127 hub
        (rng.integers(0, 3, (6, F)).astype(np.float32),
         [(0, 1, [1, 0, 0, 0]), (1, 2, [0, 0, 1, 0]), (3, 4, [0, 0, 0, 1]), (4, 5, [1, 0, 0, 0])], 4.0),
        (rng.integers(0, 3, (5, F)).astype(np.float32),                                # 4-cycle + pendant:
         [(0, 1, [1, 0, 0, 0]), (1, 2, [1, 0, 0, 0]), (2, 3, [1, 0, 0, 0]), (3, 0, [1, 0, 0, 0]),
          (0, 4, [0, 0, 0, 1])], 5.0),                                                  # automorphic ties
        (rng.integers(0, 3, (200, F)).astype(np.float32),                              # 200-node ring with
         [(i, (i + 1) % 200, [0, 0, 1, 0]) for i in range(200)] + [(0, 100, [1, 0, 0, 0])], 6.0),  # a chord: too
    ]                                                                                   # large to stage
    data = make_store(graphs, f_edge=4)
    data["f_node"] = F
    return data


@pytest.mark.parametrize("H", [32, 55, 128, 256])
def test_edge_cases_isolated_nodes_single_graph_max_degree(torch_cuda, H):
    """d = 0 nodes (C5), single-node graphs, a degree-127 hub (HG_MAX_DEGREE), a disconnected
    graph, automorphic ties and a 200-node graph (larger than the aggregation kernels' shared-
    memory staging: their global-memory path) in one ragged batch, through the product path:
    tcgen05 degree classes (the hub is its own class), at padded (32, 55 -> 128), native (128:
    fused dX -> dA kernel) and wide (256: separate dX / dA kernels) widths."""
    data = _edge_case_store()
    ctx, cfg, delta = PT.make_ctx(data, 6, H, 2, seed=9)
    res = PT.run_step_parity(data, [0, 1, 2, 3, 4, 5], ctx, cfg, delta)
    print(H, {k: (max(v.values()) if isinstance(v, dict) else v) for k, v in res.items()})
    PT.assert_parity(res)
    res = PT.run_step_parity(data, [2], ctx, cfg, delta)  # the hub alone
    PT.assert_parity(res)
    res = PT.run_step_parity(data, [5, 3], ctx, cfg, delta)  # the large graph first
    PT.assert_parity(res)
    res = PT.run_step_parity(data, [0], ctx, cfg, delta)  # one isolated node: every aggregate 0
    PT.assert_parity(res)


def test_too_many_distinct_degrees_rejected(torch_cuda):
    """A batch needs one degree class per distinct degree: more than the ctx's class slots
    (min(max_degree + 1, 32)) is rejected at pack time (HG_E_DEGREE), not computed wrongly."""
    graphs = []
    for d in range(1, 40):  # stars of every degree 1..39
        graphs.append((np.ones((d + 1, 2), np.float32), [(0, i, [1, 0, 0, 0]) for i in range(1, d + 1)], 1.0))
    data = make_store(graphs, f_edge=4)
    data["f_node"] = 2
    ctx, cfg, delta = PT.make_ctx(data, 39, 128, 1, seed=1, max_degree=127)
    with pytest.raises(hgnn.HgError) as e:
        ctx.pack(ctx._store, list(range(39)), 0)
    assert e.value.name == "HG_E_DEGREE"
    ctx.pack(ctx._store, list(range(30)), 0)  # 31 distinct degrees (1..30 and 1 for leaves): fits
    PT.assert_parity(PT.run_step_parity(data, list(range(30)), ctx, cfg, delta))


def test_graph_mode_matches_eager_bitwise(torch_cuda):
    data = PT.generate("pcqm", 600, 31)
    ids = O.shard(1, 0, 0, 1, 600)[:128]
    outs = []
    for graph in (False, True):
        ctx, cfg, delta = PT.make_ctx(data, 128, 128, 6, seed=3)
        for _ in range(2):
            ctx.pack(ctx._store, ids, 0)
            ctx.train_step(0, graph=graph)
        torch_cuda.cuda.synchronize()
        outs.append((ctx.params_get(), ctx.grads_get()))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


def test_determinism_and_batch_independence_bitwise(torch_cuda):
    """Run-to-run bitwise equality (no float atomics), and a graph's prediction
    is bitwise independent of its batch-mates (SURVEY P7 on GPU)."""
    data = PT.generate("pcqm", 600, 41)
    ids = O.shard(2, 0, 0, 1, 600)[:128]
    ctx, cfg, delta = PT.make_ctx(data, 128, 128, 6, seed=4)
    res = []
    for _ in range(2):
        ctx.pack(ctx._store, ids, 0)
        ctx.forward(0)
        ctx.backward(0)
        torch_cuda.cuda.synchronize()
        res.append((ctx.view_f32(hgnn.VIEW_YHAT)[:128].cpu().numpy().copy(), ctx.grads_get()))
    np.testing.assert_array_equal(res[0][0], res[1][0])
    np.testing.assert_array_equal(res[0][1], res[1][1])
    sub = ids[[5, 77, 3]]
    ctx.pack(ctx._store, sub, 1)
    ctx.forward(1)
    torch_cuda.cuda.synchronize()
    y3 = ctx.view_f32(hgnn.VIEW_YHAT)[:3].cpu().numpy()
    np.testing.assert_array_equal(y3, res[0][0][[5, 77, 3]])


def test_errors_surface_through_the_abi(torch_cuda):
    data = PT.generate("tiny", 200, 3)
    ctx, cfg, delta = PT.make_ctx(data, 8, 32, 2)
    with pytest.raises(hgnn.HgError) as e:
        ctx.forward(5)
    assert e.value.name == "HG_E_RANGE"
    with pytest.raises(hgnn.HgError) as e:
        ctx.pack(ctx._store, list(range(9)), 0)
    assert e.value.name == "HG_E_CAPACITY"
    ctx.pack(ctx._store, list(range(8)), 0)
    ctx.train_step(0)
    ctx.sync()
    assert ctx.launch_count() > 0


@pytest.mark.gpu
def test_pipelined_loss_readback_matches_sync_read(torch_cuda):
    """hg_loss_enqueue / hg_loss_fetch return exactly what hg_loss_get reads, one step later."""
    data = PT.generate("tiny", 300, 4)
    ctx, cfg, delta = PT.make_ctx(data, 16, 128, 2)
    hyper = dict(hgnn.DEFAULT_ADAMW)
    ids = list(range(16))
    ctx.pack(ctx._store, ids, 0)
    sync_losses, ring = [], []
    for k in range(5):
        ctx.train_step(0, graph=True, **hyper)
        ctx.loss_enqueue(k % hgnn.HG_LOSS_RING)
        sync_losses.append(ctx.loss())
        ring.append(ctx.loss_fetch(k % hgnn.HG_LOSS_RING))
    assert ring == sync_losses
    with pytest.raises(hgnn.HgError) as e:
        ctx.loss_enqueue(hgnn.HG_LOSS_RING)
    assert e.value.name == "HG_E_RANGE"


def test_small_batch_after_large_batch_class_path(torch_cuda):
    """Split-K partial buffers are reused across batches: a small batch (most node
    splits empty) after a large one must not pick up stale partials (class path)."""
    data = PT.generate("pcqm", 800, 33)
    ctx, cfg, delta = PT.make_ctx(data, 128, 128, 3, seed=9)
    big = O.shard(2, 0, 0, 1, len(data["y"]))[:128]
    PT.assert_parity(PT.run_step_parity(data, big, ctx, cfg, delta))
    small = O.shard(2, 1, 0, 1, len(data["y"]))[:3]
    res = PT.run_step_parity(data, small, ctx, cfg, delta)
    print({k: (max(v.values()) if isinstance(v, dict) else v) for k, v in res.items()})
    PT.assert_parity(res)


def test_separate_dx_da_path_wide(torch_cuda):
    """H = 256 runs the separate TMA dX and dA kernels (the fused kernel is H = 128 only)."""
    data = PT.generate("pcqm", 600, 21)
    ctx, cfg, delta = PT.make_ctx(data, 64, 256, 3, seed=5)
    ids = O.shard(23, 1, 0, 1, len(data["y"]))[:64]
    res = PT.run_step_parity(data, ids, ctx, cfg, delta)
    print({k: (max(v.values()) if isinstance(v, dict) else v) for k, v in res.items()})
    PT.assert_parity(res)


def test_many_graphs_per_batch(torch_cuda):
    """A batch of 320 small graphs: more (graph, 64-channel chunk) aggregation items than two
    waves of resident CTAs (maxB x H/64 > 592), two graph steps."""
    data = PT.generate("tiny", 1200, 4)
    B = 320
    assert B * (128 // 64) > 2 * 2 * 148
    ctx, cfg, delta = PT.make_ctx(data, B, 128, 2, seed=3)
    ids = O.shard(5, 0, 0, 1, 1200)
    for k in range(2):
        res = PT.run_step_parity(data, ids[k * B:(k + 1) * B], ctx, cfg, delta, graph=(k == 1))
        print("many graphs", k, {kk: (max(v.values()) if isinstance(v, dict) else v) for kk, v in res.items()})
        PT.assert_parity(res)
