"""The data-parallel gradient exchange on ONE GPU (
PAPER.md:206-212 "gradients are aggregated ... after each backward pass"; SPEC.md:454,
463-464 parameter consistency and averaging equivalence).

- The fused peer-memory exchange (reduce-scatter -> sharded AdamW -> all-gather, the
  k_p2p_signal / k_p2p_adamw kernels of hg_p2p_open's captured step) with W ranks emulated
  as W contexts of one process (hg_p2p_emulate; ranks that spin on one another must not share
  a GPU, so the emulation runs the ranks' kernels back to back with the flag waits elided):
  parameters bitwise identical across ranks, equal to the float64 oracle's W-rank DDP step
  (oracle.train_step(world=W), itself pinned to the union-batch step by P8) within the C19
  bars, and close to one context stepping the union batch; the sharded Adam moments are
  gathered back whole (hg_opt_state_get / hg_step after peer-memory steps).
- The bucketed NCCL path with a one-rank communicator (no world-1 short-circuit): bitwise
  the parameters of a context without a communicator, graph and eager steps.
The W-process versions of both run in tests/test_gpu_ddp.py (>= 2 GPUs)."""
import numpy as np
import pytest

import oracle as O
from paper_2207_11333_b200 import hgnn
from tests import _parity as PT
from tests._util import normwise

pytestmark = pytest.mark.gpu


def _ctxs(data, W, Bl, H, L):
    delta = O.degree_stat(data)
    maxn, maxe = PT.capacity_for(data, Bl)
    store = hgnn.Store(data)
    cfg = hgnn.make_config(data["f_node"], 4, H, L, Bl, maxn, maxe, delta, max_degree=store.stats()["max_degree"])
    ctxs = []
    for _ in range(W):
        c = hgnn.Context(cfg)
        c.params_init(5)
        ctxs.append(c)
    return ctxs, cfg, delta, store


def _well_conditioned_normwise(gpu, ref, g, params0, t=1, lr=1e-3, wd=0.01, eps=1e-8):
    """C19 one-step parameter bar with reading R-adam-eps (tests/_parity.py): compared where the
    oracle gradient is >= 100 eps and its sign is fixed by the gradient bar; elsewhere the Adam
    step bound of step t."""
    worst, viol = 0.0, 0
    bound = lr * PT.adam_ratio_bound(t, dict(beta1=hgnn.DEFAULT_ADAMW["beta1"], beta2=hgnn.DEFAULT_ADAMW["beta2"]))
    for k in ref:
        ok = np.abs(g[k]) >= max(100 * eps, PT.GRAD_TOL * float(np.abs(g[k]).max()))
        a = np.asarray(gpu[k], np.float64).reshape(ref[k].shape)
        if ok.any():
            worst = max(worst, normwise(a[ok], ref[k][ok]))
        viol += int((np.abs(a[~ok] - params0[k][~ok] * (1 - lr * wd)) > bound * 1.001 + 1e-7).sum())
    return worst, viol


@pytest.mark.parametrize("W,H,L", [(2, 128, 3), (4, 128, 2), (3, 55, 2), (8, 128, 2)])
def test_p2p_exchange_emulated_ranks_match_oracle_ddp_step(torch_cuda, W, H, L):
    data = PT.generate("pcqm", 900, 21)
    Bl = 24
    ctxs, cfg, delta, store = _ctxs(data, W, Bl, H, L)
    order = O.shard(9, 0, 0, 1, len(data["y"]))
    ocfg = PT.oracle_cfg(cfg)
    lay = ctxs[0].layout
    params = {k: np.asarray(v, np.float64) for k, v in hgnn.arena_to_dict(ctxs[0].params_get(), lay).items()}
    st = O.zero_state(params)
    hyper = dict(hgnn.DEFAULT_ADAMW)
    for k in range(3):  # step 1 from zero moments, then steps whose moments were sharded
        bg = order[k * W * Bl:(k + 1) * W * Bl]
        for r, c in enumerate(ctxs):
            c.pack(store, bg[r * Bl:(r + 1) * Bl], 0)
            c.forward(0)
            c.backward(0)
        hgnn.p2p_emulate(ctxs, **hyper)
        got = [c.params_get() for c in ctxs]
        for r in range(1, W):  # every shard reduced once and all-gathered: bitwise agreement
            np.testing.assert_array_equal(got[r].view(np.uint32), got[0].view(np.uint32))
        # the oracle's DDP step (rank sub-batches, gradient mean, AdamW) from the same state
        newp, newst, _, g = O.train_step(params, st, data, bg, ocfg, delta, hyper=hyper, world=W)
        gp = hgnn.arena_to_dict(got[0], lay)
        worst, viol = _well_conditioned_normwise(gp, newp, g, params, t=k + 1)
        print(W, H, k, "param normwise", worst, "bound violations", viol)
        assert worst <= 1e-3 and viol == 0
        # moments: sharded after the exchange; opt_state_get gathers them whole (collective)
        ms = [c.opt_state_get() for c in ctxs]
        for r in range(1, W):
            np.testing.assert_array_equal(ms[r][0], ms[0][0])
            np.testing.assert_array_equal(ms[r][1], ms[0][1])
            assert ms[r][2] == ms[0][2] == k + 1
        gm, gv = hgnn.arena_to_dict(ms[0][0], lay), hgnn.arena_to_dict(ms[0][1], lay)
        assert max(normwise(gm[q], newst["m"][q]) for q in gm) <= 1e-3
        assert max(normwise(gv[q], newst["v"][q]) for q in gv) <= 1e-3
        # next step starts from the GPU state (SURVEY §8(d) per-step re-sync)
        params = {q: np.asarray(v, np.float64) for q, v in gp.items()}
        st = {"m": {q: np.asarray(v, np.float64) for q, v in gm.items()},
              "v": {q: np.asarray(v, np.float64) for q, v in gv.items()}, "step": ms[0][2]}


def test_p2p_emulated_average_equals_union_batch_step(torch_cuda):
    """P8 on the GPU: the mean of W ranks' gradients equals the union batch's gradient (one
    context stepping all W*Bl graphs), and the exchange's parameters equal that context's
    AdamW step -- up to the order of the node sums (normwise, not bitwise)."""
    W, Bl = 2, 32
    data = PT.generate("pcqm", 600, 7)
    ctxs, cfg, delta, store = _ctxs(data, W, Bl, 128, 3)
    maxn, maxe = PT.capacity_for(data, W * Bl)
    big = hgnn.Context(hgnn.make_config(data["f_node"], 4, 128, 3, W * Bl, maxn, maxe, delta,
                                        max_degree=store.stats()["max_degree"]))
    big.params_init(5)
    bg = O.shard(4, 0, 0, 1, len(data["y"]))[:W * Bl]
    grads = []
    for r, c in enumerate(ctxs):
        c.pack(store, bg[r * Bl:(r + 1) * Bl], 0)
        c.forward(0)
        c.backward(0)
        torch_cuda.cuda.synchronize()
        grads.append(c.grads_get().astype(np.float64))
    hgnn.p2p_emulate(ctxs)
    big.pack(store, bg, 0)
    big.forward(0)
    big.backward(0)
    torch_cuda.cuda.synchronize()
    gb = hgnn.arena_to_dict(big.grads_get(), big.layout)
    gm = hgnn.arena_to_dict(np.mean(grads, axis=0), ctxs[0].layout)
    for k in gb:
        assert normwise(gm[k], gb[k]) <= 1e-5, k
    big.step()
    a = hgnn.arena_to_dict(ctxs[0].params_get(), ctxs[0].layout)
    b = hgnn.arena_to_dict(big.params_get(), big.layout)
    for k in a:
        ok = np.abs(gb[k]) >= 1e-6
        if ok.any():
            assert normwise(np.asarray(a[k])[ok], np.asarray(b[k])[ok]) <= 1e-5, k


def test_nccl_bucket_path_one_rank_communicator(torch_cuda):
    """A one-rank NCCL communicator runs the bucketed average (ncclAvg over 1 rank = the
    identity) inside the captured step and in the eager path: parameters bitwise those of a
    context without a communicator."""
    data = PT.generate("pcqm", 500, 3)
    ids = O.shard(2, 0, 0, 1, 500)
    res = []
    for force in (False, True):
        ctxs, cfg, delta, store = _ctxs(data, 1, 32, 128, 3)
        c = ctxs[0]
        c.comm_init(0, 1, force_comm=force)
        for k in range(3):
            c.pack(store, ids[k * 32:(k + 1) * 32], k % 2)
            c.train_step(k % 2, graph=True)
        c.pack(store, ids[96:128], 0)
        c.train_step(0, graph=False)  # eager: forward, backward, hg_allreduce_grads, hg_step
        c.sync()
        res.append(c.params_get())
    np.testing.assert_array_equal(res[0].view(np.uint32), res[1].view(np.uint32))


def test_fail_stop_timeout_setting(torch_cuda):
    data = PT.generate("tiny", 200, 3)
    ctxs, cfg, delta, store = _ctxs(data, 1, 8, 128, 2)
    c = ctxs[0]
    c.set_timeout(5.0)
    c.pack(store, list(range(8)), 0)
    c.train_step(0, graph=True)
    c.sync()  # completes well within the bound
    with pytest.raises(hgnn.HgError) as e:
        c.set_timeout(-1.0)
    assert e.value.name == "HG_E_INVALID"
