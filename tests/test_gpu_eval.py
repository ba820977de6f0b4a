"""GPU evaluation path (hg_eval_*) vs the oracle's evaluate."""
import numpy as np
import pytest

import oracle as O
from paper_2207_11333_b200 import hgnn
from tests import _parity as PT


@pytest.mark.gpu
@pytest.mark.parametrize("H,graph", [(32, False), (128, True), (128, False)])
def test_eval_matches_oracle(torch_cuda, H, graph):
    data = PT.generate("tiny", 300, 8)
    B = 24
    ctx, cfg, delta = PT.make_ctx(data, B, H, 2, seed=5)
    ocfg = PT.oracle_cfg(cfg)
    p0 = ctx.params_get()
    params = {k: np.asarray(v, np.float64) for k, v in hgnn.arena_to_dict(p0, ctx.layout).items()}
    batches = [list(range(k * B, (k + 1) * B)) for k in range(3)]
    ref = O.evaluate(params, data, batches, ocfg, delta)
    ctx.eval_reset()
    pairs = []
    for k, ids in enumerate(batches):
        ctx.pack(ctx._store, ids, k % 2)
        ctx.eval_batch(k % 2, graph=graph)
        pairs.append(ctx.eval_pairs(k % 2))
    res = ctx.eval_result()
    assert res["count"] == 3 * B
    assert abs(res["mse"] - ref["mse"]) <= PT.FWD_TOL * ref["mse"]
    assert abs(res["mae"] - ref["mae"]) <= PT.FWD_TOL * ref["mae"]
    pairs = np.concatenate(pairs)
    np.testing.assert_array_equal(pairs[:, 0], ref["pairs"][:, 0].astype(np.float32))
    yh_ref = ref["pairs"][:, 1]
    assert np.max(np.abs(pairs[:, 1] - yh_ref)) <= PT.FWD_TOL * np.max(np.abs(yh_ref))
    # evaluation does not touch the parameters
    np.testing.assert_array_equal(ctx.params_get(), p0)


@pytest.mark.gpu
def test_eval_empty_is_an_error(torch_cuda):
    data = PT.generate("tiny", 100, 2)
    ctx, cfg, delta = PT.make_ctx(data, 8, 32, 2)
    ctx.eval_reset()
    with pytest.raises(hgnn.HgError) as e:
        ctx.eval_result()
    assert e.value.name == "HG_E_EMPTY"
