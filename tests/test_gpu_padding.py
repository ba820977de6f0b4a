"""Channel-padded widths (the paper's own H = 55 and H = 200):
the kernels run at the internal width of hg_config_internal (roundup to 128, the
tensor-core tile) and must compute the logical model exactly (SURVEY §8(d)
"Padding hazard"): parity against the float64 oracle at the logical width, and
every padded parameter / gradient / Adam-moment entry exactly zero after
training steps."""
import numpy as np
import pytest

import oracle as O
from paper_2207_11333_b200 import hgnn
from tests import _parity as PT

pytestmark = pytest.mark.gpu


def padded_index(cfg, icfg):
    """Logical arena position -> internal arena position (test-side restatement of
    the include/hgnn.h hg_config_internal contract: rows keep their index, column
    q*W + c of a tensor with nb column blocks of width W moves to q*Wp + c; nb = 12
    for U, whose columns are (s*4+a)*H + c)."""
    ll, nl = hgnn.hg_param_layout(cfg)
    lp, npad = hgnn.hg_param_layout(icfg)
    src, dst = [], []
    for (name, off, r, c), (name2, off2, r2, c2) in zip(ll, lp):
        assert name == name2
        nb = 12 if name.endswith(".U") else 1
        W, Wp = c // nb, c2 // nb
        rr, qq, cc = np.meshgrid(np.arange(r), np.arange(nb), np.arange(W), indexing="ij")
        src.append(off + (rr * c + qq * W + cc).ravel())
        dst.append(off2 + (rr * c2 + qq * Wp + cc).ravel())
    return np.concatenate(src), np.concatenate(dst), npad


@pytest.mark.parametrize("H,L,B", [
    (55, 2, 64),     # paper width -> 128 channels
    (200, 2, 32),    # paper width -> 256 channels
    (32, 2, 64),     # config A's width -> 128 channels
    (100, 3, 48),    # another ragged width, deeper
])
def test_padded_width_parity_and_zero_padding(torch_cuda, H, L, B):
    flags = 0
    data = PT.generate("pcqm", 800, 31)
    ctx, cfg, delta = PT.make_ctx(data, B, H, L, seed=7)
    icfg = ctx.internal_cfg
    q = 128
    assert icfg.hidden == (H + q - 1) // q * q and icfg.fc_hidden == icfg.hidden
    ids = O.shard(17, 0, 0, 1, len(data["y"]))
    # per-step parity at the logical width (3 steps: moments become non-zero)
    for k in range(3):
        res = PT.run_step_parity(data, ids[k * B:(k + 1) * B], ctx, cfg, delta)
        print(H, flags, k, res["overrides_by"], {kk: (max(v.values()) if isinstance(v, dict) else v) for kk, v in res.items()})
        PT.assert_parity(res)
    # graph-replayed steps, then the internal arenas: logical image == public get,
    # everything else exactly zero
    for k in range(3, 6):
        ctx.pack(ctx._store, ids[k * B:(k + 1) * B], k % 2)
        ctx.train_step(k % 2, graph=True)
    torch_cuda.cuda.synchronize()
    src, idx, npad = padded_index(cfg, icfg)
    pad_mask = np.ones(npad, bool)
    pad_mask[idx] = False
    for what, public in ((hgnn.VIEW_PARAMS, ctx.params_get()), (hgnn.VIEW_GRADS, ctx.grads_get())):
        arena = ctx.view_f32(what)[:npad].cpu().numpy()
        np.testing.assert_array_equal(arena[idx], public[src])
        assert not np.any(arena[pad_mask]), f"non-zero padded entries in view {what}"
    m, v, _ = ctx.opt_state_get()
    assert np.any(m) and np.any(v)
    # the padded X channels are exactly zero
    N = int(np.diff(data["node_offset"])[ids[5 * B:6 * B]].sum())
    Hp = icfg.hidden
    for l in range(L):
        X = ctx.view_f32(hgnn.VIEW_X, l)[:N * Hp].cpu().numpy().reshape(N, Hp)
        assert not np.any(X[:, H:])


def test_padded_set_get_roundtrip(torch_cuda):
    data = PT.generate("tiny", 300, 3)
    ctx, cfg, _ = PT.make_ctx(data, 32, 55, 2, seed=1)
    rng = np.random.default_rng(0)
    p = hgnn.dict_to_arena({name: rng.standard_normal(r * c) for name, off, r, c in ctx.layout}, ctx.layout,
                           ctx.n_params)  # alignment gaps between tensors stay zero
    ctx.params_set(p)
    np.testing.assert_array_equal(ctx.params_get(), p)
    np.testing.assert_array_equal(ctx.params_get(), p)
    ref = hgnn.hg_params_init_host(cfg, 9)
    ctx.params_init(9)
    np.testing.assert_array_equal(ctx.params_get(), ref)
