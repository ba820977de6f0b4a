"""C-ABI host-side tests (no GPU): the library loads, exports every symbol
include/hgnn.h declares, and its host logic (store validation, shard, collate,
degree statistic, parameter init) matches the oracle bit-exactly."""
import ctypes
import os
import re

import numpy as np
import pytest

import molgen
import oracle as O
from paper_2207_11333_b200 import hgnn
from tests._util import make_store

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "hgnn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = hgnn.load()
    decl = _declared_symbols()
    assert len(decl) >= 30
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(hgnn.SIGNATURES), set(decl) ^ set(hgnn.SIGNATURES)
    assert lib.hg_abi_version() == 2


@pytest.fixture(scope="module")
def tiny():
    return molgen.generate("tiny", 1000, seed=1)


@pytest.fixture(scope="module")
def pcqm():
    return molgen.generate("pcqm", 3000, seed=11)


@pytest.mark.parametrize("seed,epoch,world,n", [(3, 0, 1, 1000), (3, 1, 3, 10), (7, 2, 8, 12345), (0, 0, 2, 1)])
def test_shard_bit_exact_vs_oracle(seed, epoch, world, n):
    for rank in range(world):
        np.testing.assert_array_equal(hgnn.hg_shard(seed, epoch, rank, world, n), O.shard(seed, epoch, rank, world, n))


def test_shard_errors():
    with pytest.raises(hgnn.HgError) as e:
        hgnn.hg_shard(1, 0, 2, 2, 10)
    assert e.value.name == "HG_E_INVALID"


def _cfg_for(data, B, H=32, L=2, maxn=None):
    nn = np.diff(data["node_offset"])
    ne = np.diff(data["edge_offset"])
    return hgnn.make_config(data["f_node"], 4, H, L, B, int(maxn or nn.max() * B), int(ne.max() * B), 1.0)


@pytest.mark.parametrize("which", ["tiny", "pcqm"])
def test_pack_bit_exact_vs_oracle(which, tiny, pcqm):
    data = tiny if which == "tiny" else pcqm
    store = hgnn.Store(data)
    n = len(data["y"])
    B = 64 if which == "tiny" else 128
    cfg = _cfg_for(data, B)
    ids = O.shard(3, 0, 0, 1, n)[:B]
    blob = hgnn.hg_pack_host(store, ids, cfg)
    got = hgnn.unpack_blob(blob)
    ref = O.pack(data, ids)
    for k in ("graph_ptr", "y", "rowptr", "col", "x", "eattr", "slot"):
        a, b = np.asarray(got[k]), np.asarray(ref[k])
        assert a.dtype == b.dtype, k
        np.testing.assert_array_equal(a.view(np.uint8), b.view(np.uint8), err_msg=k)  # bitwise
    assert got["B"] == B and got["N"] == len(ref["x"]) and got["E"] == len(ref["col"])


def test_pack_errors(tiny):
    store = hgnn.Store(tiny)
    cfg = _cfg_for(tiny, 8)
    with pytest.raises(hgnn.HgError) as e:
        hgnn.hg_pack_host(store, [], cfg)
    assert e.value.name == "HG_E_EMPTY"
    with pytest.raises(hgnn.HgError) as e:
        hgnn.hg_pack_host(store, [0, 10 ** 6], cfg)
    assert e.value.name == "HG_E_RANGE"
    with pytest.raises(hgnn.HgError) as e:
        hgnn.hg_pack_host(store, list(range(9)), cfg)
    assert e.value.name == "HG_E_CAPACITY"
    bad = hgnn.make_config(tiny["f_node"] + 1, 4, 32, 2, 8, 400, 800, 1.0)
    with pytest.raises(hgnn.HgError) as e:
        hgnn.hg_pack_host(store, [0], bad)
    assert e.value.name == "HG_E_SHAPE"


def test_store_validation_errors():
    good = make_store([(np.zeros((3, 2)), [(0, 1, [1.0, 0.0]), (1, 2, [0.0, 1.0])], 0.0)])
    hgnn.Store(good)
    d = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in good.items()}
    d["edge_attr"][0, 0] = 5.0  # 0->1 attr differs from 1->0
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store(d)
    assert e.value.name == "HG_E_ASYMMETRIC"
    d = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in good.items()}
    d["edge_index"] = d["edge_index"][:, ::-1].copy()
    d["edge_attr"] = d["edge_attr"][::-1].copy()
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store(d)
    assert e.value.name == "HG_E_UNSORTED"
    d = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in good.items()}
    d["edge_index"][1, 0] = 7
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store(d)
    assert e.value.name == "HG_E_RANGE"
    star = make_store([(np.zeros((130, 1)), [(0, i, [1.0]) for i in range(1, 130)], 0.0)])
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store(star)
    assert e.value.name == "HG_E_DEGREE"
    empty = make_store([(np.zeros((2, 1)), [], 0.0)])
    empty["node_offset"] = np.array([0, 0, 2], np.int64)
    empty["edge_offset"] = np.array([0, 0, 0], np.int64)
    empty["y"] = np.zeros(2, np.float32)
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store(empty)
    assert e.value.name == "HG_E_EMPTY"


def test_store_stats_and_degree_stat(pcqm):
    store = hgnn.Store(pcqm)
    s = store.stats()
    assert s["graphs"] == 3000 and s["nodes"] == pcqm["node_offset"][-1] and s["edges"] == pcqm["edge_offset"][-1]
    assert s["max_nodes_per_graph"] == np.diff(pcqm["node_offset"]).max() and 1 <= s["max_degree"] <= 8
    assert abs(store.degree_stat() - O.degree_stat(pcqm)) <= 1e-13
    ids = np.arange(0, 3000, 7)
    assert abs(store.degree_stat(ids) - O.degree_stat(pcqm, ids)) <= 1e-13


@pytest.mark.parametrize("H,Hf,Hp,Hfp", [
    (55, 55, 128, 128),     # paper width -> tensor-core tile
    (200, 200, 256, 256),   # paper width
    (32, 32, 128, 128),     # config A's width
    (55, 40, 128, 40),      # fc_hidden != hidden is left as given
    (128, 128, 128, 128),   # multiples of 128 are not padded
    (96, 96, 128, 128),
    (512, 512, 512, 512),
])
def test_config_internal_padding(H, Hf, Hp, Hfp):
    cfg = hgnn.make_config(34, 4, H, 2, 4, 100, 400, 1.0, fc_hidden=Hf)
    ic = hgnn.hg_config_internal(cfg)
    assert (ic.hidden, ic.fc_hidden) == (Hp, Hfp)
    assert (ic.layers, ic.max_nodes, ic.flags) == (cfg.layers, cfg.max_nodes, cfg.flags)
    # the public arena stays logical: init matches the oracle at the logical width
    lay, _ = hgnn.hg_param_layout(cfg)
    flat = hgnn.hg_params_init_host(cfg, 3)
    ref = O.init_params({"f_node": 34, "f_edge": 4, "hidden": H, "layers": 2, "fc_hidden": Hf}, 3)
    for name, off, r, c in lay:
        np.testing.assert_array_equal(flat[off:off + r * c], ref[name].reshape(-1).astype(np.float32), err_msg=name)


@pytest.mark.parametrize("H", [0, -3, 1025])
def test_config_hidden_range(H):
    cfg = hgnn.make_config(34, 4, H, 2, 4, 100, 400, 1.0, fc_hidden=32)
    with pytest.raises(hgnn.HgError) as e:
        hgnn.hg_config_internal(cfg)
    assert e.value.name == "HG_E_INVALID"


@pytest.mark.parametrize("F0,H,L,Hf", [(34, 32, 2, 32), (9, 128, 6, 128), (1, 32, 1, 8)])
def test_param_init_bit_exact_vs_oracle(F0, H, L, Hf):
    cfg = hgnn.make_config(F0, 4, H, L, 4, 100, 400, 1.0, fc_hidden=Hf)
    lay, total = hgnn.hg_param_layout(cfg)
    flat = hgnn.hg_params_init_host(cfg, 12345)
    ref = O.init_params({"f_node": F0, "f_edge": 4, "hidden": H, "layers": L, "fc_hidden": Hf}, 12345)
    assert [n for n, *_ in lay] == list(ref)
    for name, off, r, c in lay:
        a = flat[off:off + r * c]
        b = ref[name].reshape(-1).astype(np.float32)
        np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32), err_msg=name)
        assert off % 64 == 0
    # padding is zero
    used = np.zeros(total, bool)
    for name, off, r, c in lay:
        used[off:off + r * c] = True
    assert np.all(flat[~used] == 0)


def test_batch_offsets_alignment():
    o = hgnn.hg_batch_offsets(3, 17, 33, 34, 4)
    for k in ("graph_ptr", "y", "rowptr", "col", "x", "eattr", "slot"):
        assert o[k] % 16 == 0
    assert o["total"] >= o["slot"] + 33


def test_unknown_flags_rejected():
    cfg = hgnn.make_config(34, 4, 128, 2, 4, 100, 400, 1.0, flags=1 << 20)
    with pytest.raises(hgnn.HgError) as e:
        hgnn.hg_config_internal(cfg)
    assert e.value.name == "HG_E_INVALID"


@pytest.mark.parametrize("L,H", [(1, 128), (2, 32), (6, 128), (8, 512), (7, 55)])
def test_bucket_layout_partitions_the_arena(L, H):
    """The NCCL gradient buckets (hg_bucket_layout) are contiguous, in backward order (head and
    the last layers first, conv0 last), and cover the internal arena exactly once, so the
    bucketed average touches every gradient once."""
    cfg = hgnn.make_config(34, 4, H, L, 4, 100, 400, 1.0)
    icfg = hgnn.hg_config_internal(cfg)
    lay, total = hgnn.hg_param_layout(icfg)
    b = hgnn.bucket_layout(cfg)
    assert b[-1][0] == 0 and b[0][1] == total
    for (b0, e0), (b1, e1) in zip(b, b[1:]):
        assert e1 == b0 and b1 < e1 and b0 < e0  # descending, adjacent, non-empty
    covered = np.zeros(total, np.int32)
    for beg, end in b:
        covered[beg:end] += 1
    assert np.all(covered == 1)
    off = {name: o for name, o, r, c in lay}
    assert b[-1] == (0, off["conv1.M_x"] if L > 1 else total)  # conv0 alone in the last bucket
    assert b[0][0] <= off["head.W1"]


def test_pack_rejects_more_distinct_degrees_than_class_slots():
    graphs = []
    for d in range(1, 40):  # stars of every degree 1..39
        graphs.append((np.ones((d + 1, 2), np.float32), [(0, i, [1, 0, 0, 0]) for i in range(1, d + 1)], 1.0))
    data = make_store(graphs, f_edge=4)
    store = hgnn.Store(data)
    cfg = hgnn.make_config(2, 4, 128, 1, 40, 1000, 2000, 1.0, max_degree=127)
    with pytest.raises(hgnn.HgError) as e:
        hgnn.hg_pack_host(store, list(range(39)), cfg)
    assert e.value.name == "HG_E_DEGREE"
    hgnn.hg_pack_host(store, list(range(30)), cfg)  # degrees 1..30: 30 distinct <= 32 slots
    cfg5 = hgnn.make_config(2, 4, 128, 1, 40, 1000, 2000, 1.0, max_degree=4)  # 5 slots
    with pytest.raises(hgnn.HgError) as e:
        hgnn.hg_pack_host(store, [4], cfg5)  # degree 5 > max_degree 4
    assert e.value.name == "HG_E_CAPACITY"


def test_pack_threads_setting_does_not_change_the_bytes(pcqm):
    store = hgnn.Store(pcqm)
    cfg = _cfg_for(pcqm, 64)
    ids = np.arange(64) * 7
    ref = hgnn.hg_pack_host(store, ids, cfg)
    for t in (1, 3, 8):
        hgnn.pack_threads_set(t)
        np.testing.assert_array_equal(hgnn.hg_pack_host(store, ids, cfg), ref)
    hgnn.pack_threads_set(4)
    with pytest.raises(hgnn.HgError):
        hgnn.pack_threads_set(0)


@pytest.mark.parametrize("flags,scalers", [(2, 0), (0, 31), (2, 1 | 8), (2, 31)])
def test_variant_param_layout_and_init_match_the_oracle(flags, scalers):
    """Model variants (self-term: M_s after M_x, U_x after U; scaler sets: U = [H, 4SH]): the
    C-ABI layout and the counter-based init equal the oracle's param_specs / init_params."""
    cfg = hgnn.make_config(34, 4, 128, 2, 4, 100, 400, 1.0, flags=flags, scalers=scalers, delta_lin=2.0)
    lay, total = hgnn.hg_param_layout(cfg)
    flat = hgnn.hg_params_init_host(cfg, 77)
    ocfg = {"f_node": 34, "f_edge": 4, "hidden": 128, "layers": 2, "fc_hidden": 128,
            "self_term": bool(flags & 2), "scalers": hgnn.scaler_names(scalers), "delta_lin": 2.0}
    ref = O.init_params(ocfg, 77)
    assert [n for n, *_ in lay] == list(ref)
    for name, off, r, c in lay:
        np.testing.assert_array_equal(flat[off:off + r * c], ref[name].reshape(-1).astype(np.float32), err_msg=name)


def test_variant_config_validation():
    for kw in ({"scalers": 2}, {"scalers": 8 | 1, "delta_lin": 0.0}, {"scalers": 64}):
        cfg = hgnn.make_config(34, 4, 128, 2, 4, 100, 400, 1.0, **kw)
        with pytest.raises(hgnn.HgError) as e:
            hgnn.hg_config_internal(cfg)
        assert e.value.name == "HG_E_INVALID"
    cfg = hgnn.make_config(200, 4, 128, 2, 4, 100, 400, 1.0, flags=hgnn.HG_FLAG_SELF_TERM)  # f_node > hidden
    with pytest.raises(hgnn.HgError):
        hgnn.hg_config_internal(cfg)


def test_degree_stat_linear_matches_oracle(pcqm):
    store = hgnn.Store(pcqm)
    assert abs(store.degree_stat_linear() - O.degree_stat_linear(pcqm)) <= 1e-14
    ids = np.arange(5, 3000, 11)
    assert abs(store.degree_stat_linear(ids) - O.degree_stat_linear(pcqm, ids)) <= 1e-14
