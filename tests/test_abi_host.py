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
    assert lib.hg_abi_version() == 1


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


@pytest.mark.parametrize("H,Hf,flags,Hp,Hfp", [
    (55, 55, 0, 128, 128),     # paper width -> tensor-core tile
    (200, 200, 0, 256, 256),   # paper width
    (55, 55, 1, 64, 64),       # SIMT path pads to the warp width
    (55, 40, 0, 128, 40),      # fc_hidden != hidden is left as given
    (128, 128, 0, 128, 128),   # multiples of 32 are not padded
    (96, 96, 0, 96, 96),
])
def test_config_internal_padding(H, Hf, flags, Hp, Hfp):
    cfg = hgnn.make_config(34, 4, H, 2, 4, 100, 400, 1.0, fc_hidden=Hf, flags=flags)
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
