"""One shared copy of the Table-1 store for every rank of a node (SURVEY §8(e), §8(b)
hg_store_open_shared). CPU only: created in this process, attached from another
process; both collate bit-identical batches (pinning needs a GPU: pin=False here)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import molgen
from paper_2207_11333_b200 import hgnn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cfg(data, B):
    nn = np.diff(data["node_offset"])
    ne = np.diff(data["edge_offset"])
    return hgnn.make_config(data["f_node"], 4, 128, 2, B, int(nn.max() * B), int(ne.max() * B), 1.0)


def test_shared_store_roundtrip_across_processes(tmp_path):
    data = molgen.generate("pcqm", 400, 17)
    data["y_node"] = np.arange(len(data["x"]), dtype=np.float32)
    name = f"/hgnn_test_{os.getpid()}"
    try:
        shared = hgnn.Store(data, shared_name=name)
        private = hgnn.Store(data)
        assert shared.stats() == private.stats()
        cfg = _cfg(data, 32)
        ids = np.arange(0, 400, 13)[:32]
        ref = hgnn.hg_pack_host(private, ids, cfg)
        np.testing.assert_array_equal(hgnn.hg_pack_host(shared, ids, cfg), ref)
        np.save(tmp_path / "ids.npy", ids)
        np.save(tmp_path / "ref.npy", ref)
        code = (f"import sys, numpy as np; sys.path.insert(0, {ROOT!r}); from paper_2207_11333_b200 import hgnn;"
                f"s = hgnn.Store.open_shared({name!r}); cfg = hgnn.make_config({data['f_node']}, 4, 128, 2, 32, "
                f"{cfg.max_nodes}, {cfg.max_edges}, 1.0); ids = np.load({str(tmp_path / 'ids.npy')!r});"
                f"b = hgnn.hg_pack_host(s, ids, cfg); ref = np.load({str(tmp_path / 'ref.npy')!r});"
                f"assert np.array_equal(b, ref); print('ok', s.stats()['graphs'])")
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0 and "ok 400" in r.stdout, r.stdout + r.stderr
        blob = hgnn.unpack_blob(ref)  # the node-level targets travel with the batch
        np.testing.assert_array_equal(blob["y_node"][:5], data["y_node"][data["node_offset"][ids[0]]:][:5])
    finally:
        hgnn.Store.unlink_shared(name)


def test_shared_store_errors():
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store.open_shared("/hgnn_no_such_store_xyz")
    assert e.value.name == "HG_E_IO"
    data = molgen.generate("tiny", 20, 1)
    name = f"/hgnn_test_dup_{os.getpid()}"
    try:
        hgnn.Store(data, shared_name=name)
        with pytest.raises(hgnn.HgError) as e:  # the name exists
            hgnn.Store(data, shared_name=name)
        assert e.value.name == "HG_E_IO"
    finally:
        hgnn.Store.unlink_shared(name)
