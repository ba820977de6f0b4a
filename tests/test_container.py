"""On-disk packed container with subfiles and the object-per-graph backend
(PAPER.md:183-192, 232-253, 341-347). CPU only."""
import os

import numpy as np
import pytest

import molgen
from paper_2207_11333_b200 import hgnn


def _cfg(data, store, B):
    st = store.stats()
    return hgnn.make_config(data["f_node"], 4, 32, 2, B, B * st["max_nodes_per_graph"],
                            B * int(np.diff(np.asarray(data["edge_offset"])).max()), 1.0)


@pytest.mark.parametrize("n_sub", [1, 3, 7])
def test_container_roundtrip_is_bit_exact(tmp_path, n_sub):
    data = molgen.generate("pcqm", 500, 21)
    src = hgnn.Store(data)
    path = str(tmp_path / "c.hgpk")
    src.write_container(path, n_sub, threads=4)
    info = hgnn.container_info(path)
    assert info["graphs"] == 500 and info["subfiles"] == n_sub
    assert info["nodes"] == int(data["node_offset"][-1]) and info["edges"] == int(data["edge_offset"][-1])
    assert info["avg_nodes_per_graph"] == info["nodes"] / 500
    back = hgnn.Store.from_container(path, threads=3)
    assert back.stats() == src.stats()
    cfg = _cfg(data, src, 32)
    rng = np.random.default_rng(0)
    for _ in range(5):  # random reads in any order return the same graphs (packed bit-identically)
        ids = rng.choice(500, 32, replace=False)
        np.testing.assert_array_equal(hgnn.hg_pack_host(back, ids, cfg), hgnn.hg_pack_host(src, ids, cfg))


def test_objfiles_roundtrip_matches_container(tmp_path):
    data = molgen.generate("tiny", 300, 5)
    src = hgnn.Store(data)
    src.write_objfiles(str(tmp_path / "obj"), threads=4)
    assert len(os.listdir(tmp_path / "obj")) == 300  # one file per graph
    back = hgnn.Store.from_objfiles(str(tmp_path / "obj"), 300, threads=2)
    assert back.stats() == src.stats()
    cfg = _cfg(data, src, 64)
    ids = np.arange(64) * 4
    np.testing.assert_array_equal(hgnn.hg_pack_host(back, ids, cfg), hgnn.hg_pack_host(src, ids, cfg))


def test_container_detects_corruption_and_missing_subfiles(tmp_path):
    data = molgen.generate("tiny", 200, 9)
    src = hgnn.Store(data)
    path = tmp_path / "c"
    src.write_container(str(path), 4)
    # flip one byte inside subfile 2's data
    p2 = path / "data.2"
    raw = bytearray(p2.read_bytes())
    raw[len(raw) // 2] ^= 0x40
    p2.write_bytes(bytes(raw))
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store.from_container(str(path))
    assert e.value.name == "HG_E_IO"
    # truncated trailing subfile
    src.write_container(str(path), 4)
    p3 = path / "data.3"
    p3.write_bytes(p3.read_bytes()[:-7])
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store.from_container(str(path))
    assert e.value.name == "HG_E_IO"
    # missing subfile, corrupt index
    src.write_container(str(path), 4)
    os.remove(path / "data.1")
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store.from_container(str(path))
    assert e.value.name == "HG_E_IO"
    src.write_container(str(path), 4)
    meta = path / "meta.idx"
    raw = bytearray(meta.read_bytes())
    raw[60] ^= 1
    meta.write_bytes(bytes(raw))
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store.from_container(str(path))
    assert e.value.name == "HG_E_IO"
    with pytest.raises(hgnn.HgError) as e:
        hgnn.Store.from_container(str(tmp_path / "nowhere"))
    assert e.value.name == "HG_E_IO"


def test_container_is_smaller_than_object_store(tmp_path):
    """SPEC.md gpack property / PAPER Table 2 analogue (22 GB vs 34 GB): the packed
    container occupies fewer filesystem blocks than one file per graph."""
    data = molgen.generate("tiny", 2000, 3)
    src = hgnn.Store(data)
    src.write_container(str(tmp_path / "c"), 2)
    src.write_objfiles(str(tmp_path / "o"))

    def blocks(d):
        return sum(os.stat(os.path.join(d, f)).st_blocks for f in os.listdir(d))
    assert blocks(tmp_path / "c") < blocks(tmp_path / "o")


def _crc32c(data: bytes, crc: int = 0) -> int:
    """CRC-32C (Castagnoli, reflected 0x82F63B78, initial and final inversion), the checksum
    csrc/container.cpp computes with the SSE4.2 crc32 instruction."""
    tbl = []
    for i in range(256):
        c = i
        for _ in range(8):
            c = (c >> 1) ^ (0x82F63B78 if c & 1 else 0)
        tbl.append(c)
    crc ^= 0xFFFFFFFF
    for b in data:
        crc = (crc >> 8) ^ tbl[(crc ^ b) & 0xFF]
    return crc ^ 0xFFFFFFFF


def test_checksum_consistent_but_malformed_index_is_rejected(tmp_path):
    """A meta.idx whose CRC is right but whose subfile table or offsets are out of order must be
    rejected before any of its values is used as a read destination (container.cpp)."""
    data = molgen.generate("tiny", 60, 5)
    src = hgnn.Store(data)
    path = str(tmp_path / "c.hgpk")
    src.write_container(path, 3)
    raw = bytearray(open(os.path.join(path, "meta.idx"), "rb").read())
    hdr = 48  # MetaHead: magic, version, G, N, E, F0, Fe, n_sub, reserved
    assert _crc32c(bytes(raw[:-4])) == int.from_bytes(raw[-4:], "little")  # our CRC matches the writer's
    G = int.from_bytes(raw[8:16], "little")
    sub_off = hdr + 16 * (G + 1)

    def corrupt(off, value):
        bad = bytearray(raw)
        bad[off:off + 8] = int(value).to_bytes(8, "little", signed=True)
        bad[-4:] = _crc32c(bytes(bad[:-4])).to_bytes(4, "little")
        open(os.path.join(path, "meta.idx"), "wb").write(bad)
        with pytest.raises(hgnn.HgError) as e:
            hgnn.Store.from_container(path)
        assert e.value.name == "HG_E_IO"

    corrupt(sub_off + 8, 10 ** 12)      # sub[1] far past G
    corrupt(sub_off + 8, -5)            # sub[1] negative
    corrupt(hdr + 8 * 5, 10 ** 9)       # node_offset[5] past N
    corrupt(hdr + 8 * (G + 1) + 8 * 7, -1)  # edge_offset[7] negative
    corrupt(8, 10 ** 15)                # G absurd: sizes checked before any allocation
    open(os.path.join(path, "meta.idx"), "wb").write(raw)
    assert hgnn.Store.from_container(path).stats() == src.stats()
