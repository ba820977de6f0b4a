"""Checkpoint / resume (versioned little-endian binary of config + named parameter
tensors + optimizer state with a CRC; include/hgnn.h hg_checkpoint_save / hg_checkpoint_load):
a resumed run continues bitwise like the uninterrupted one; corrupt, truncated and
mismatched files are rejected without touching the ctx."""
import struct

import numpy as np
import pytest

import oracle as O
from paper_2207_11333_b200 import hgnn
from tests import _parity as PT

pytestmark = pytest.mark.gpu


def _steps(ctx, store, ids, B, k0, k1):
    for k in range(k0, k1):
        ctx.pack(store, ids[k * B:(k + 1) * B], k % 2)
        ctx.train_step(k % 2, graph=False)


def test_checkpoint_resume_is_bitwise(torch_cuda, tmp_path):
    data = PT.generate("pcqm", 600, 17)
    B = 32
    a, cfg, _ = PT.make_ctx(data, B, 128, 3, seed=4)
    ids = O.shard(9, 0, 0, 1, len(data["y"]))
    _steps(a, a._store, ids, B, 0, 3)
    path = str(tmp_path / "run.ckpt")
    a.checkpoint_save(path)
    raw = open(path, "rb").read()
    assert raw[:8] == b"HGNNCKPT" and struct.unpack("<I", raw[8:12])[0] == 1
    # a fresh ctx (different init) resumes from the file
    b, _, _ = PT.make_ctx(data, B, 128, 3, seed=99)
    b.checkpoint_load(path)
    pa, pb = a.params_get(), b.params_get()
    np.testing.assert_array_equal(pa.view(np.uint32), pb.view(np.uint32))
    ma, va, sa = a.opt_state_get()
    mb, vb, sb = b.opt_state_get()
    assert sa == sb == 3
    np.testing.assert_array_equal(ma.view(np.uint32), mb.view(np.uint32))
    np.testing.assert_array_equal(va.view(np.uint32), vb.view(np.uint32))
    # both continue identically
    _steps(a, a._store, ids, B, 3, 5)
    _steps(b, b._store, ids, B, 3, 5)
    np.testing.assert_array_equal(a.params_get().view(np.uint32), b.params_get().view(np.uint32))


def test_checkpoint_rejects_bad_files(torch_cuda, tmp_path):
    data = PT.generate("pcqm", 300, 18)
    a, cfg, _ = PT.make_ctx(data, 16, 128, 2, seed=4)
    path = str(tmp_path / "a.ckpt")
    a.checkpoint_save(path)
    before = a.params_get()
    raw = bytearray(open(path, "rb").read())
    # corrupt one parameter byte: CRC mismatch
    bad = bytearray(raw)
    bad[len(bad) // 2] ^= 0x40
    p_bad = str(tmp_path / "bad.ckpt")
    open(p_bad, "wb").write(bytes(bad))
    with pytest.raises(hgnn.HgError) as e:
        a.checkpoint_load(p_bad)
    assert e.value.code == 12  # HG_E_IO
    # truncated
    open(p_bad, "wb").write(bytes(raw[:-100]))
    with pytest.raises(hgnn.HgError):
        a.checkpoint_load(p_bad)
    # missing
    with pytest.raises(hgnn.HgError):
        a.checkpoint_load(str(tmp_path / "missing.ckpt"))
    np.testing.assert_array_equal(before.view(np.uint32), a.params_get().view(np.uint32))
    # another model (3 layers): HG_E_SHAPE
    c, _, _ = PT.make_ctx(data, 16, 128, 3, seed=4)
    with pytest.raises(hgnn.HgError) as e:
        c.checkpoint_load(path)
    assert e.value.code == 2  # HG_E_SHAPE
