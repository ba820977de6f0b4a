"""molgen — seeded synthetic molecular graphs in the Table-1 layout.

INPUT GENERATOR ONLY (shared by ``oracle/`` and the CUDA product path; holds
none of the method's arithmetic). The C source ``molgen.c`` documents the
recipe; DESIGN.md "Input recipe" states it with the calibration targets of
PAPER.md:305-306 (Table 2: 29.4 / 52.4 nodes per graph, 2.028 / 1.998 directed
edges per node).

``generate(preset, n_graphs, seed)`` returns a dict with the Table-1 global
arrays:
    node_offset int64 [G+1], edge_offset int64 [G+1],
    x float32 [N, F0], edge_index int32 [2, E] (graph-local, per graph sorted
    by (src, dst)), edge_attr float32 [E, 4], y float32 [G]
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

PRESETS = {"tiny": 0, "pcqm": 1, "aisd": 2}

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "molgen.c")
_LIB = os.path.join(_HERE, "libmolgen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile libmolgen.so in-tree with gcc (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-pthread", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i32p = ctypes.POINTER(ctypes.c_int32)
        i64p = ctypes.POINTER(ctypes.c_int64)
        f32p = ctypes.POINTER(ctypes.c_float)
        lib.molgen_preset_info.argtypes = [ctypes.c_int, i32p, i32p, i32p, i32p, i32p]
        lib.molgen_count.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                     i32p, i32p, ctypes.c_int]
        lib.molgen_fill.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                    i64p, i64p, ctypes.c_int64, f32p, i32p, f32p, f32p, ctypes.c_int]
        _lib = lib
    return _lib


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def preset_info(preset: str) -> dict:
    lib = _load()
    nv, fn, fe, mx = (ctypes.c_int32() for _ in range(4))
    z = np.zeros(64, np.int32)
    rc = lib.molgen_preset_info(PRESETS[preset], ctypes.byref(nv), ctypes.byref(fn), ctypes.byref(fe),
                                ctypes.byref(mx), _ptr(z, ctypes.c_int32))
    if rc:
        raise ValueError(preset)
    return {"n_vocab": nv.value, "f_node": fn.value, "f_edge": fe.value, "max_nodes": mx.value,
            "vocab_z": z[: nv.value].copy()}


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def generate(preset: str, n_graphs: int, seed: int, first_id: int = 0, threads: int | None = None) -> dict:
    lib = _load()
    threads = threads or default_threads()
    info = preset_info(preset)
    n = int(n_graphs)
    nodes = np.zeros(n, np.int32)
    edges = np.zeros(n, np.int32)
    rc = lib.molgen_count(PRESETS[preset], seed, first_id, n, _ptr(nodes, ctypes.c_int32),
                          _ptr(edges, ctypes.c_int32), threads)
    if rc:
        raise RuntimeError(f"molgen_count failed: {rc}")
    node_offset = np.zeros(n + 1, np.int64)
    edge_offset = np.zeros(n + 1, np.int64)
    np.cumsum(nodes, out=node_offset[1:])
    np.cumsum(edges, out=edge_offset[1:])
    N, E, F = int(node_offset[-1]), int(edge_offset[-1]), info["f_node"]
    x = np.empty((N, F), np.float32)
    ei = np.empty((2, E), np.int32)
    ea = np.empty((E, 4), np.float32)
    y = np.empty(n, np.float32)
    rc = lib.molgen_fill(PRESETS[preset], seed, first_id, n, _ptr(node_offset, ctypes.c_int64),
                         _ptr(edge_offset, ctypes.c_int64), E, _ptr(x, ctypes.c_float),
                         _ptr(ei, ctypes.c_int32), _ptr(ea, ctypes.c_float), _ptr(y, ctypes.c_float), threads)
    if rc:
        raise RuntimeError(f"molgen_fill failed: {rc}")
    return {"node_offset": node_offset, "edge_offset": edge_offset, "x": x, "edge_index": ei,
            "edge_attr": ea, "y": y, "f_node": F, "f_edge": 4, "vocab_z": info["vocab_z"],
            "preset": preset, "seed": seed}


def perturb_features(data: dict, seed: int, scale: float = 0.05) -> dict:
    """Return a copy whose x/edge_attr carry small seeded continuous jitter.

    Used only by finite-difference pins: exact one-hot
    inputs create automorphic ties (identical messages), and FD across a
    max/min/ReLU kink is undefined; jitter moves every kink away from h.
    """
    rng = np.random.default_rng(seed)
    out = dict(data)
    out["x"] = (data["x"] + scale * rng.standard_normal(data["x"].shape)).astype(np.float32)
    ea = data["edge_attr"].copy()
    # keep edge attributes symmetric: jitter per undirected bond
    src, dst = data["edge_index"]
    eo = data["edge_offset"]
    g_of_e = np.repeat(np.arange(len(eo) - 1), np.diff(eo))
    key = np.minimum(src, dst).astype(np.int64) * 1000 + np.maximum(src, dst) + g_of_e.astype(np.int64) * 1000003
    uniq, inv = np.unique(key, return_inverse=True)
    jit = scale * rng.standard_normal((len(uniq), ea.shape[1]))
    out["edge_attr"] = (ea + jit[inv]).astype(np.float32)
    return out


_ARRAYS = ("node_offset", "edge_offset", "x", "edge_index", "edge_attr", "y")


def generate_to(dirpath: str, preset: str, n_graphs: int, seed: int, threads: int | None = None) -> dict:
    """Generate straight into .npy files under ``dirpath`` (memory-mapped), so
    several processes on one host can share one copy of a multi-GB store via
    the page cache (``load_dir``). Idempotent: a complete directory is reused."""
    import json
    lib = _load()
    threads = threads or default_threads()
    meta_path = os.path.join(dirpath, "meta.json")
    if os.path.exists(meta_path):
        return load_dir(dirpath)
    os.makedirs(dirpath, exist_ok=True)
    info = preset_info(preset)
    n = int(n_graphs)
    nodes = np.zeros(n, np.int32)
    edges = np.zeros(n, np.int32)
    rc = lib.molgen_count(PRESETS[preset], seed, 0, n, _ptr(nodes, ctypes.c_int32), _ptr(edges, ctypes.c_int32),
                          threads)
    if rc:
        raise RuntimeError(f"molgen_count failed: {rc}")
    mm = np.lib.format.open_memmap
    no = mm(os.path.join(dirpath, "node_offset.npy"), "w+", np.int64, (n + 1,))
    eo = mm(os.path.join(dirpath, "edge_offset.npy"), "w+", np.int64, (n + 1,))
    no[0] = 0
    eo[0] = 0
    np.cumsum(nodes, out=no[1:])
    np.cumsum(edges, out=eo[1:])
    N, E, F = int(no[-1]), int(eo[-1]), info["f_node"]
    x = mm(os.path.join(dirpath, "x.npy"), "w+", np.float32, (N, F))
    ei = mm(os.path.join(dirpath, "edge_index.npy"), "w+", np.int32, (2, E))
    ea = mm(os.path.join(dirpath, "edge_attr.npy"), "w+", np.float32, (E, 4))
    y = mm(os.path.join(dirpath, "y.npy"), "w+", np.float32, (n,))
    rc = lib.molgen_fill(PRESETS[preset], seed, 0, n, _ptr(no, ctypes.c_int64), _ptr(eo, ctypes.c_int64), E,
                         _ptr(x, ctypes.c_float), _ptr(ei, ctypes.c_int32), _ptr(ea, ctypes.c_float),
                         _ptr(y, ctypes.c_float), threads)
    if rc:
        raise RuntimeError(f"molgen_fill failed: {rc}")
    for a in (no, eo, x, ei, ea, y):
        a.flush()
    with open(meta_path, "w") as f:
        json.dump({"preset": preset, "n_graphs": n, "seed": seed, "f_node": F, "vocab_z": info["vocab_z"].tolist()}, f)
    return load_dir(dirpath)


def load_dir(dirpath: str) -> dict:
    import json
    with open(os.path.join(dirpath, "meta.json")) as f:
        meta = json.load(f)
    d = {k: np.load(os.path.join(dirpath, k + ".npy"), mmap_mode="r") for k in _ARRAYS}
    d.update({"f_node": meta["f_node"], "f_edge": 4, "vocab_z": np.asarray(meta["vocab_z"]), "preset": meta["preset"],
              "seed": meta["seed"]})
    return d
