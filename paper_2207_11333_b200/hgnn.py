"""Thin ctypes binding of libhgnn (include/hgnn.h). Argument marshalling only:
every step of the training path runs inside the library's CUDA kernels.

PyTorch is used only for device memory (the workspace is a uint8 CUDA tensor),
the caller's CUDA stream and process groups (to ship the NCCL unique id).
If the shared library is missing or fails to load this module raises; there
is no CPU fallback.

Function names mirror the C-ABI (hg_pack, hg_forward, hg_backward,
hg_allreduce_grads, hg_step, ...); ``Store`` and ``Context`` hold the opaque
handles and keep the borrowed arrays / workspace alive.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))

HG_OK = 0
STATUS = {0: "HG_OK", 1: "HG_E_INVALID", 2: "HG_E_SHAPE", 3: "HG_E_RANGE", 4: "HG_E_EMPTY", 5: "HG_E_ASYMMETRIC",
          6: "HG_E_DEGREE", 7: "HG_E_CAPACITY", 8: "HG_E_CUDA", 9: "HG_E_NCCL", 10: "HG_E_STATE", 11: "HG_E_UNSORTED",
          12: "HG_E_IO"}
HG_MAX_DEGREE = 127

PHASES = ["scalers", "proj", "agg_fwd", "update", "head_fwd", "head_bwd", "dA", "dU", "agg_bwd", "dMx", "dX",
          "allreduce", "adamw"]

P2P_HANDLE_BYTES = 72  # include/hgnn.h HG_P2P_HANDLE_BYTES
VIEW_P, VIEW_A, VIEW_ARG, VIEW_X, VIEW_SLOT, VIEW_YHAT, VIEW_LOSS, VIEW_HPRE, VIEW_PARAMS, VIEW_GRADS, \
    VIEW_AMP, VIEW_ATT, VIEW_NODE_YHAT, VIEW_NODE_HPRE = range(14)


class HgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class hg_store_desc(ctypes.Structure):
    _fields_ = [("num_graphs", ctypes.c_int64), ("num_nodes", ctypes.c_int64), ("num_edges", ctypes.c_int64),
                ("f_node", ctypes.c_int32), ("f_edge", ctypes.c_int32),
                ("node_offset", ctypes.c_void_p), ("edge_offset", ctypes.c_void_p), ("x", ctypes.c_void_p),
                ("edge_index", ctypes.c_void_p), ("edge_attr", ctypes.c_void_p), ("y", ctypes.c_void_p),
                ("y_node", ctypes.c_void_p)]


class hg_config(ctypes.Structure):
    _fields_ = [("f_node", ctypes.c_int32), ("f_edge", ctypes.c_int32), ("hidden", ctypes.c_int32),
                ("layers", ctypes.c_int32), ("fc_hidden", ctypes.c_int32), ("max_graphs", ctypes.c_int32),
                ("max_nodes", ctypes.c_int32), ("max_edges", ctypes.c_int32), ("n_slots", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("delta", ctypes.c_double), ("var_floor", ctypes.c_float),
                ("max_degree", ctypes.c_int32), ("scalers", ctypes.c_int32), ("delta_lin", ctypes.c_double),
                ("node_weight", ctypes.c_float)]


class hg_adamw(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float)]


class hg_batch_offsets_t(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in ("graph_ptr", "y", "y_node", "rowptr", "col", "x", "eattr", "slot",
                                              "total")]


_P = ctypes.c_void_p
_I32, _I64, _U64, _SZ, _D = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_double
_I32P, _I64P, _SZP, _DP = (ctypes.POINTER(t) for t in (_I32, _I64, _SZ, _D))
_CP = ctypes.POINTER(ctypes.c_char_p)

# C signature table: name -> argtypes (restype is hg_status == int32 except where noted)
SIGNATURES = {
    "hg_last_error": [],
    "hg_abi_version": [],
    "hg_store_create": [ctypes.POINTER(hg_store_desc), _I32, _I32, ctypes.POINTER(_P)],
    "hg_store_destroy": [_P],
    "hg_store_create_shared": [ctypes.POINTER(hg_store_desc), ctypes.c_char_p, _I32, _I32, ctypes.POINTER(_P)],
    "hg_store_open_shared": [ctypes.c_char_p, _I32, ctypes.POINTER(_P)],
    "hg_store_unlink_shared": [ctypes.c_char_p],
    "hg_store_stats": [_P, _I64P, _I64P, _I64P, _I32P, _I32P],
    "hg_degree_stat": [_P, _P, _I64, _DP],
    "hg_degree_stat_linear": [_P, _P, _I64, _DP],
    "hg_shard": [_U64, _I64, _I32, _I32, _I64, _P, _I64P],
    "hg_batch_offsets_get": [_I32, _I32, _I32, _I32, _I32, ctypes.POINTER(hg_batch_offsets_t)],
    "hg_pack_host": [_P, _P, _I32, ctypes.POINTER(hg_config), _P, _SZ, _SZP],
    "hg_config_internal": [ctypes.POINTER(hg_config), ctypes.POINTER(hg_config)],
    "hg_param_layout": [ctypes.POINTER(hg_config), _I32P, _I64P],
    "hg_param_layout_info": [ctypes.POINTER(hg_config), _I32, _CP, _I64P, _I32P, _I32P],
    "hg_params_init_host": [ctypes.POINTER(hg_config), _U64, _P],
    "hg_workspace_bytes": [ctypes.POINTER(hg_config), _SZP],
    "hg_ctx_create": [ctypes.POINTER(hg_config), _I32, _P, _SZ, _P, ctypes.POINTER(_P)],
    "hg_ctx_destroy": [_P],
    "hg_param_count": [_P, _I32P, _I64P],
    "hg_param_info": [_P, _I32, _CP, _I64P, _I32P, _I32P],
    "hg_params_init": [_P, _U64],
    "hg_params_set": [_P, _P, _I32],
    "hg_params_get": [_P, _P, _I32],
    "hg_grads_get": [_P, _P, _I32],
    "hg_opt_state_get": [_P, _P, _P, _I64P, _I32],
    "hg_opt_state_set": [_P, _P, _P, _I64, _I32],
    "hg_checkpoint_save": [_P, ctypes.c_char_p],
    "hg_checkpoint_load": [_P, ctypes.c_char_p],
    "hg_workspace_view": [_P, _I32, _I32, _I64P, _I64P],
    "hg_batch_get": [_P, _I32, _P, _SZ, _SZP],
    "hg_pack": [_P, _P, _P, _I32, _I32],
    "hg_upload_packed": [_P, _P, _SZ, _I32],
    "hg_forward": [_P, _I32],
    "hg_backward": [_P, _I32],
    "hg_nccl_unique_id": [_P],
    "hg_comm_init": [_P, _P, _I32, _I32],
    "hg_allreduce_grads": [_P],
    "hg_p2p_handle": [_P, _P],
    "hg_p2p_open": [_P, _P],
    "hg_step": [_P, ctypes.POINTER(hg_adamw)],
    "hg_train_step": [_P, _I32, ctypes.POINTER(hg_adamw), _I32],
    "hg_capture_step": [_P, _I32, ctypes.POINTER(hg_adamw)],
    "hg_profile_step": [_P, _I32, ctypes.POINTER(hg_adamw), _P, _P],
    "hg_loss_get": [_P, ctypes.POINTER(ctypes.c_float)],
    "hg_loss_enqueue": [_P, ctypes.c_int32],
    "hg_eval_reset": [_P],
    "hg_container_write": [_P, ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32],
    "hg_container_open": [ctypes.c_char_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)],
    "hg_container_info": [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                          ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32)],
    "hg_objfiles_write": [_P, ctypes.c_char_p, ctypes.c_int32],
    "hg_objfiles_open": [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)],
    "hg_eval_batch": [_P, ctypes.c_int32, ctypes.c_int32],
    "hg_eval_result": [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                       ctypes.POINTER(ctypes.c_int64)],
    "hg_eval_pairs": [_P, ctypes.c_int32, _P, _P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)],
    "hg_loss_fetch": [_P, ctypes.c_int32, ctypes.POINTER(ctypes.c_float)],
    "hg_sync": [_P],
    "hg_set_timeout": [_P, _D],
    "hg_p2p_emulate": [ctypes.POINTER(_P), _I32, ctypes.POINTER(hg_adamw)],
    "hg_bucket_layout": [ctypes.POINTER(hg_config), _I64P, _I32, _I32P],
    "hg_pack_threads_set": [_I32],
    "hg_exchange_time": [_P, ctypes.POINTER(hg_adamw), _I32, ctypes.POINTER(ctypes.c_float)],
    "hg_launch_count": [_P, _I64P],
}

_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libhgnn.so (building it in-tree with nvcc if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing and _build.needs_build():
        _build.build()
    if not os.path.exists(_build.LIB):
        raise RuntimeError(f"libhgnn.so not found at {_build.LIB}; the CUDA extension is required (no CPU fallback)")
    lib = ctypes.CDLL(_build.LIB, mode=ctypes.RTLD_GLOBAL)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _I32
    lib.hg_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _check(st: int):
    if st != HG_OK:
        raise HgError(st, _lib.hg_last_error().decode())


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


# --------------------------------------------------------------------------- config
DEFAULT_ADAMW = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)


HG_LOSS_RING = 4  # include/hgnn.h
HG_FLAG_TF32 = 1  # reduced-precision (single-pass TF32) GEMM mode
HG_FLAG_SELF_TERM = 2  # PNA self-term variant (x_i into M and U)
HG_FLAG_NODE_HEAD = 4  # node-level head beside the graph head (multitask)
SCALER_BITS = {"identity": 1, "amplification": 2, "attenuation": 4, "linear": 8, "inverse_linear": 16}


def scaler_mask(names) -> int:
    m = 0
    for n in names:
        m |= SCALER_BITS[n]
    return m


def scaler_names(mask: int) -> tuple:
    """The U block order of a scaler bit set (bit order), as the oracle's cfg['scalers']."""
    mask = mask or 7
    return tuple(n for n, b in SCALER_BITS.items() if mask & b)


def make_config(f_node, f_edge, hidden, layers, max_graphs, max_nodes, max_edges, delta, fc_hidden=None,
                n_slots=2, var_floor=1e-10, flags=0, max_degree=0, scalers=0, delta_lin=0.0,
                node_weight=1.0) -> hg_config:
    return hg_config(f_node=f_node, f_edge=f_edge, hidden=hidden, layers=layers, fc_hidden=fc_hidden or hidden,
                     max_graphs=max_graphs, max_nodes=max_nodes, max_edges=max_edges, n_slots=n_slots, flags=flags,
                     delta=float(delta), var_floor=var_floor, max_degree=max_degree, scalers=int(scalers),
                     delta_lin=float(delta_lin), node_weight=float(node_weight))


def make_adamw(**kw) -> hg_adamw:
    d = dict(DEFAULT_ADAMW)
    d.update(kw)
    return hg_adamw(**d)


# --------------------------------------------------------------------------- store
class Store:
    """Table-1 store. Borrows the numpy arrays (copy=0) and
    keeps them alive for the store's lifetime."""

    def __init__(self, data: dict, copy: bool = False, threads: int = 0, shared_name: str = None, pin: bool = False):
        """shared_name: create the POSIX shared-memory store of that name (hg_store_create_shared;
        other processes attach with Store.open_shared); the arrays are copied into it."""
        load()
        self._arrays = {
            "node_offset": np.ascontiguousarray(data["node_offset"], np.int64),
            "edge_offset": np.ascontiguousarray(data["edge_offset"], np.int64),
            "x": np.ascontiguousarray(data["x"], np.float32),
            "edge_index": np.ascontiguousarray(data["edge_index"], np.int32),
            "edge_attr": np.ascontiguousarray(data["edge_attr"], np.float32),
            "y": np.ascontiguousarray(data["y"], np.float32),
        }
        if "y_node" in data:
            self._arrays["y_node"] = np.ascontiguousarray(data["y_node"], np.float32)
        a = self._arrays
        G = len(a["node_offset"]) - 1
        self.f_node = int(a["x"].shape[1])
        self.f_edge = int(a["edge_attr"].shape[1]) if a["edge_attr"].ndim == 2 else int(data.get("f_edge", 4))
        d = hg_store_desc(num_graphs=G, num_nodes=int(a["node_offset"][-1]), num_edges=int(a["edge_offset"][-1]),
                          f_node=self.f_node, f_edge=self.f_edge, node_offset=a["node_offset"].ctypes.data,
                          edge_offset=a["edge_offset"].ctypes.data, x=a["x"].ctypes.data,
                          edge_index=a["edge_index"].ctypes.data, edge_attr=a["edge_attr"].ctypes.data,
                          y=a["y"].ctypes.data, y_node=a["y_node"].ctypes.data if "y_node" in a else None)
        h = ctypes.c_void_p()
        if shared_name:
            _check(_lib.hg_store_create_shared(ctypes.byref(d), shared_name.encode(), int(pin), int(threads),
                                               ctypes.byref(h)))
            self.handle = h
            self._arrays = None
            return
        _check(_lib.hg_store_create(ctypes.byref(d), int(copy), int(threads), ctypes.byref(h)))
        self.handle = h
        if copy:
            self._arrays = None

    @classmethod
    def _adopt(cls, handle):
        s = cls.__new__(cls)
        s.handle = handle
        s._arrays = None
        g, n, e, mn, md = _I64(), _I64(), _I64(), _I32(), _I32()
        _check(_lib.hg_store_stats(handle, ctypes.byref(g), ctypes.byref(n), ctypes.byref(e), ctypes.byref(mn),
                                   ctypes.byref(md)))
        return s

    @classmethod
    def open_shared(cls, name: str, pin: bool = False) -> "Store":
        """Attach to a store another process created with shared_name (hg_store_open_shared)."""
        load()
        h = ctypes.c_void_p()
        _check(_lib.hg_store_open_shared(name.encode(), int(pin), ctypes.byref(h)))
        return cls._adopt(h)

    @staticmethod
    def unlink_shared(name: str):
        load()
        _check(_lib.hg_store_unlink_shared(name.encode()))

    @classmethod
    def from_container(cls, path: str, threads: int = 0) -> "Store":
        """Open an on-disk packed container (hg_container_open); the store owns its memory."""
        load()
        h = ctypes.c_void_p()
        _check(_lib.hg_container_open(path.encode(), int(threads), ctypes.byref(h)))
        return cls._adopt(h)

    @classmethod
    def from_objfiles(cls, path: str, num_graphs: int, threads: int = 0) -> "Store":
        """Load the object-per-graph comparison backend (hg_objfiles_open)."""
        load()
        h = ctypes.c_void_p()
        _check(_lib.hg_objfiles_open(path.encode(), int(num_graphs), int(threads), ctypes.byref(h)))
        return cls._adopt(h)

    def write_container(self, path: str, n_subfiles: int, threads: int = 0):
        _check(_lib.hg_container_write(self.handle, path.encode(), int(n_subfiles), int(threads)))

    def write_objfiles(self, path: str, threads: int = 0):
        _check(_lib.hg_objfiles_write(self.handle, path.encode(), int(threads)))

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.hg_store_destroy(self.handle)
            self.handle = None

    def stats(self) -> dict:
        g, n, e = _I64(), _I64(), _I64()
        mn, md = _I32(), _I32()
        _check(_lib.hg_store_stats(self.handle, ctypes.byref(g), ctypes.byref(n), ctypes.byref(e), ctypes.byref(mn),
                                   ctypes.byref(md)))
        return {"graphs": g.value, "nodes": n.value, "edges": e.value, "max_nodes_per_graph": mn.value,
                "max_degree": md.value}

    def degree_stat_linear(self, ids=None) -> float:
        out = _D()
        if ids is None:
            _check(_lib.hg_degree_stat_linear(self.handle, None, 0, ctypes.byref(out)))
        else:
            ids = np.ascontiguousarray(ids, np.int64)
            _check(_lib.hg_degree_stat_linear(self.handle, _ptr(ids), len(ids), ctypes.byref(out)))
        return out.value

    def degree_stat(self, ids=None) -> float:
        out = _D()
        if ids is None:
            _check(_lib.hg_degree_stat(self.handle, None, 0, ctypes.byref(out)))
        else:
            ids = np.ascontiguousarray(ids, np.int64)
            _check(_lib.hg_degree_stat(self.handle, _ptr(ids), len(ids), ctypes.byref(out)))
        return out.value


def hg_store_create(data: dict, copy: bool = False, threads: int = 0) -> Store:
    return Store(data, copy, threads)


def hg_shard(seed: int, epoch: int, rank: int, world: int, n: int) -> np.ndarray:
    load()
    out = np.empty(max(1, n // max(1, world)), np.int64)
    cnt = _I64()
    _check(_lib.hg_shard(seed, epoch, rank, world, n, _ptr(out), ctypes.byref(cnt)))
    return out[:cnt.value].copy()


def hg_batch_offsets(B, N, E, f_node, f_edge) -> dict:
    load()
    o = hg_batch_offsets_t()
    _check(_lib.hg_batch_offsets_get(B, N, E, f_node, f_edge, ctypes.byref(o)))
    return {k: getattr(o, k) for k, _ in hg_batch_offsets_t._fields_}


def container_info(path: str) -> dict:
    """Counts from a container's index (hg_container_info), no data read."""
    load()
    g, n, e, k = _I64(), _I64(), _I64(), _I32()
    _check(_lib.hg_container_info(path.encode(), ctypes.byref(g), ctypes.byref(n), ctypes.byref(e), ctypes.byref(k)))
    return {"graphs": g.value, "nodes": n.value, "edges": e.value, "subfiles": k.value,
            "avg_nodes_per_graph": n.value / g.value}


def hg_pack_host(store: Store, ids, cfg: hg_config) -> np.ndarray:
    """Host collate into a packed blob (uint8 array) in the device slot layout."""
    load()
    ids = np.ascontiguousarray(ids, np.int64)
    cap = hg_batch_offsets(cfg.max_graphs, cfg.max_nodes, cfg.max_edges, cfg.f_node, cfg.f_edge)["total"]
    buf = np.zeros(cap, np.uint8)
    used = _SZ()
    _check(_lib.hg_pack_host(store.handle, _ptr(ids), len(ids), ctypes.byref(cfg), _ptr(buf), cap,
                             ctypes.byref(used)))
    return buf[:used.value].copy()


def unpack_blob(blob: np.ndarray) -> dict:
    """Split a packed blob into its arrays (views) using hg_batch_offsets."""
    h = blob[:64].view(np.int32)
    B, N, E, F0, Fe = (int(v) for v in h[:5])
    o = hg_batch_offsets(B, N, E, F0, Fe)
    def arr(key, dtype, count):
        return blob[o[key]:o[key] + count * np.dtype(dtype).itemsize].view(dtype)
    return {"B": B, "N": N, "E": E, "graph_ptr": arr("graph_ptr", np.int32, B + 1), "y": arr("y", np.float32, B),
            "y_node": arr("y_node", np.float32, N),
            "rowptr": arr("rowptr", np.int32, N + 1), "col": arr("col", np.int32, E),
            "x": arr("x", np.float32, N * F0).reshape(N, F0), "eattr": arr("eattr", np.float32, E * Fe).reshape(E, Fe),
            "slot": arr("slot", np.uint8, E)}


def hg_param_layout(cfg: hg_config):
    """[(name, offset, rows, cols)], total floats — the flat arena layout."""
    load()
    nt, ne = _I32(), _I64()
    _check(_lib.hg_param_layout(ctypes.byref(cfg), ctypes.byref(nt), ctypes.byref(ne)))
    out = []
    for i in range(nt.value):
        name = ctypes.c_char_p()
        off, r, c = _I64(), _I32(), _I32()
        _check(_lib.hg_param_layout_info(ctypes.byref(cfg), i, ctypes.byref(name), ctypes.byref(off), ctypes.byref(r),
                                         ctypes.byref(c)))
        out.append((name.value.decode(), off.value, r.value, c.value))
    return out, ne.value


def hg_config_internal(cfg: hg_config) -> hg_config:
    """The configuration the kernels run (channel-padded when hidden % 32 != 0)."""
    load()
    out = hg_config()
    _check(_lib.hg_config_internal(ctypes.byref(cfg), ctypes.byref(out)))
    return out


def hg_params_init_host(cfg: hg_config, seed: int) -> np.ndarray:
    load()
    _, total = hg_param_layout(cfg)
    out = np.empty(total, np.float32)
    _check(_lib.hg_params_init_host(ctypes.byref(cfg), seed, _ptr(out)))
    return out


def arena_to_dict(flat: np.ndarray, layout) -> dict:
    """Flat arena -> {name: array of the tensor's shape} (1-row tensors become vectors)."""
    out = {}
    for name, off, r, c in layout:
        v = flat[off:off + r * c]
        out[name] = v.reshape(r, c) if (r > 1 or name.endswith(("W2", "M_x", "M_e", ".U", "W1"))) else v.reshape(c)
    return out


def dict_to_arena(d: dict, layout, total: int) -> np.ndarray:
    flat = np.zeros(total, np.float32)
    for name, off, r, c in layout:
        flat[off:off + r * c] = np.asarray(d[name], np.float32).reshape(-1)
    return flat


# --------------------------------------------------------------------------- device context
class Context:
    """One device context per rank (include/hgnn.h hg_ctx)."""

    def __init__(self, cfg: hg_config, device: int = 0, stream=None):
        import torch  # device memory + the caller's stream only
        load()
        self.cfg = cfg
        self.device = device
        nbytes = _SZ()
        _check(_lib.hg_workspace_bytes(ctypes.byref(cfg), ctypes.byref(nbytes)))
        self.workspace = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=f"cuda:{device}")
        base = self.workspace.data_ptr()
        self._ws_off = (-base) % 256
        self.ws_ptr = base + self._ws_off
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = ctypes.c_void_p()
        _check(_lib.hg_ctx_create(ctypes.byref(cfg), device, ctypes.c_void_p(self.ws_ptr), nbytes.value,
                                  ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)))
        self.handle = h
        self.layout, self.n_params = hg_param_layout(cfg)
        self.internal_cfg = hg_config_internal(cfg)  # widths of the workspace views

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.hg_ctx_destroy(self.handle)
            self.handle = None

    # ---- workspace views (torch tensors aliasing device memory; no copies)
    def view(self, what: int, layer: int = 0):
        off, nb = _I64(), _I64()
        _check(_lib.hg_workspace_view(self.handle, what, layer, ctypes.byref(off), ctypes.byref(nb)))
        o = self._ws_off + off.value
        return self.workspace[o:o + nb.value]

    def batch_get(self, slot: int) -> dict:
        """The packed batch of `slot`, copied to the host and unpacked (hg_batch_get)."""
        cap = self.view(VIEW_SLOT, slot).numel()
        out = np.zeros(cap, np.uint8)
        used = _SZ()
        _check(_lib.hg_batch_get(self.handle, slot, _ptr(out), cap, ctypes.byref(used)))
        return unpack_blob(out[:used.value])

    def view_f32(self, what: int, layer: int = 0):
        import torch
        return self.view(what, layer).view(torch.float32)

    # ---- params / optimizer state
    def params_init(self, seed: int):
        _check(_lib.hg_params_init(self.handle, seed))

    def params_get(self) -> np.ndarray:
        out = np.empty(self.n_params, np.float32)
        _check(_lib.hg_params_get(self.handle, _ptr(out), 0))
        return out

    def params_set(self, flat: np.ndarray):
        flat = np.ascontiguousarray(flat, np.float32)
        assert flat.size == self.n_params
        _check(_lib.hg_params_set(self.handle, _ptr(flat), 0))

    def grads_get(self) -> np.ndarray:
        out = np.empty(self.n_params, np.float32)
        _check(_lib.hg_grads_get(self.handle, _ptr(out), 0))
        return out

    def opt_state_get(self):
        m = np.empty(self.n_params, np.float32)
        v = np.empty(self.n_params, np.float32)
        step = _I64()
        _check(_lib.hg_opt_state_get(self.handle, _ptr(m), _ptr(v), ctypes.byref(step), 0))
        return m, v, step.value

    def opt_state_set(self, m, v, step: int):
        m = np.ascontiguousarray(m, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        _check(_lib.hg_opt_state_set(self.handle, _ptr(m), _ptr(v), step, 0))

    def checkpoint_save(self, path: str):
        """hg_checkpoint_save: config + named parameters + Adam state, CRC-32C."""
        _check(_lib.hg_checkpoint_save(self.handle, os.fsencode(path)))

    def checkpoint_load(self, path: str):
        _check(_lib.hg_checkpoint_load(self.handle, os.fsencode(path)))

    # ---- the training path
    def pack(self, store: Store, ids, slot: int = 0):
        ids = np.ascontiguousarray(ids, np.int64)
        _check(_lib.hg_pack(self.handle, store.handle, _ptr(ids), len(ids), slot))

    def upload(self, blob: np.ndarray, slot: int = 0):
        blob = np.ascontiguousarray(blob, np.uint8)
        _check(_lib.hg_upload_packed(self.handle, _ptr(blob), blob.nbytes, slot))

    def forward(self, slot: int = 0):
        _check(_lib.hg_forward(self.handle, slot))

    def backward(self, slot: int = 0):
        _check(_lib.hg_backward(self.handle, slot))

    def comm_init(self, rank: int, world: int, group=None, force_comm: bool = False):
        """Create the NCCL communicator; the 128-byte id travels over torch.distributed.
        world == 1: no communicator (the exchange is a no-op) unless force_comm, which creates
        a one-rank communicator (the bucketed NCCL path then runs as in a W-rank job)."""
        if world == 1:
            buf = None
            if force_comm:
                buf = np.zeros(128, np.uint8)
                _check(_lib.hg_nccl_unique_id(_ptr(buf)))
            _check(_lib.hg_comm_init(self.handle, _ptr(buf) if buf is not None else None, rank, world))
            return
        buf = nccl_unique_id_broadcast(rank, world, group, device=self.device)
        _check(_lib.hg_comm_init(self.handle, _ptr(buf), rank, world))

    def set_timeout(self, seconds: float):
        """Fail-stop bound of the exchange's device waits and of sync() (hg_set_timeout)."""
        _check(_lib.hg_set_timeout(self.handle, float(seconds)))

    def p2p_init(self, rank: int, world: int, group=None):
        """Map every rank's workspace (CUDA IPC) for the fused peer-memory gradient
        exchange (include/hgnn.h hg_p2p_open); call after comm_init on every rank."""
        import torch
        import torch.distributed as dist
        backend = dist.get_backend(group)
        dev = f"cuda:{self.device}" if backend == "nccl" else "cpu"

        def all_ok(ok: bool) -> bool:  # every rank takes the same path
            f = torch.tensor([1 if ok else 0], device=dev)
            dist.all_reduce(f, op=dist.ReduceOp.MIN, group=group)
            return bool(f.item())

        rec = np.zeros(P2P_HANDLE_BYTES, np.uint8)
        err = None
        try:
            _check(_lib.hg_p2p_handle(self.handle, _ptr(rec)))
        except HgError as e:
            err = e
        if not all_ok(err is None):
            raise err or HgError(8, "peer-memory exchange unavailable on another rank")  # HG_E_CUDA
        t = torch.from_numpy(rec).to(dev)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t, group=group)
        allh = np.ascontiguousarray(np.concatenate([a.cpu().numpy() for a in allt]))
        try:
            _check(_lib.hg_p2p_open(self.handle, _ptr(allh)))
        except HgError as e:
            err = e
        if not all_ok(err is None):
            _lib.hg_p2p_open(self.handle, None)  # back to NCCL everywhere
            raise err or HgError(8, "peer-memory exchange unavailable on another rank")  # HG_E_CUDA

    def p2p_close(self):
        """Back to the NCCL exchange (hg_p2p_open(x, NULL)); gathers the sharded moments."""
        _check(_lib.hg_p2p_open(self.handle, None))

    def exchange_time(self, iters: int = 20, **hyper) -> float:
        """Mean device ms of this ctx's gradient exchange alone (hg_exchange_time; collective)."""
        h = make_adamw(**hyper)
        out = ctypes.c_float()
        _check(_lib.hg_exchange_time(self.handle, ctypes.byref(h), int(iters), ctypes.byref(out)))
        return out.value

    def allreduce_grads(self):
        _check(_lib.hg_allreduce_grads(self.handle))

    def step(self, **hyper):
        h = make_adamw(**hyper)
        _check(_lib.hg_step(self.handle, ctypes.byref(h)))

    def train_step(self, slot: int = 0, graph: bool = True, **hyper):
        h = make_adamw(**hyper)
        _check(_lib.hg_train_step(self.handle, slot, ctypes.byref(h), int(graph)))

    def capture_step(self, slot: int = 0, **hyper):
        h = make_adamw(**hyper)
        _check(_lib.hg_capture_step(self.handle, slot, ctypes.byref(h)))

    def profile_step(self, slot: int = 0, **hyper):
        """Instrumented eager step: {phase: (ms, launches)}."""
        h = make_adamw(**hyper)
        ms = np.zeros(len(PHASES), np.float32)
        nl = np.zeros(len(PHASES), np.int64)
        _check(_lib.hg_profile_step(self.handle, slot, ctypes.byref(h), _ptr(ms), _ptr(nl)))
        return {p: (float(ms[i]), int(nl[i])) for i, p in enumerate(PHASES)}

    def loss(self) -> float:
        out = ctypes.c_float()
        _check(_lib.hg_loss_get(self.handle, ctypes.byref(out)))
        return out.value

    # ---- forward-only evaluation (hg_eval_*)
    def eval_reset(self):
        _check(_lib.hg_eval_reset(self.handle))

    def eval_batch(self, slot: int, graph: bool = True):
        _check(_lib.hg_eval_batch(self.handle, slot, 1 if graph else 0))

    def eval_result(self) -> dict:
        mse, mae, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _check(_lib.hg_eval_result(self.handle, ctypes.byref(mse), ctypes.byref(mae), ctypes.byref(n)))
        return {"mse": mse.value, "mae": mae.value, "count": n.value}

    def eval_pairs(self, slot: int) -> np.ndarray:
        """(y, yhat) parity pairs of the last forward of `slot`, shape [B, 2]."""
        cap = self.cfg.max_graphs
        y, yh = np.zeros(cap, np.float32), np.zeros(cap, np.float32)
        n = ctypes.c_int32()
        _check(_lib.hg_eval_pairs(self.handle, slot, _ptr(y), _ptr(yh), cap, ctypes.byref(n)))
        return np.stack([y[:n.value], yh[:n.value]], axis=1)

    def loss_enqueue(self, i: int):
        """Start the D2H copy of the last loss into pinned ring entry i (no sync)."""
        _check(_lib.hg_loss_enqueue(self.handle, i))

    def loss_fetch(self, i: int) -> float:
        """Wait for ring entry i's copy and return the loss it holds."""
        out = ctypes.c_float()
        _check(_lib.hg_loss_fetch(self.handle, i, ctypes.byref(out)))
        return out.value

    def sync(self):
        _check(_lib.hg_sync(self.handle))

    def launch_count(self) -> int:
        c = _I64()
        _check(_lib.hg_launch_count(self.handle, ctypes.byref(c)))
        return c.value


def nccl_unique_id_broadcast(rank: int, world: int, group=None, device: int = 0) -> np.ndarray:
    """Rank 0 creates the NCCL unique id (hg_nccl_unique_id); torch.distributed
    broadcasts the 128 bytes to every rank (gloo: CPU tensor, nccl: CUDA tensor)."""
    load()
    buf = np.zeros(128, np.uint8)
    if world <= 1:
        return buf
    import torch
    import torch.distributed as dist
    if rank == 0:
        _check(_lib.hg_nccl_unique_id(_ptr(buf)))
    backend = dist.get_backend(group)
    dev = f"cuda:{device}" if backend == "nccl" else "cpu"
    t = torch.from_numpy(buf).to(dev)
    dist.broadcast(t, src=0, group=group)
    return t.cpu().numpy().copy()


def p2p_emulate(ctxs, **hyper):
    """hg_p2p_emulate: the peer-memory exchange of len(ctxs) ranks emulated on one device."""
    load()
    h = make_adamw(**hyper)
    arr = (_P * len(ctxs))(*[c.handle.value for c in ctxs])
    _check(_lib.hg_p2p_emulate(arr, len(ctxs), ctypes.byref(h)))


def bucket_layout(cfg: hg_config) -> list:
    """[(begin, end)] float ranges of the gradient buckets in launch order (hg_bucket_layout)."""
    load()
    n = _I32()
    _check(_lib.hg_bucket_layout(ctypes.byref(cfg), None, 0, ctypes.byref(n)))
    r = np.zeros(2 * n.value, np.int64)
    _check(_lib.hg_bucket_layout(ctypes.byref(cfg), r.ctypes.data_as(_I64P), n.value, ctypes.byref(n)))
    return [(int(r[2 * i]), int(r[2 * i + 1])) for i in range(n.value)]


def pack_threads_set(threads: int):
    load()
    _check(_lib.hg_pack_threads_set(int(threads)))


# C-named module-level entry points (same names as include/hgnn.h)
def hg_ctx_create(cfg, device=0, stream=None) -> Context:
    return Context(cfg, device, stream)


def hg_pack(ctx: Context, store: Store, ids, slot: int = 0):
    ctx.pack(store, ids, slot)


def hg_forward(ctx: Context, slot: int = 0):
    ctx.forward(slot)


def hg_backward(ctx: Context, slot: int = 0):
    ctx.backward(slot)


def hg_allreduce_grads(ctx: Context):
    ctx.allreduce_grads()


def hg_step(ctx: Context, **hyper):
    ctx.step(**hyper)


def hg_train_step(ctx: Context, slot: int = 0, graph: bool = True, **hyper):
    ctx.train_step(slot, graph, **hyper)


def exported_symbols() -> list:
    return list(SIGNATURES)
