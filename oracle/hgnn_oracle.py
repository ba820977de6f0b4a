"""CPU float64 oracle for the HydraGNN (PNA-GCNN) training step — TEST INFRASTRUCTURE.

This module is the plain, slow, obviously-correct definition of what the CUDA
path computes. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import it. The product package
(``paper_2207_11333_b200``) never imports it, and it never imports the
product package: the only code both sides share is the seeded input generator
``molgen`` (no method arithmetic).

Each function cites the passage it follows (PAPER.md = /root/reference/PAPER.md,
SPEC.md = /root/reference/SPEC.md, SURVEY = /root/repo/SURVEY.md §8(c) readings
C1..C21; DESIGN.md "Readings" restates them).

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): hand-derived worked examples
(P1 two-node graph, P2 star graph, tests/golden/), delta by hand (P3), SPEC
closed forms (P4), central finite differences (P5), permutation invariance
(P6), batch independence (P7), DDP split equivalence (P8), an independent
torch.autograd float64 implementation of the same definition, the dense
textbook special case {mean} x {identity} (P9iii), and torch.optim.AdamW in
float64 (P9ii). Every function below is pinned by at least one of them.

Data model: a *store* is the Table-1 dict of PAPER.md:232-253 (as produced by
``molgen.generate``); a *batch* is the packed layout of SURVEY §8(a2).
Floating-point math is float64 throughout (inputs are fp32 values upcast).
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
KEY2 = 0xD1B54A32D192ED03
VAR_FLOOR = 1e-10  # epsilon_v


# --------------------------------------------------------------------------
# counter-based RNG: splitmix64 finalizer, all arithmetic mod 2^64
# --------------------------------------------------------------------------
def splitmix64(x: np.ndarray) -> np.ndarray:
    """z = x + 0x9E3779B97F4A7C15; z = (z ^ z>>30)*0xBF58476D1CE4E5B9;
    z = (z ^ z>>27)*0x94D049BB133111EB; return z ^ z>>31."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _mul64(a: int, b: np.ndarray) -> np.ndarray:
    return np.asarray(b, dtype=np.uint64) * np.uint64(a & MASK64)


# --------------------------------------------------------------------------
# model configuration and parameters
# --------------------------------------------------------------------------
SCALERS = ("identity", "amplification", "attenuation", "linear", "inverse_linear")
DEFAULT_SCALERS = ("identity", "amplification", "attenuation")


def model_scalers(cfg: dict) -> tuple:
    """The configured scaler list (SPEC.md:326 'scalers subset of {identity, amplification,
    attenuation}', identity present; SURVEY C2 default: all three). Model variant (SURVEY §8(f)
    row 3, reading R-scalers): PNA's linear d/delta_lin and inverse_linear delta_lin/d scalers."""
    sc = tuple(cfg.get("scalers", DEFAULT_SCALERS))
    if not sc or sc[0] != "identity" or len(set(sc)) != len(sc) or any(x not in SCALERS for x in sc):
        raise ValueError("scalers: identity first, then distinct names from %s" % (SCALERS,))
    return sc


def param_specs(cfg: dict) -> list:
    """Ordered (name, shape, fan_in, fan_out) list; the order is tensor_idx.

    Per conv layer l: message matrix M = [M_x | M_e]
    of shape [H, F_l + Fe] stored as two tensors (same init scale, fan of the
    whole M), bias b_M [H]; update matrix U [H, 4SH] with column index
    (s*4 + a)*H + c, s over the configured scalers (default identity,
    amplification, attenuation: 12H), a in (mean, min, max, std); bias b_U [H].
    Self-term variant (cfg['self_term'], reading R-self):
    M = [M_x | M_s | M_e] (M_s [H, F_l] multiplies the destination's own x_i) and the update
    matrix [U | U_x] (U_x [H, F_l] multiplies x_i), each stored as separate tensors with the
    whole matrix's fan; order M_x, M_s, M_e, b_M, U, U_x, b_U.
    Head: W1 [Hf, H], b1, W2 [1, Hf], b2.
    """
    H, L, F0, Fe = cfg["hidden"], cfg["layers"], cfg["f_node"], cfg["f_edge"]
    Hf = cfg.get("fc_hidden", H)
    S = len(model_scalers(cfg))
    st = bool(cfg.get("self_term", False))
    out = []
    for l in range(L):
        Fl = F0 if l == 0 else H
        fm = (2 * Fl if st else Fl) + Fe
        fu = 4 * S * H + (Fl if st else 0)
        out.append((f"conv{l}.M_x", (H, Fl), fm, H))
        if st:
            out.append((f"conv{l}.M_s", (H, Fl), fm, H))
        out.append((f"conv{l}.M_e", (H, Fe), fm, H))
        out.append((f"conv{l}.b_M", (H,), 0, 0))
        out.append((f"conv{l}.U", (H, 4 * S * H), fu, H))
        if st:
            out.append((f"conv{l}.U_x", (H, Fl), fu, H))
        out.append((f"conv{l}.b_U", (H,), 0, 0))
    out.append(("head.W1", (Hf, H), H, Hf))
    out.append(("head.b1", (Hf,), 0, 0))
    out.append(("head.W2", (1, Hf), Hf, 1))
    out.append(("head.b2", (1,), 0, 0))
    if cfg.get("node_head", False):  # node-level head (reading R-node-head): same shape, per node
        out.append(("head_n.W1", (Hf, H), H, Hf))
        out.append(("head_n.b1", (Hf,), 0, 0))
        out.append(("head_n.W2", (1, Hf), Hf, 1))
        out.append(("head_n.b2", (1,), 0, 0))
    return out


def init_params(cfg: dict, seed: int) -> dict:
    """w ~ uniform(+-sqrt(6/(fan_in+fan_out))), biases zero.

    RNG per SURVEY C12: key = seed ^ (tensor_idx*0x9E3779B97F4A7C15) ^
    (elem_idx*0xD1B54A32D192ED03); u = (splitmix64(key) >> 11) * 2^-53;
    w = (2u - 1) * a in f64, rounded to fp32 (round-to-nearest-even), returned
    as float64 holding fp32 values.
    """
    params = {}
    for t, (name, shape, fi, fo) in enumerate(param_specs(cfg)):
        n = int(np.prod(shape))
        if fi == 0:
            params[name] = np.zeros(shape, np.float64)
            continue
        a = math.sqrt(6.0 / (fi + fo))
        idx = np.arange(n, dtype=np.uint64)
        key = np.uint64(seed & MASK64) ^ np.uint64((t * GOLDEN) & MASK64) ^ _mul64(KEY2, idx)
        u = (splitmix64(key) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        w = ((2.0 * u - 1.0) * a).astype(np.float32).astype(np.float64)
        params[name] = w.reshape(shape)
    return params


# --------------------------------------------------------------------------
# sharding
# --------------------------------------------------------------------------
def shard(seed: int, epoch: int, rank: int, world: int, n: int) -> np.ndarray:
    """Global per-epoch permutation of [0, n): ascending by (key_i, i) with
    key_i = splitmix64(seed ^ (epoch*GOLDEN) ^ (i*KEY2)); rank r takes the
    permuted positions p = r (mod world), truncated to floor(n/world) (drop-last)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    i = np.arange(n, dtype=np.uint64)
    key = splitmix64(np.uint64(seed & MASK64) ^ np.uint64((epoch * GOLDEN) & MASK64) ^ _mul64(KEY2, i))
    perm = np.lexsort((np.arange(n), key))  # primary key, then index
    per = n // world
    return perm[rank::world][:per].astype(np.int64)


# --------------------------------------------------------------------------
# degree statistic delta
# --------------------------------------------------------------------------
def degree_stat(store: dict, ids=None) -> float:
    """delta = mean over all nodes of the (training) graphs of ln(d + 1), d = in-degree."""
    no, eo = store["node_offset"], store["edge_offset"]
    if ids is None:
        ids = np.arange(len(no) - 1)
    tot, cnt = 0.0, 0
    src = store["edge_index"][0]
    for g in np.asarray(ids):
        n = int(no[g + 1] - no[g])
        d = np.bincount(store["edge_index"][1][eo[g]:eo[g + 1]], minlength=n) if n else np.zeros(0)
        _ = src  # edges are symmetric: in-degree == out-degree
        tot += float(np.log(d.astype(np.float64) + 1.0).sum())
        cnt += n
    return tot / cnt


def degree_stat_linear(store: dict, ids=None) -> float:
    """delta_lin = mean in-degree over all nodes of the (training) graphs: the normaliser of
    PNA's linear / inverse_linear scalers (model variant, reading R-scalers; C4's convention
    of the global training set)."""
    no, eo = store["node_offset"], store["edge_offset"]
    if ids is None:
        ids = np.arange(len(no) - 1)
    ne = sum(int(eo[g + 1] - eo[g]) for g in np.asarray(ids))
    nn = sum(int(no[g + 1] - no[g]) for g in np.asarray(ids))
    return ne / nn  # symmetric edge lists: sum of in-degrees = number of directed edges


# --------------------------------------------------------------------------
# pack / collate
# --------------------------------------------------------------------------
def pack(store: dict, ids) -> dict:
    """Disjoint union of the graphs ``ids`` in input order.

    graph_ptr [B+1] i32 (cumulative node counts); x [N, F0]; y [B];
    CSR over destination nodes: rowptr [N+1] i32, col [E] i32 (in-neighbour
    ids, ascending within a row), eattr [E, Fe] (attribute of the edge
    col -> row); slot [E] u8: for entry k of row r with col[k] = c, the
    position of r inside row c.  Integers only, compared bit-exactly.
    """
    ids = np.asarray(ids, dtype=np.int64)
    if len(ids) == 0:
        raise ValueError("EmptyBatch (SPEC.md:279)")
    no, eo = store["node_offset"], store["edge_offset"]
    xs, eas, srcs, dsts, ys, yns, counts = [], [], [], [], [], [], [0]
    base = 0
    for g in ids:
        n0, n1, e0, e1 = int(no[g]), int(no[g + 1]), int(eo[g]), int(eo[g + 1])
        if n1 == n0:
            raise ValueError("EmptyGraphSlot (SPEC.md:356)")
        xs.append(store["x"][n0:n1])
        s = store["edge_index"][0][e0:e1].astype(np.int64)
        d = store["edge_index"][1][e0:e1].astype(np.int64)
        srcs.append(s + base)  # SPEC.md:283 offset arithmetic
        dsts.append(d + base)
        eas.append(store["edge_attr"][e0:e1])
        ys.append(store["y"][g])
        yns.append(store["y_node"][n0:n1] if "y_node" in store else np.zeros(n1 - n0, np.float32))
        base += n1 - n0
        counts.append(base)
    N = base
    src = np.concatenate(srcs) if srcs else np.zeros(0, np.int64)
    dst = np.concatenate(dsts) if dsts else np.zeros(0, np.int64)
    ea = np.concatenate(eas).astype(np.float32)
    # destination-major CSR: row i = edges (j -> i), ordered by source j ascending
    order = np.lexsort((src, dst))
    row, col, eattr = dst[order], src[order], ea[order]
    rowptr = np.zeros(N + 1, np.int64)
    np.add.at(rowptr, row + 1, 1)
    rowptr = np.cumsum(rowptr)
    pos = np.arange(len(row)) - rowptr[row]
    # slot: position of r inside row c, found by brute-force search
    slot = np.zeros(len(row), np.int64)
    for k in range(len(row)):
        c, r = col[k], row[k]
        seg = col[rowptr[c]:rowptr[c + 1]]
        w = np.nonzero(seg == r)[0]
        if len(w) != 1:
            raise ValueError("edge list not symmetric (SPEC.md:103)")
        slot[k] = w[0]
    return {
        "graph_ptr": np.asarray(counts, np.int32),
        "x": np.concatenate(xs).astype(np.float32),
        "y": np.asarray(ys, np.float32),
        "y_node": np.concatenate(yns).astype(np.float32),
        "rowptr": rowptr.astype(np.int32),
        "col": col.astype(np.int32),
        "eattr": eattr,
        "slot": slot.astype(np.uint8),
        "pos": pos.astype(np.int64),
        "row": row.astype(np.int64),
    }


# --------------------------------------------------------------------------
# forward
# --------------------------------------------------------------------------
def _seg_reduce(ufunc, vals: np.ndarray, rowptr: np.ndarray, fill: float) -> np.ndarray:
    """Per-row reduction of vals [E, C] over CSR rows; empty rows get ``fill``.
    (np.ufunc.reduceat returns a wrong value for empty segments, so they are masked.)"""
    N = len(rowptr) - 1
    out = np.full((N, vals.shape[1]), fill, np.float64)
    deg = np.diff(rowptr)
    ne = np.nonzero(deg > 0)[0]
    if len(ne):
        out[ne] = ufunc.reduceat(vals, rowptr[ne], axis=0)
    return out


def scalers(deg: np.ndarray, delta: float):
    """Degree scalers: amplification
    ln(d+1)/delta, attenuation delta/ln(d+1); both 1 when d = 0."""
    ld = np.log(deg.astype(np.float64) + 1.0)
    amp = np.where(deg > 0, ld / delta, 1.0)
    att = np.where(deg > 0, delta / np.where(deg > 0, ld, 1.0), 1.0)
    return amp, att


def scaler_values(deg: np.ndarray, delta: float, names=DEFAULT_SCALERS, delta_lin: float = None) -> list:
    """Per-node value of each configured scaler (reading
    R-scalers for the PNA variants): identity 1, amplification ln(d+1)/delta, attenuation
    delta/ln(d+1), linear d/delta_lin, inverse_linear delta_lin/d; every scaler is 1 at d = 0."""
    amp, att = scalers(deg, delta)
    d = deg.astype(np.float64)
    has = deg > 0
    out = []
    for nm in names:
        if nm == "identity":
            out.append(np.ones(len(deg)))
        elif nm == "amplification":
            out.append(amp)
        elif nm == "attenuation":
            out.append(att)
        elif nm == "linear":
            out.append(np.where(has, d / delta_lin, 1.0))
        elif nm == "inverse_linear":
            out.append(np.where(has, delta_lin / np.where(has, d, 1.0), 1.0))
        else:
            raise ValueError(nm)
    return out


def conv_forward(Xl: np.ndarray, batch: dict, p: dict, l: int, delta: float, var_floor: float = VAR_FLOOR,
                 cfg: dict = None):
    """One PNA-style GC layer.

    m_{j->i} = M [x_j || e_ji] + b_M over in-neighbours j of i;
    aggregates mean, min, max (first position attaining it), std =
    sqrt(max(var, eps_v)) with the population variance computed two-pass
    (SURVEY C6); d = 0 rows are all zero (C5); S = [A || amp*A || att*A]
    (scaler-major, C3); Z = S U^T + b_U; X_{l+1} = max(Z, 0).
    Variants (cfg): other scaler lists (S = [s_1 A || s_2 A || ...]); self_term: the message
    is M [x_j || x_i || e_ji] + b_M and Z = [S || x_i] [U | U_x]^T + b_U.
    """
    cfg = cfg or {}
    names = model_scalers(cfg)
    self_t = bool(cfg.get("self_term", False))
    rowptr = batch["rowptr"].astype(np.int64)
    col = batch["col"].astype(np.int64)
    row, pos = batch["row"], batch["pos"]
    deg = np.diff(rowptr)
    if self_t:
        M = np.concatenate([p[f"conv{l}.M_x"], p[f"conv{l}.M_s"], p[f"conv{l}.M_e"]], axis=1)
        cat = np.concatenate([Xl[col], Xl[row], batch["eattr"].astype(np.float64)], axis=1)
    else:
        M = np.concatenate([p[f"conv{l}.M_x"], p[f"conv{l}.M_e"]], axis=1)
        cat = np.concatenate([Xl[col], batch["eattr"].astype(np.float64)], axis=1)
    msg = cat @ M.T + p[f"conv{l}.b_M"]
    N = len(deg)
    dd = np.maximum(deg, 1).astype(np.float64)[:, None]
    mean = _seg_reduce(np.add, msg, rowptr, 0.0) / dd
    mx = _seg_reduce(np.maximum, msg, rowptr, 0.0)
    mn = _seg_reduce(np.minimum, msg, rowptr, 0.0)
    big = np.iinfo(np.int64).max
    posb = np.broadcast_to(pos[:, None], msg.shape)
    argmax = _seg_reduce(np.minimum, np.where(msg == mx[row], posb, big).astype(np.float64), rowptr, 0).astype(np.int64)
    argmin = _seg_reduce(np.minimum, np.where(msg == mn[row], posb, big).astype(np.float64), rowptr, 0).astype(np.int64)
    cen = msg - mean[row]
    var = _seg_reduce(np.add, cen * cen, rowptr, 0.0) / dd
    std = np.sqrt(np.maximum(var, var_floor))
    empty = deg == 0
    std[empty] = 0.0
    A = np.concatenate([mean, mn, mx, std], axis=1)
    amp, att = scalers(deg, delta)
    sv = scaler_values(deg, delta, names, cfg.get("delta_lin"))
    S = np.concatenate([s[:, None] * A for s in sv], axis=1)
    Uf = p[f"conv{l}.U"]
    if self_t:
        S = np.concatenate([S, Xl], axis=1)
        Uf = np.concatenate([Uf, p[f"conv{l}.U_x"]], axis=1)
    Z = S @ Uf.T + p[f"conv{l}.b_U"]
    X1 = np.maximum(Z, 0.0)
    cache = dict(Xl=Xl, cat=cat, msg=msg, mean=mean, mn=mn, mx=mx, argmax=argmax, argmin=argmin,
                 var=var, std=std, A=A, S=S, Z=Z, amp=amp, att=att, sv=sv, deg=deg, N=N)
    return X1, cache


def forward(params: dict, batch: dict, cfg: dict, delta: float):
    """Full forward: L GC layers -> global mean pool ->
    FC head ReLU(G W1^T + b1) W2^T + b2 -> MSE."""
    X = batch["x"].astype(np.float64)
    caches = []
    for l in range(cfg["layers"]):
        X, c = conv_forward(X, batch, params, l, delta, cfg.get("var_floor", VAR_FLOOR), cfg)
        caches.append(c)
    gp = batch["graph_ptr"].astype(np.int64)
    ng = np.diff(gp)
    if np.any(ng == 0):
        raise ValueError("EmptyGraphSlot (SPEC.md:356)")
    G = np.add.reduceat(X, gp[:-1], axis=0) / ng[:, None]
    hpre = G @ params["head.W1"].T + params["head.b1"]
    hid = np.maximum(hpre, 0.0)
    yhat = (hid @ params["head.W2"].T)[:, 0] + params["head.b2"][0]
    y = batch["y"].astype(np.float64)
    loss = float(np.mean((yhat - y) ** 2))
    head = dict(XL=X, G=G, hpre=hpre, hid=hid, yhat=yhat, ng=ng, gp=gp)
    if cfg.get("node_head", False):
        # node-level head ("hybrid node-level and graph-level properties";
        # reading R-node-head): per node ReLU(X_L W1n^T + b1n) W2n^T + b2n, node MSE over the
        # batch's nodes, added to the graph MSE with weight node_weight
        hn_pre = X @ params["head_n.W1"].T + params["head_n.b1"]
        hn = np.maximum(hn_pre, 0.0)
        yn = (hn @ params["head_n.W2"].T)[:, 0] + params["head_n.b2"][0]
        loss_n = float(np.mean((yn - batch["y_node"].astype(np.float64)) ** 2))
        loss = loss + cfg.get("node_weight", 1.0) * loss_n
        head.update(hn_pre=hn_pre, hn=hn, yn=yn, loss_n=loss_n)
    return loss, yhat, dict(layers=caches, head=head)


# --------------------------------------------------------------------------
# backward
# --------------------------------------------------------------------------
def backward(params: dict, batch: dict, cfg: dict, cache: dict, decisions: dict | None = None) -> dict:
    """Reverse-mode gradients of the mean MSE loss w.r.t. every parameter.

    Subgradients: ReLU'(0) = 0 (C8); min/max route to the first position
    attaining the extremum (C7); the std derivative is
    (m_k - mu)/(d * std) when var > eps_v and 0 otherwise (C6).
    ``decisions`` (optional, per layer index) replaces the oracle's own
    discrete decisions in the ambiguity band (SURVEY C8 decision replay):
    keys 'relu' (bool [N,H], Z > 0), 'argmax'/'argmin' (int [N,H]),
    'varflag' (bool [N,H], var > eps_v); 'head_relu' (bool [B,Hf]) at top level.
    """
    decisions = decisions or {}
    h = cache["head"]
    B = len(h["yhat"])
    y = batch["y"].astype(np.float64)
    g = {}
    dy = 2.0 * (h["yhat"] - y) / B
    g["head.W2"] = (dy @ h["hid"])[None, :]
    g["head.b2"] = np.array([dy.sum()])
    dhid = dy[:, None] * params["head.W2"][0][None, :]
    hmask = decisions.get("head_relu", h["hpre"] > 0)
    dhpre = dhid * hmask
    g["head.W1"] = dhpre.T @ h["G"]
    g["head.b1"] = dhpre.sum(0)
    dG = dhpre @ params["head.W1"]
    gp, ng = h["gp"], h["ng"]
    gid = np.repeat(np.arange(B), ng)
    dX = dG[gid] / ng[gid][:, None]
    if cfg.get("node_head", False):
        Nn = len(h["yn"])
        dyn = 2.0 * cfg.get("node_weight", 1.0) * (h["yn"] - batch["y_node"].astype(np.float64)) / Nn
        g["head_n.W2"] = (dyn @ h["hn"])[None, :]
        g["head_n.b2"] = np.array([dyn.sum()])
        nmask = decisions.get("node_relu", h["hn_pre"] > 0)
        dhn = dyn[:, None] * params["head_n.W2"][0][None, :] * nmask
        g["head_n.W1"] = dhn.T @ h["XL"]
        g["head_n.b1"] = dhn.sum(0)
        dX = dX + dhn @ params["head_n.W1"]
    col = batch["col"].astype(np.int64)
    row, pos = batch["row"], batch["pos"]
    H = cfg["hidden"]
    self_t = bool(cfg.get("self_term", False))
    nS = len(model_scalers(cfg))
    for l in reversed(range(cfg["layers"])):
        c = cache["layers"][l]
        dec = decisions.get(l, {})
        relu = dec.get("relu", c["Z"] > 0)
        dZ = dX * relu
        F = c["Xl"].shape[1]
        dUf = dZ.T @ c["S"]
        g[f"conv{l}.U"] = dUf[:, :4 * nS * H]
        Uf = params[f"conv{l}.U"]
        if self_t:
            g[f"conv{l}.U_x"] = dUf[:, 4 * nS * H:]
            Uf = np.concatenate([Uf, params[f"conv{l}.U_x"]], axis=1)
        g[f"conv{l}.b_U"] = dZ.sum(0)
        dS = dZ @ Uf
        dA = sum(s[:, None] * dS[:, k * 4 * H:(k + 1) * 4 * H] for k, s in enumerate(c["sv"]))
        dX_self = dS[:, 4 * nS * H:] if self_t else None
        dmean, dmin, dmax, dstd = (dA[:, a * H:(a + 1) * H] for a in range(4))
        argmax = dec.get("argmax", c["argmax"])
        argmin = dec.get("argmin", c["argmin"])
        varflag = dec.get("varflag", c["var"] > cfg.get("var_floor", VAR_FLOOR))
        deg = np.maximum(c["deg"], 1).astype(np.float64)
        dr = deg[row][:, None]
        p2 = pos[:, None]
        dm = (dmean[row] / dr
              + (p2 == argmax[row]) * dmax[row]
              + (p2 == argmin[row]) * dmin[row]
              + varflag[row] * dstd[row] * (c["msg"] - c["mean"][row]) / (dr * np.where(c["std"][row] > 0, c["std"][row], 1.0)))
        dM = dm.T @ c["cat"]
        g[f"conv{l}.M_x"] = dM[:, :F]
        if self_t:
            g[f"conv{l}.M_s"] = dM[:, F:2 * F]
            g[f"conv{l}.M_e"] = dM[:, 2 * F:]
        else:
            g[f"conv{l}.M_e"] = dM[:, F:]
        g[f"conv{l}.b_M"] = dm.sum(0)
        if l > 0:
            dX = np.zeros_like(c["Xl"])
            np.add.at(dX, col, dm @ params[f"conv{l}.M_x"])  # through the sources x_j
            if self_t:
                np.add.at(dX, row, dm @ params[f"conv{l}.M_s"])  # through the destinations x_i
                dX = dX + dX_self  # through the update's x_i block
    return g


# --------------------------------------------------------------------------
# AdamW
# --------------------------------------------------------------------------
def adamw_step(params: dict, grads: dict, state: dict, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01):
    """Decoupled weight decay then bias-corrected Adam (Loshchilov & Hutter,
    PyTorch ordering), applied to every tensor including biases.
    state = {'m': {...}, 'v': {...}, 'step': int}; returns (params, state) new copies."""
    t = state["step"] + 1
    newp, m, v = {}, {}, {}
    for k, th in params.items():
        gk = grads[k]
        th = th * (1.0 - lr * weight_decay)
        m[k] = beta1 * state["m"][k] + (1.0 - beta1) * gk
        v[k] = beta2 * state["v"][k] + (1.0 - beta2) * gk * gk
        mhat = m[k] / (1.0 - beta1 ** t)
        vhat = v[k] / (1.0 - beta2 ** t)
        newp[k] = th - lr * mhat / (np.sqrt(vhat) + eps)
    return newp, {"m": m, "v": v, "step": t}


def zero_state(params: dict) -> dict:
    return {"m": {k: np.zeros_like(v) for k, v in params.items()},
            "v": {k: np.zeros_like(v) for k, v in params.items()}, "step": 0}


# --------------------------------------------------------------------------
# DDP
# --------------------------------------------------------------------------
def allreduce_mean(per_rank: list) -> dict:
    """Elementwise mean over ranks (rank-ascending sum, then divide)."""
    W = len(per_rank)
    out = {}
    for k in per_rank[0]:
        acc = np.zeros_like(per_rank[0][k])
        for r in range(W):
            acc = acc + per_rank[r][k]
        out[k] = acc / W
    return out


def train_step(params, state, store, ids, cfg, delta, hyper=None, world=1):
    """One DDP iteration simulated in-process: each of ``world``
    ranks packs its equal sub-batch, runs forward+backward; gradients are
    averaged; every rank applies the identical AdamW step."""
    hyper = hyper or {}
    ids = np.asarray(ids)
    B = len(ids) // world
    grads, losses = [], []
    for r in range(world):
        b = pack(store, ids[r * B:(r + 1) * B])
        loss, _, cache = forward(params, b, cfg, delta)
        grads.append(backward(params, b, cfg, cache))
        losses.append(loss)
    g = allreduce_mean(grads)
    newp, newstate = adamw_step(params, g, state, **hyper)
    return newp, newstate, float(np.mean(losses)), g


# --------------------------------------------------------------------------
# decision replay for parity
# --------------------------------------------------------------------------
def replay(cache: dict, gpu: list, tau_arg: float = 1e-6, tau_relu=1e-6, tau_head: float = 1e-6,
           head_relu_gpu=None, node_relu_gpu=None):
    """Decision replay for parity: where several discrete
    decisions are correct, adopt the GPU's; check the rest.

    A GPU decision is *valid* if it is optimal within a band in the oracle's own
    float64 values:
      argmax: m[gpu position] >= max - tau_arg*|m|_inf   (argmin symmetric),
              tau_arg = 1e-6;
      relu:   Z >= -tau*|Z|_inf if the GPU kept the unit, Z <= tau*|Z|_inf if not,
              tau = tau_relu (per layer: a float, or a list with one value per
              layer) -- the parity harness passes the GPU's measured forward error
              bound of that layer (reading R-replay); tau_head for the head;
      varflag: var within 0.5*eps_v of eps_v, or the same side as the GPU.
    Valid GPU decisions are adopted (exact ties such as automorphic atoms, whose
    float64 and fp32 roundings can break the tie differently, are legitimately
    resolved either way); invalid ones are counted and the oracle keeps its own
    decision, so they show up in the gradient error too.
    Overrides whose two candidates are equal to float64 rounding (|gap| <= 1e-12 of
    the layer's max, i.e. algebraic ties such as automorphic atoms, where the
    oracle's own summation order decides) are counted apart as 'tie_overrides'.
    Returns (decisions, {'overrides', 'tie_overrides', 'overrides_by', 'out_of_band',
    'out_of_band_by'})."""
    dec, n, bad, nt = {}, 0, 0, 0
    TIE = 1e-12
    by = {"relu": 0, "argmax": 0, "argmin": 0, "varflag": 0, "head_relu": 0}
    ov = dict(by)  # overrides per decision kind (diagnostic)
    for l, (c, gdec) in enumerate(zip(cache["layers"], gpu)):
        tau_r = float(tau_relu[l]) if np.ndim(tau_relu) else float(tau_relu)
        zs = np.abs(c["Z"]).max() if c["Z"].size else 0.0
        msg = c["msg"]
        ms = np.abs(msg).max() if msg.size else 0.0
        deg = c["deg"]
        rowptr = np.concatenate([[0], np.cumsum(deg)])
        has = (deg > 0)[:, None]
        own = dict(relu=c["Z"] > 0, argmax=c["argmax"], argmin=c["argmin"], varflag=c["var"] > VAR_FLOOR)
        d = dict(own)
        if "relu" in gdec:
            g = np.asarray(gdec["relu"])
            valid = np.where(g, c["Z"] >= -tau_r * zs, c["Z"] <= tau_r * zs)
            diff = g != own["relu"]
            tie = np.abs(c["Z"]) <= TIE * zs
            n += int((valid & diff & ~tie).sum())
            nt += int((valid & diff & tie).sum())
            ov["relu"] += int((valid & diff).sum())
            nb = int((~valid & diff).sum())
            bad += nb
            by["relu"] += nb
            d["relu"] = np.where(valid, g, own["relu"])
        for k, sign in (("argmax", 1.0), ("argmin", -1.0)):
            if k not in gdec:
                continue
            g = np.asarray(gdec[k]).astype(np.int64)
            gpos = np.clip(g, 0, np.maximum(deg - 1, 0)[:, None])
            idx = rowptr[:-1][:, None] + gpos
            idx = np.where(has, idx, 0)
            chan = np.broadcast_to(np.arange(msg.shape[1] if msg.size else g.shape[1]), g.shape)
            gval = msg[idx, chan] if msg.size else np.zeros(g.shape)
            ext = c["mx"] if sign > 0 else c["mn"]
            valid = (sign * (gval - ext) >= -tau_arg * ms) & (g < np.maximum(deg, 1)[:, None])
            valid |= ~has
            diff = (g != own[k]) & has
            tie = np.abs(gval - ext) <= TIE * ms
            n += int((valid & diff & ~tie).sum())
            nt += int((valid & diff & tie).sum())
            ov[k] += int((valid & diff).sum())
            nb = int((~valid & diff).sum())
            bad += nb
            by[k] += nb
            d[k] = np.where(valid & has, g, own[k])
        if "varflag" in gdec:
            g = np.asarray(gdec["varflag"])
            band = np.abs(c["var"] - VAR_FLOOR) < 0.5 * VAR_FLOOR
            diff = (g != own["varflag"]) & has
            n += int((band & diff).sum())
            ov["varflag"] += int((band & diff).sum())
            nb = int((~band & diff).sum())
            bad += nb
            by["varflag"] += nb
            d["varflag"] = np.where(band, g, own["varflag"])
        dec[l] = d
    if head_relu_gpu is not None:
        hp = cache["head"]["hpre"]
        hs = np.abs(hp).max() if hp.size else 0.0
        g = np.asarray(head_relu_gpu)
        own = hp > 0
        valid = np.where(g, hp >= -tau_head * hs, hp <= tau_head * hs)
        diff = g != own
        tie = np.abs(hp) <= TIE * hs
        n += int((valid & diff & ~tie).sum())
        nt += int((valid & diff & tie).sum())
        ov["head_relu"] += int((valid & diff).sum())
        nb = int((~valid & diff).sum())
        bad += nb
        by["head_relu"] += nb
        dec["head_relu"] = np.where(valid, g, own)
    if node_relu_gpu is not None:  # the node-level head's hidden units (variant), same rule
        hp = cache["head"]["hn_pre"]
        hs = np.abs(hp).max() if hp.size else 0.0
        g = np.asarray(node_relu_gpu)
        own = hp > 0
        valid = np.where(g, hp >= -tau_head * hs, hp <= tau_head * hs)
        diff = g != own
        tie = np.abs(hp) <= TIE * hs
        n += int((valid & diff & ~tie).sum())
        nt += int((valid & diff & tie).sum())
        ov["head_relu"] += int((valid & diff).sum())
        nb = int((~valid & diff).sum())
        bad += nb
        by["head_relu"] += nb
        dec["node_relu"] = np.where(valid, g, own)
    return dec, {"overrides": n, "tie_overrides": nt, "overrides_by": ov, "out_of_band": bad,
                 "out_of_band_by": by}


# ---------------------------------------------------------------- evaluation
def regression_metrics(yhat, y) -> dict:
    """MSE and MAE of predictions (SPEC.md:385-389 `evaluate`; "measured in mean
    absolute error (MAE)"): MSE = (1/n) sum (yhat - y)^2, MAE = (1/n) sum |yhat - y|, n = #graphs."""
    yhat = np.asarray(yhat, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if yhat.shape != y.shape or yhat.size == 0:
        raise ValueError("need equally long, non-empty prediction and target vectors")
    e = yhat - y
    return {"mse": float(np.mean(e * e)), "mae": float(np.mean(np.abs(e))), "count": int(y.size)}


def evaluate(params: dict, store: dict, batches, cfg: dict, delta: float) -> dict:
    """Forward-only evaluation over a list of batches: metrics over all
    graphs of all batches plus the (y, yhat) parity pairs in batch order."""
    ys, yh = [], []
    for ids in batches:
        batch = pack(store, ids)
        _, yhat, _ = forward(params, batch, cfg, delta)
        ys.append(batch["y"])
        yh.append(yhat)
    y = np.concatenate(ys)
    yhat = np.concatenate(yh)
    out = regression_metrics(yhat, y)
    out["pairs"] = np.stack([y, yhat], axis=1)
    return out
