"""Small helpers shared by the tests (no method arithmetic)."""
import numpy as np


def make_store(graphs, f_edge=None):
    """Build a Table-1 store dict from explicit graphs.

    graphs: list of (x [n, F] array-like, bonds list of (a, b, attr-vector), y).
    Each undirected bond becomes two directed edges with identical attributes
    (SPEC.md:103); per graph edges sorted by (src, dst).
    """
    xs, srcs, dsts, eas, ys = [], [], [], [], []
    no, eo = [0], [0]
    for x, bonds, y in graphs:
        x = np.asarray(x, np.float32)
        if x.ndim == 1:
            x = x[:, None]
        es = []
        for a, b, attr in bonds:
            attr = np.atleast_1d(np.asarray(attr, np.float32))
            es.append((a, b, attr))
            es.append((b, a, attr))
        es.sort(key=lambda t: (t[0], t[1]))
        xs.append(x)
        for s, d, at in es:
            srcs.append(s)
            dsts.append(d)
            eas.append(at)
        ys.append(y)
        no.append(no[-1] + len(x))
        eo.append(eo[-1] + len(es))
    fe = f_edge if f_edge is not None else (len(eas[0]) if eas else 1)
    return {
        "node_offset": np.asarray(no, np.int64),
        "edge_offset": np.asarray(eo, np.int64),
        "x": np.concatenate(xs).astype(np.float32),
        "edge_index": np.asarray([srcs, dsts], np.int32).reshape(2, -1),
        "edge_attr": np.asarray(eas, np.float32).reshape(-1, fe),
        "y": np.asarray(ys, np.float32),
        "f_node": xs[0].shape[1],
        "f_edge": fe,
    }


def subset_store(store, ids):
    """Store restricted to graphs ``ids`` (renumbered 0..len-1)."""
    graphs = []
    no, eo = store["node_offset"], store["edge_offset"]
    for g in ids:
        x = store["x"][no[g]:no[g + 1]]
        s = store["edge_index"][0][eo[g]:eo[g + 1]]
        d = store["edge_index"][1][eo[g]:eo[g + 1]]
        a = store["edge_attr"][eo[g]:eo[g + 1]]
        bonds = [(int(si), int(di), a[k]) for k, (si, di) in enumerate(zip(s, d)) if si < di]
        graphs.append((x, bonds, store["y"][g]))
    return make_store(graphs, f_edge=store["edge_attr"].shape[1])


def max_scaled(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.abs(b).max()
    if den == 0:
        return float(np.abs(a - b).max()) if a.size else 0.0
    return float(np.abs(a - b).max() / den)


def normwise(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    if den == 0:
        return float(np.linalg.norm(a - b))
    return float(np.linalg.norm(a - b) / den)


def small_cfg(F0, H, L, Fe=4, Hf=None):
    return {"f_node": F0, "f_edge": Fe, "hidden": H, "layers": L, "fc_hidden": Hf or H}
