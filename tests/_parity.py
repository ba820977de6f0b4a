"""GPU-vs-oracle parity harness (used by tests/test_gpu_*.py and smoke()).

Runs one training step through the C-ABI (paper_2207_11333_b200.hgnn) and the
float64 oracle on the same seeded inputs and parameters, and returns the
comparison metrics of SURVEY §8(c) C19:
  forward (yhat, loss, per-layer X): max |diff| / max |ref|    (bar 1e-4)
  gradients: per tensor max-scaled and normwise                (bar 1e-3)
  one-step Adam moments m1, v1: per tensor normwise            (bar 1e-3)
  one-step params: per tensor normwise over the components whose oracle
  gradient is >= 100 eps (bar 1e-3); the others -- where Adam's first step
  lr*g/(|g|+eps) is ill-conditioned -- are counted and checked against the
  step bound |theta1 - theta0 (1 - lr wd)| <= lr (reading R-adam-eps)
  decision replay (C8): oracle decisions inside the ambiguity band (argmin /
  argmax 1e-6, ReLU the GPU's measured forward error of that layer) are
  replaced by the GPU's; the override count is reported.
Every oracle input is the oracle's own (or the GPU's parameters / moments it
re-syncs to before the step, SURVEY §8(d) "Per-step re-sync"); no GPU output
enters the oracle's arithmetic.
"""
import numpy as np

import molgen
import oracle as O
from paper_2207_11333_b200 import hgnn
from tests._util import max_scaled, normwise  # noqa: F401

FWD_TOL = 1e-4
GRAD_TOL = 1e-3
PARAM_TOL = 1e-3


def capacity_for(data, B):
    nn = np.diff(data["node_offset"])
    ne = np.diff(data["edge_offset"])
    return int(np.sort(nn)[-B:].sum()), int(max(1, np.sort(ne)[-B:].sum()))


def oracle_cfg(cfg):
    """The oracle's model dict of a C-ABI configuration (variants: scaler set, self-term)."""
    return {"f_node": cfg.f_node, "f_edge": cfg.f_edge, "hidden": cfg.hidden, "layers": cfg.layers,
            "fc_hidden": cfg.fc_hidden, "var_floor": float(np.float32(cfg.var_floor)),
            "scalers": hgnn.scaler_names(cfg.scalers), "self_term": bool(cfg.flags & hgnn.HG_FLAG_SELF_TERM),
            "delta_lin": float(cfg.delta_lin), "node_head": bool(cfg.flags & hgnn.HG_FLAG_NODE_HEAD),
            "node_weight": float(np.float32(cfg.node_weight))}


def gpu_X(ctx, l, N, H):
    """X_{l+1} [N, H] (the logical channels of the internal-width workspace view)."""
    Hp = ctx.internal_cfg.hidden
    return ctx.view_f32(hgnn.VIEW_X, l)[:N * Hp].cpu().numpy().reshape(N, Hp)[:, :H]


def gpu_decisions(ctx, N, H, L):
    dec = []
    Hp = ctx.internal_cfg.hidden
    for l in range(L):
        arg = ctx.view(hgnn.VIEW_ARG, l)[:N * 2 * Hp].cpu().numpy().reshape(N, 2 * Hp)
        X = gpu_X(ctx, l, N, H)
        amn = arg[:, :H].astype(np.int64)
        amx = (arg[:, Hp:Hp + H] & 0x7F).astype(np.int64)
        flag = (arg[:, Hp:Hp + H] & 0x80) != 0
        dec.append(dict(relu=X > 0, argmax=amx, argmin=amn, varflag=flag))
    return dec


class StepResult(dict):
    pass


def adam_ratio_bound(t, hyper):
    """Largest |m^_t / sqrt(v^_t)| any gradient sequence can give at Adam step t (Cauchy-Schwarz
    on m_t = (1-b1) sum_k b1^k g_(t-k), v_t = (1-b2) sum_k b2^k g_(t-k)^2, with the bias
    corrections): 1 at t = 1, slightly above 1 later (b1^2 < b2)."""
    b1, b2 = hyper["beta1"], hyper["beta2"]
    r = sum((b1 * b1 / b2) ** k for k in range(t))
    return (1 - b1) / np.sqrt(1 - b2) * np.sqrt(r) * np.sqrt(1 - b2 ** t) / (1 - b1 ** t)


def run_step_parity(data, ids, ctx, cfg, delta, hyper=None, do_step=True, graph=False, tau_arg=1e-6,
                    grad_bar=None):
    """One step on GPU (ctx must hold the parameters) and on the oracle from the
    GPU's current parameters / optimizer state. Returns StepResult of metrics."""
    import torch
    hyper = hyper or dict(hgnn.DEFAULT_ADAMW)
    layout = ctx.layout
    p0 = ctx.params_get()
    m0, v0, step0 = ctx.opt_state_get()
    params = {k: np.asarray(v, np.float64) for k, v in hgnn.arena_to_dict(p0, layout).items()}
    st = {"m": {k: np.asarray(v, np.float64) for k, v in hgnn.arena_to_dict(m0, layout).items()},
          "v": {k: np.asarray(v, np.float64) for k, v in hgnn.arena_to_dict(v0, layout).items()}, "step": step0}
    store = ctx._store
    ctx.pack(store, ids, 0)
    if graph:
        ctx.train_step(0, graph=True, **hyper)
        torch.cuda.synchronize()
    else:
        ctx.forward(0)
        ctx.backward(0)
        torch.cuda.synchronize()
    ocfg = oracle_cfg(cfg)
    b = O.pack(data, ids)
    N, H, L, B = len(b["x"]), cfg.hidden, cfg.layers, len(ids)
    loss, yhat, cache = O.forward(params, b, ocfg, delta)
    res = StepResult()
    gy = ctx.view_f32(hgnn.VIEW_YHAT)[:B].cpu().numpy()
    res["yhat"] = float(np.abs(gy - yhat).max() / max(np.abs(yhat).max(), 1e-30))
    gl = float(ctx.view_f32(hgnn.VIEW_LOSS)[0].item()) if not graph else None
    if gl is not None:
        res["loss"] = abs(gl - loss) / max(abs(loss), 1e-30)
    xs = []
    for l in range(L):
        X = gpu_X(ctx, l, N, H)
        ref = np.maximum(cache["layers"][l]["Z"], 0)
        xs.append(float(np.abs(X - ref).max() / max(np.abs(ref).max(), 1e-30)))
    res["X"] = max(xs)
    node_relu = None
    if cfg.flags & hgnn.HG_FLAG_NODE_HEAD:  # node-level head outputs (variant)
        yn = ctx.view_f32(hgnn.VIEW_NODE_YHAT)[:N].cpu().numpy()
        ref_n = cache["head"]["yn"]
        res["yhat_node"] = float(np.abs(yn - ref_n).max() / max(np.abs(ref_n).max(), 1e-30))
        Hfi = ctx.internal_cfg.fc_hidden
        node_relu = ctx.view_f32(hgnn.VIEW_NODE_HPRE)[:N * Hfi].cpu().numpy().reshape(N, Hfi)[:, :cfg.fc_hidden] > 0
    Hfp = ctx.internal_cfg.fc_hidden
    hpre = ctx.view_f32(hgnn.VIEW_HPRE)[:B * Hfp].cpu().numpy().reshape(B, Hfp)[:, :cfg.fc_hidden]
    # ReLU replay band per layer: the GPU's measured forward error of that layer (x2), at least
    # C8's 1e-6 -- a unit whose |Z| exceeds the demonstrated error cannot legitimately flip
    tau_relu = [max(1e-6, 2.0 * e) for e in xs]
    hp_ref = cache["head"]["hpre"]
    tau_head = max(1e-6, 2.0 * float(np.abs(hpre - hp_ref).max() / max(np.abs(hp_ref).max(), 1e-30)))
    res["tau_relu"] = max(tau_relu)
    if tau_arg is None:  # (reduced-precision mode: argmin/argmax band at the measured forward error too)
        tau_arg = max(tau_relu)
    dec, counts = O.replay(cache, gpu_decisions(ctx, N, H, L), tau_arg=tau_arg, tau_relu=tau_relu, tau_head=tau_head,
                           head_relu_gpu=hpre > 0, node_relu_gpu=node_relu)
    res["overrides"] = counts["overrides"]
    res["overrides_by"] = counts["overrides_by"]
    res["tie_overrides"] = counts["tie_overrides"]
    res["out_of_band"] = counts["out_of_band"]
    res["out_of_band_by"] = counts["out_of_band_by"]
    res["cells"] = int(sum(c["Z"].size * 4 for c in cache["layers"]))
    g = O.backward(params, b, ocfg, cache, dec)
    gg = hgnn.arena_to_dict(ctx.grads_get(), layout) if not graph or not do_step else None
    if gg is not None:
        res["grad_maxscaled"] = {k: max_scaled(gg[k], g[k]) for k in g}
        res["grad_normwise"] = {k: normwise(gg[k], g[k]) for k in g}
    if do_step:
        if not graph:
            ctx.step(**hyper)
            torch.cuda.synchronize()
        newp, newst = O.adamw_step(params, g, st, **{k: hyper[k] for k in ("lr", "beta1", "beta2", "eps",
                                                                            "weight_decay")})
        gp = hgnn.arena_to_dict(ctx.params_get(), layout)
        m1, v1, step1 = ctx.opt_state_get()
        gm, gv = hgnn.arena_to_dict(m1, layout), hgnn.arena_to_dict(v1, layout)
        res["step"] = (step1, newst["step"])
        # the moments are well-conditioned functions of the gradient
        res["m_normwise"] = {k: normwise(gm[k], newst["m"][k]) for k in g}
        res["v_normwise"] = {k: normwise(gv[k], newst["v"][k]) for k in g}
        # DESIGN.md reading R-adam-eps: theta1 = theta0 (1 - lr wd) - lr m^/(sqrt(v^) + eps) has
        # sensitivity lr/eps = 1e5 to g at g = 0 and is ~ -lr sign(g) elsewhere, so theta1 is
        # compared only where the oracle gradient is >= 100 eps AND its sign is fixed by the
        # gradient bar (|g| >= grad_bar max|g| of its tensor: the GPU gradient may differ by up to
        # that much); elsewhere the GPU's step must respect |m^/(sqrt(v^)+eps)| <= 1. The mask
        # uses oracle values only.
        floor = 100.0 * hyper["eps"]
        gbar = GRAD_TOL if grad_bar is None else grad_bar
        pn, n_ill, bound_bad = {}, 0, 0
        decay = 1.0 - hyper["lr"] * hyper["weight_decay"]
        for k in g:
            ok = np.abs(g[k]) >= max(floor, gbar * float(np.abs(g[k]).max()))
            a_ = np.asarray(gp[k], np.float64).reshape(g[k].shape)
            n_ill += int((~ok).sum())
            if ok.any():
                pn[k] = normwise(a_[ok], newp[k][ok])
            step_ = np.abs(a_[~ok] - params[k][~ok] * decay)
            bound_bad += int((step_ > hyper["lr"] * adam_ratio_bound(newst["step"], hyper) * (1 + 1e-3) + 1e-7).sum())
        res["param_normwise"] = pn
        res["adam_ill_conditioned"] = n_ill
        res["adam_step_bound_violations"] = bound_bad
    res["oracle_loss"] = loss
    return res


def make_ctx(data, B, H, L, seed=2, n_slots=2, Hf=None, flags=0, max_degree=None, scalers=0, node_weight=1.0):
    """A ctx sized for the B largest graphs of `data`, parameters from the C12 init
    (scalers: an HG_SCALER_* bit set; flags: HG_FLAG_*)."""
    delta = O.degree_stat(data)
    delta_lin = O.degree_stat_linear(data)
    maxn, maxe = capacity_for(data, B)
    store = hgnn.Store(data)
    if max_degree is None:
        max_degree = store.stats()["max_degree"]
    cfg = hgnn.make_config(data["f_node"], 4, H, L, B, maxn, maxe, delta, fc_hidden=Hf, n_slots=n_slots,
                           flags=flags, max_degree=max_degree, scalers=scalers, delta_lin=delta_lin,
                           node_weight=node_weight)
    ctx = hgnn.Context(cfg)
    ctx.params_init(seed)
    ctx._store = store
    return ctx, cfg, delta


def assert_parity(res, fwd_tol=FWD_TOL, grad_tol=GRAD_TOL, param_tol=PARAM_TOL, override_frac=1e-4):
    bad = []
    if res["yhat"] > fwd_tol:
        bad.append(("yhat", res["yhat"]))
    if "loss" in res and res["loss"] > fwd_tol:
        bad.append(("loss", res["loss"]))
    if res["X"] > fwd_tol:
        bad.append(("X", res["X"]))
    if res.get("yhat_node", 0.0) > fwd_tol:
        bad.append(("yhat_node", res["yhat_node"]))
    # GPU discrete decisions (ReLU masks, argmin/argmax, std floor) must agree with the
    # oracle wherever the oracle's margin exceeds tau; in-band
    # overrides are equally valid choices and only bounded loosely; overrides at
    # algebraic ties (tie_overrides: candidates equal to float64 rounding, where the
    # oracle's own summation order picks the position) are not bounded.
    if res["out_of_band"] > max(2, 1e-5 * res["cells"]):
        bad.append(("out_of_band", res["out_of_band"], res["out_of_band_by"]))
    if res["overrides"] > override_frac * res["cells"]:  # overrides < 1e-4 of the cells
        bad.append(("overrides", res["overrides"], res["cells"]))
    if "grad_maxscaled" in res:
        for k, v in res["grad_maxscaled"].items():
            if v > grad_tol:
                bad.append(("grad_maxscaled", k, v))
        for k, v in res["grad_normwise"].items():
            if v > grad_tol:
                bad.append(("grad_normwise", k, v))
    if "param_normwise" in res:
        for key in ("param_normwise", "m_normwise", "v_normwise"):
            for k, v in res[key].items():
                if v > param_tol:
                    bad.append((key, k, v))
        if res["adam_step_bound_violations"]:
            bad.append(("adam_step_bound_violations", res["adam_step_bound_violations"]))
        if res["step"][0] != res["step"][1]:
            bad.append(("adam step counter", res["step"]))
    assert not bad, bad


def generate(preset, n, seed):
    return molgen.generate(preset, n, seed)
