"""Pins of the oracle's evaluation path."""
import numpy as np
import pytest

import molgen
import oracle as O


def test_perfect_predictor_has_zero_error():
    y = np.array([1.5, -2.0, 0.25])
    m = O.regression_metrics(y, y)
    assert m["mae"] == 0.0 and m["mse"] == 0.0 and m["count"] == 3


def test_constant_mean_predictor_mae_is_mean_absolute_deviation():
    # SPEC.md:389 "constant predictor at mean(y) -> MAE = mean absolute deviation of y"
    y = np.array([1.0, 2.0, 4.0, 9.0])  # mean 4: deviations 3, 2, 0, 5
    m = O.regression_metrics(np.full(4, 4.0), y)
    assert m["mae"] == pytest.approx(10.0 / 4, abs=0)
    assert m["mse"] == pytest.approx((9 + 4 + 0 + 25) / 4, abs=0)


def test_mae_bounded_by_rmse_jensen():
    rng = np.random.default_rng(5)
    for _ in range(20):
        y, yh = rng.normal(size=50), rng.normal(size=50) * rng.uniform(0.1, 3)
        m = O.regression_metrics(yh, y)
        assert m["mae"] <= np.sqrt(m["mse"]) + 1e-15


def test_evaluate_matches_forward_and_is_batch_order_independent():
    data = molgen.generate("tiny", 60, 11)
    cfg = {"f_node": data["f_node"], "f_edge": 4, "hidden": 16, "layers": 2, "fc_hidden": 16}
    params = O.init_params(cfg, 3)
    delta = O.degree_stat(data)
    b1, b2 = list(range(0, 20)), list(range(20, 45))
    ev = O.evaluate(params, data, [b1, b2], cfg, delta)
    # the pairs are the forward's predictions, graph by graph
    _, yh1, _ = O.forward(params, O.pack(data, b1), cfg, delta)
    _, yh2, _ = O.forward(params, O.pack(data, b2), cfg, delta)
    np.testing.assert_array_equal(ev["pairs"][:, 1], np.concatenate([yh1, yh2]))
    np.testing.assert_array_equal(ev["pairs"][:, 0], np.asarray(data["y"], np.float64)[b1 + b2])
    # metrics do not depend on how the graphs are batched (SPEC.md batch independence)
    ev2 = O.evaluate(params, data, [b1 + b2], cfg, delta)
    assert ev2["mse"] == pytest.approx(ev["mse"], rel=1e-12)
    assert ev2["mae"] == pytest.approx(ev["mae"], rel=1e-12)
    # and the MSE equals the training loss definition on the same batch
    loss, _, _ = O.forward(params, O.pack(data, b1 + b2), cfg, delta)
    assert ev2["mse"] == pytest.approx(loss, rel=1e-12)
