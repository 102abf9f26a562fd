"""Pin the CPU oracle to the reference's own outputs (golden fixtures made by
tests/golden/make_golden.py from fedsim 0.1.0), before trusting it as the
checker of the GPU path."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import port
from tests.helpers import CONFIGS, golden_rows, oracle_model, oracle_run, product_datasets, users_of


@pytest.mark.parametrize("name", ["mlp_dp", "logistic_dp", "mlp_noclip", "cnn_dp", "mlp_adam_dp", "logistic_fedprox",
                                  "mlp_adafedprox", "mlp_scaffold_dp", "logistic_scaffold", "cnn_scaffold"])
def test_oracle_reproduces_reference_run(name, golden):
    g = golden(name)
    cfg = CONFIGS[name]
    thetas, rows, digest = oracle_run(cfg)
    assert digest == str(g["digest"])  # cohorts bit-exact
    keep = g["keep"] if "keep" in g else slice(None)
    np.testing.assert_allclose(thetas[:, keep], g["thetas"], rtol=1e-9, atol=1e-12)
    ref_rows = golden_rows(g)
    assert [r[:3] for r in rows] == [r[:3] for r in ref_rows]
    np.testing.assert_allclose([r[3] for r in rows], [r[3] for r in ref_rows], rtol=1e-9)
    np.testing.assert_allclose([r[4] for r in rows], [r[4] for r in ref_rows], rtol=1e-12)


@pytest.mark.parametrize("name", ["mlp_dp", "logistic_dp", "cnn_dp"])
def test_oracle_iteration0_deltas(name, golden):
    g = golden(name)
    cfg = CONFIGS[name]
    ds = product_datasets(cfg)
    users = users_of(ds[next(iter(ds))])
    model = oracle_model(cfg)
    theta = model.init(cfg["init_seed"])
    ctx = port.cohort_seed(cfg["run_seed"], 0, "train")
    cohort = port.sample_cohort(tuple(users), cfg["cohort"], ctx)
    assert list(cohort) == [str(u) for u in g["cohort0"]]
    keep = g["keep"] if "keep" in g else slice(None)
    for i, uid in enumerate(cohort):
        X, y = users[uid]
        after = port.fit_local(model, theta, X, y, port.user_perms(ctx, uid, X.shape[0], cfg["epochs"]),
                               cfg["lr"], cfg["batch"])
        d = port.flat(theta, model.dims) - port.flat(after, model.dims)
        np.testing.assert_allclose(d[keep], g["deltas0"][i], rtol=1e-9, atol=1e-14)
        if "deltas0_l2" in g:
            np.testing.assert_allclose(np.linalg.norm(d), g["deltas0_l2"][i], rtol=1e-9)


def test_oracle_queues_match_reference(golden):
    g = golden("logistic_dp")
    cfg = CONFIGS["logistic_dp"]
    ds = product_datasets(cfg)
    users = users_of(ds[next(iter(ds))])
    w = {u: float(users[u][0].shape[0]) for u in g["cohort0"]}
    queues, _ = port.lpt_queues(w, cfg["workers"], port.lower_median(list(w.values())))
    assert ["|".join(q) for q in queues] == [str(q) for q in g["queues0"]]


def test_cnn_oracle_gradient_matches_autograd():
    """The reference pins gradients by finite differences (tests/test_models.py:27-63);
    the ReLU/max-pool CNN has kinks in nearly every coordinate direction, so
    the CNN oracle is pinned against float64 autograd of the same network
    (torch on CPU, test-only) instead, plus one smooth directional check."""
    import torch
    import torch.nn.functional as F

    m = port.Cnn()
    rng = np.random.default_rng(0)
    p = m.init(3)
    X = rng.normal(size=(4, 3072))
    y = np.array([1, 7, 7, 0])
    loss, g = m.loss_and_grad(p, X, y)
    t = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in p.items()}
    x = torch.tensor(X).reshape(4, 3, 32, 32)
    a1 = F.relu(F.conv2d(x, t["conv1/weights"].reshape(32, 3, 3, 3), t["conv1/bias"]))
    a2 = F.relu(F.conv2d(a1, t["conv2/weights"].reshape(64, 32, 3, 3), t["conv2/bias"]))
    flat = F.max_pool2d(a2, 2).reshape(4, -1)
    a3 = F.relu(flat @ t["fc1/weights"].reshape(12544, 128) + t["fc1/bias"])
    logits = a3 @ t["fc2/weights"].reshape(128, 10) + t["fc2/bias"]
    ref = F.cross_entropy(logits, torch.tensor(y))
    ref.backward()
    assert abs(loss - ref.item()) <= 1e-12 * abs(ref.item())
    for name in m.dims:
        np.testing.assert_allclose(g[name], t[name].grad.numpy(), rtol=1e-9, atol=1e-15, err_msg=name)


def test_cnn_eval_counts_consistent_with_loss():
    m = port.Cnn()
    rng = np.random.default_rng(1)
    p = m.init(0)
    X = rng.normal(size=(5, 3072))
    y = rng.integers(0, 10, 5)
    loss_mean, _ = m.loss_and_grad(p, X, y)
    loss_sum, correct = m.eval_counts(p, X, y)
    assert np.isclose(loss_sum, 5 * loss_mean, rtol=1e-12)
    assert 0 <= correct <= 5
