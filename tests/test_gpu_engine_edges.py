"""Engine / loop edge cases of the reference (tests/test_engine.py:331-535 in
fedsim), replayed on GpuSimulationEngine with the sm_100a kernels: eval-only
contexts, empty Poisson cohorts, zero iterations, early stop, bitwise
reproducible reruns, digests tracking the seed, zero local epochs, one-point
users, missing populations."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2404_06430_b200 as fb
from tests.helpers import CONFIGS, product_datasets, product_run_parts, run_sim

pytestmark = pytest.mark.gpu


def _alg(cfg, **over):
    cfg = {**cfg, **over}
    alg, post = product_run_parts(cfg)
    return cfg, alg, post


def _run(cfg, alg, post, callbacks=(), **engine_kw):
    eng = fb.GpuSimulationEngine(product_datasets(cfg), postprocessors=post, **engine_kw)
    thetas = []
    res = run_sim(alg, eng, callbacks=[lambda p, rows, t: thetas.append(p.flat_host()) and False,
                                                 *callbacks])
    return res, np.array(thetas)


def test_eval_only_context_yields_metrics_without_aggregate():
    cfg, alg, post = _alg(CONFIGS["mlp_dp"])
    eng = fb.GpuSimulationEngine(product_datasets(cfg), postprocessors=post)
    state = alg.initial_state()
    val = alg.get_next_central_contexts(state, 0)[1]  # iteration 0 has a val context
    assert not val.do_training
    res = eng.run_iteration(alg, state, (val,))
    assert res.aggregates == (None,)
    m = res.metrics
    assert set(name for _, name in m) == {"accuracy", "loss", "per_user_accuracy"}
    assert m[("val", "loss")].denominator == cfg["eval_cohort"] * cfg["ppu"]


def test_empty_poisson_cohort_produces_no_aggregate_and_keeps_theta():
    cfg, alg, post = _alg(CONFIGS["mlp_dp"], iterations=1)
    eng = fb.GpuSimulationEngine(product_datasets(cfg), postprocessors=post, cohort_mode="poisson",
                                 poisson_rate=1e-12)
    state = alg.initial_state()
    theta0 = fb.DeviceParams.from_host(state.params, eng.device).flat_host()
    ctxs = alg.get_next_central_contexts(state, 0)
    res = eng.run_iteration(alg, state, ctxs)
    assert res.aggregates[0] is None and res.metrics == {}
    assert res.cohorts[0] == ("train", ())
    state = alg.process_aggregated_statistics_all_contexts(state, ctxs, res.aggregates, res.metrics, [])
    np.testing.assert_array_equal(state.params.flat_host(), theta0)


def _run_fedsim_loop(cfg, alg, post, callbacks=()):
    """fedsim's own run_simulation (fedsim/engine/loop.py:45-88) driving the engine."""
    from tests.fedsim_ref import fedsim

    fedsim()
    from fedsim.engine import run_simulation

    eng = fb.GpuSimulationEngine(product_datasets(cfg), postprocessors=post)
    thetas = []
    res = run_simulation(alg, eng, callbacks=[lambda p, rows, t: thetas.append(p.flat_host()) and False,
                                              *callbacks])
    return res, np.array(thetas)


def test_zero_iterations_returns_initial_state():
    cfg, alg, post = _alg(CONFIGS["mlp_dp"], iterations=0)
    res, thetas = _run_fedsim_loop(cfg, alg, post)
    assert res.iterations_run == 0 and res.metrics_rows == [] and res.iteration_seconds == []
    assert len(thetas) == 0


def test_early_stop_callback_runs_exactly_six_iterations():
    cfg, alg, post = _alg(CONFIGS["logistic_dp"], iterations=1500)
    res, _ = _run_fedsim_loop(cfg, alg, post, callbacks=[lambda p, rows, t: t == 5])
    assert res.iterations_run == 6 and len(res.iteration_seconds) == 6
    assert {row[0] for row in res.metrics_rows} == set(range(6))


@pytest.mark.parametrize("noise_source", ["numpy", "philox"])
def test_reruns_are_bitwise_reproducible_and_rows_sorted(noise_source):
    cfg = CONFIGS["mlp_dp"]
    runs = []
    for _ in range(2):
        alg, post = product_run_parts(cfg, noise_source=noise_source)
        runs.append(_run(cfg, alg, post))
    (a, ta), (b, tb) = runs
    assert a.metrics_rows == b.metrics_rows and a.cohort_digest == b.cohort_digest
    np.testing.assert_array_equal(ta, tb)
    per_it = {}
    for row in a.metrics_rows:
        per_it.setdefault(row[0], []).append((row[1], row[2]))
    for names in per_it.values():
        assert names == sorted(names)


def test_cohort_digest_tracks_sampling_seed():
    cfg = CONFIGS["logistic_dp"]
    d = []
    for seed in (1, 2):
        c, alg, post = _alg(cfg, run_seed=seed, iterations=2)
        d.append(_run(c, alg, post)[0].cohort_digest)
    assert d[0] != d[1]


def test_zero_local_epochs_leaves_theta_unchanged_without_noise():
    """local_train_sgd with zero epochs returns a copy (fedsim/models/models.py:250-251):
    every delta is zero, so the central step with sigma = 0 keeps theta."""
    cfg, alg, post = _alg(CONFIGS["mlp_dp"], epochs=0, sigma=0.0, iterations=2)
    res, thetas = _run(cfg, alg, post)
    theta0 = np.concatenate([v.ravel() for v in alg.model.init_params(cfg["init_seed"]).values()])
    np.testing.assert_allclose(thetas[-1], theta0, rtol=0, atol=1e-7)
    assert any(r[2] == "update_norm" and r[3] == 0.0 for r in res.metrics_rows)


@pytest.mark.parametrize("model", ["mlp", "cnn"])
def test_one_point_users_and_tail_batches_match_oracle(model):
    """Users of 1..B+1 points: single-row and partial tail batches (tests/test_models.py:137-149)."""
    import torch

    from oracle import port
    from tests.conftest import assert_close_fp32

    rng = np.random.default_rng(7)
    sizes = [1, 2, 1, 11, 3] if model == "mlp" else [1, 4, 1]
    dim = 3072 if model == "cnn" else 8
    users = {}
    for i, n in enumerate(sizes):
        uid = f"u{i:03d}"
        users[uid] = fb.UserDataset(uid, rng.normal(size=(n, dim)), rng.integers(0, 4, size=n).astype(np.int64))
    ds = fb.FederatedDataset(users=users, population=fb.Population.TRAIN)
    m = fb.MLP(dim, 16, 4) if model == "mlp" else fb.CNN()
    om = port.Mlp(dim, 16, 4) if model == "mlp" else port.Cnn()
    alg = fb.FedAvg(m, fb.SGDOptimizer(1.0), total_iterations=1, cohort_size=len(sizes), local_learning_rate=0.1,
                    local_num_epochs=2, local_batch_size=2, eval_frequency=10, eval_cohort_size=1,
                    weighting="datapoints", run_seed=3, init_seed=4)
    eng = fb.GpuSimulationEngine({fb.Population.TRAIN: ds, fb.Population.VAL: ds})
    res = run_sim(alg, eng)
    theta0 = om.init(4)
    ref = port.run_context(om, theta0, {u.user_id: (u.features.astype(np.float32).astype(np.float64), u.labels)
                                        for u in ds.users.values()}, len(sizes),
                           port.cohort_seed(3, 0, "train"), train=(0.1, 2, 2), weighting="datapoints")
    want = port.central_sgd(port.flat(theta0, om.dims), ref.aggregate, ref.weight, 1.0)
    got = res.params.flat_host()
    if model == "mlp":
        assert_close_fp32(got, want)
    else:  # CNN: ReLU / max-pool decision flips at fp32 resolution are possible (test_gpu_cnn.py)
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5


def test_missing_population_dataset_is_engine_error():
    cfg, alg, post = _alg(CONFIGS["mlp_dp"])
    ds = product_datasets(cfg)
    eng = fb.GpuSimulationEngine({fb.Population.TRAIN: ds[fb.Population.TRAIN]}, postprocessors=post)
    state = alg.initial_state()
    with pytest.raises(fb.EngineError, match="no dataset for population 'val'"):
        eng.run_iteration(alg, state, alg.get_next_central_contexts(state, 0))
