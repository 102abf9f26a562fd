"""Host side of the product (no GPU): bit-exact sampling, LPT shard map,
seeds, data generators, contexts, metrics and the server postprocessors,
checked against the reference's golden vectors."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2404_06430_b200 as fb
from paper_2404_06430_b200 import privacy
from tests.helpers import CONFIGS, product_datasets


def _ids(n):
    return {f"u{i:05d}": fb.UserDataset(f"u{i:05d}", np.zeros((1, 1)), np.zeros(1, dtype=np.int64)) for i in range(n)}


@pytest.mark.parametrize("N,C,seed", [(1000, 50, 7), (1000, 1000, 8), (20000, 100, 9), (20000, 1000, 10), (30, 30, 11)])
def test_sample_cohort_bit_exact(golden, N, C, seed):
    ds = fb.FederatedDataset(users=_ids(N), population=fb.Population.TRAIN)
    assert list(fb.sample_cohort(ds, C, seed)) == [str(u) for u in golden("sampling")[f"cohort_{N}_{C}_{seed}"]]


@pytest.mark.parametrize("m", [1, 2, 3, 8])
def test_schedule_users_bit_exact(golden, m):
    g = golden("sampling")
    weights = {f"c{i:04d}": float(s) for i, s in enumerate(g["sched_sizes"])}
    base = fb.compute_base_weight(list(weights.values()), "median")
    got = ["|".join(q) for q in fb.schedule_users(weights, m, base).queues]
    assert got == [str(q) for q in g[f"queues_m{m}"]]


def test_permutations_and_seeds_bit_exact(golden):
    g = golden("sampling")
    for i in range(50):
        ctx = fb.derive_seed(1, "cohort", i, "train")
        (got,) = fb.client_permutations(ctx, [f"train{i:05d}"], [50], 2)
        np.testing.assert_array_equal(got, g["perms"][i])
    seeds = [fb.derive_seed(0, "pool"), fb.user_seed(7, "train00042"), fb.cohort_seed(0, 3, "val"),
             fb.derive_seed(0, "noise-stream", 0)]
    assert seeds == [int(s) for s in g["seeds"]]


def test_datasets_regenerate_reference_cohorts(golden):
    """The product's data generators replay the reference's draws: the first
    cohort of every fixture config is reproduced exactly."""
    for name, cfg in CONFIGS.items():
        ds = product_datasets(cfg)
        ctx = fb.cohort_seed(cfg["run_seed"], 0, "train")
        got = fb.sample_cohort(ds[fb.Population.TRAIN], cfg["cohort"], ctx)
        assert list(got) == [str(u) for u in golden(name)["cohort0"]], name


def test_contexts_follow_fedavg_schedule():
    alg = fb.FedAvg(fb.MLP(4, 3, 2), fb.SGDOptimizer(1.0), total_iterations=3, cohort_size=2,
                    local_learning_rate=fb.HyperParam(0.4, fb.LinearWarmup(2)), local_num_epochs=1,
                    local_batch_size=2, eval_frequency=2, eval_cohort_size=1)
    st = alg.initial_state()
    c0 = alg.get_next_central_contexts(st, 0)
    assert [c.population for c in c0] == [fb.Population.TRAIN, fb.Population.VAL]
    assert c0[0].local_params.learning_rate == pytest.approx(0.2)
    assert len(alg.get_next_central_contexts(st, 1)) == 1
    assert alg.get_next_central_contexts(st, 3) == ()
    with pytest.raises(NotImplementedError):
        alg.simulate_one_user(st, None, c0[0], 0)


def test_mlp_init_matches_reference_draw_order(golden):
    cfg = CONFIGS["mlp_dp"]
    m = fb.MLP(cfg["dim"], cfg["hidden"], cfg["classes"])
    p = m.init_params(cfg["init_seed"])
    np.testing.assert_array_equal(np.concatenate([p[n] for n in m.param_dims]), golden("mlp_dp")["theta0"])


def test_cnn_layout():
    m = fb.CNN()
    assert m.num_params == 1_626_442
    assert m.flat_dim == 12544
    assert m.forward_flops_per_sample() == 33_670_400  # 2 x 16,835,200 MACs
    p = m.init_params(1)
    assert list(p) == list(m.param_dims)
    assert np.abs(p["fc1/weights"]).max() <= 1 / np.sqrt(12544)


def test_clip_server_metrics_and_strip():
    """fedsim tests/test_engine.py:431-445 shape: [3,4] x 4 users at S=1."""
    clip = fb.ClippingPostprocessor(1.0)
    agg = fb.Statistics({"w": np.array([2.4, 3.2]), privacy.CLIPPED_KEY: np.array([4.0]),
                         privacy.COUNT_KEY: np.array([4.0]), privacy.NORM_KEY: np.array([20.0])}, 4.0)
    out, metrics = clip.postprocess_server(agg, None)
    assert out.names == ("w",)
    assert metrics["clip_fraction"].value == 1.0
    assert metrics["update_norm"].value == 5.0
    assert metrics["clipping_bound"].value == 1.0


def test_adaptive_clip_moves_bound_after_use():
    clip = fb.ClippingPostprocessor(1.0, adaptive=fb.AdaptiveClipConfig(quantile=0.5, learning_rate=0.2))
    agg = fb.Statistics({"w": np.zeros(2), privacy.CLIPPED_KEY: np.array([1.0]),
                         privacy.COUNT_KEY: np.array([1.0]), privacy.NORM_KEY: np.array([2.0])}, 1.0)
    _, metrics = clip.postprocess_server(agg, None)
    assert metrics["clipping_bound"].value == 1.0
    assert clip.current_bound == pytest.approx(np.exp(-0.2 * 0.5))


def test_validate_pipeline_and_mechanism_args():
    clip = fb.ClippingPostprocessor(0.4)
    mech = fb.GaussianCentralMechanism(clip, sigma=1.0, r=0.1, noise_base_seed=0)
    fb.validate_pipeline([clip, mech])
    with pytest.raises(fb.NotClippedUpstream):
        fb.validate_pipeline([mech, clip])
    with pytest.raises(ValueError):
        fb.GaussianCentralMechanism(fb.ClippingPostprocessor(1.0, norm_order=1.0), sigma=1.0, r=1.0,
                                    noise_base_seed=0)
    with pytest.raises(ValueError):
        fb.GaussianCentralMechanism(clip, sigma=-1.0, r=1.0, noise_base_seed=0)
    assert mech.noise_std() == pytest.approx(0.04)


def test_snr_unit_case():
    """fedsim tests/test_privacy.py:235-242: ||delta||=2, d=100, sigma=0.1 -> 2.0."""
    agg = fb.Statistics({"w": np.r_[2.0, np.zeros(99)]}, 1.0)
    assert fb.snr(agg, 0.1, 100) == pytest.approx(2.0)


def test_statistics_validation_and_algebra():
    with pytest.raises(ValueError):
        fb.Statistics.from_entries({"a": [np.nan]}, 1.0)
    with pytest.raises(ValueError):
        fb.Statistics.from_entries({"a": [1.0]}, 0.0)
    a = fb.weighted({"a": np.array([1.0, 2.0])}, 2.0)
    b = fb.weighted({"a": np.array([3.0, 4.0])}, 1.0)
    m = fb.average(fb.accumulate(a, b))
    np.testing.assert_allclose(m.entries["a"], [5 / 3, 8 / 3])
    with pytest.raises(fb.ZeroWeight):
        fb.average(fb.Statistics.zeros({"a": 2}))
    assert fb.global_norm(fb.Statistics({"a": np.array([3.0]), "b": np.array([4.0])}, 1.0)) == 5.0


def test_metric_values():
    a = fb.MetricValue.from_user(fb.MetricKind.PER_USER, 3, 4)
    assert (a.numerator, a.denominator) == (0.75, 1.0)
    with pytest.raises(fb.IncompatibleShapes):
        a + fb.MetricValue(fb.MetricKind.CENTRAL, 1.0, 1.0)
    assert fb.metric_aggregate([fb.MetricValue(fb.MetricKind.CENTRAL, 1.0, 2.0)] * 3) == 0.5


def test_engine_refuses_without_cuda():
    """No CPU fallback: constructing the engine without a device fails loudly."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    cfg = CONFIGS["mlp_dp"]
    with pytest.raises(fb.NativeUnavailable):
        fb.GpuSimulationEngine(product_datasets(cfg))


def test_native_permutations_bit_exact_with_numpy(golden):
    """fb_user_permutations (native SHA-256 + SeedSequence + PCG64 +
    permutation) == the reference's numpy draws, ragged sizes, 2 epochs."""
    from paper_2404_06430_b200 import native

    if not native.LIB_PATH.exists():
        pytest.skip("library not built")
    from paper_2404_06430_b200.engine import native_permutations

    g = golden("sampling")
    for i in range(50):
        ctx = fb.derive_seed(1, "cohort", i, "train")
        got = native_permutations(ctx, [f"train{i:05d}"], np.array([50]), 2, np.array([0]))
        np.testing.assert_array_equal(got, g["perms"][i])
    rng = np.random.default_rng(0)
    ids = [f"u{i}" for i in range(300)] + ["user with space", "ünïcode", "quote'd"]
    sizes = rng.integers(1, 200, size=len(ids))
    off = np.concatenate([[0], np.cumsum(sizes * 3)[:-1]])
    got = native_permutations(12345, ids, sizes, 3, off)
    want = np.concatenate(fb.client_permutations(12345, ids, sizes.tolist(), 3))
    np.testing.assert_array_equal(got, want)


def test_adam_host_step_matches_reference_analytic_first_step():
    """tests/test_models.py:197-215 of the reference: first step = -lr g / (|g| + eps);
    zero delta leaves the parameters unchanged."""
    lr, eps = 0.1, 0.3
    opt = fb.AdamOptimizer(learning_rate=lr, adaptivity_degree=eps)
    rng = np.random.default_rng(5)
    params = {"a": rng.normal(size=6)}
    g = rng.normal(size=6)
    out = opt.step(params, {"a": g}, iteration=0)
    np.testing.assert_allclose(out["a"], params["a"] - lr * g / (np.abs(g) + eps), rtol=1e-12)
    assert opt.step_count == 1
    z = fb.AdamOptimizer(0.1).step({"a": np.array([3.0, -1.0])}, {"a": np.zeros(2)}, 0)
    np.testing.assert_array_equal(z["a"], [3.0, -1.0])
    with pytest.raises(ValueError):
        fb.AdamOptimizer(0.1, beta1=1.0)
    with pytest.raises(ValueError):
        fb.AdamOptimizer(0.1, adaptivity_degree=0.0)


def test_adafedprox_mu_rule_and_scaffold_validation():
    assert fb.adafedprox_update_mu(0.5, 1.0, 0.9) == pytest.approx(0.45)
    assert fb.adafedprox_update_mu(0.95, 1.0, 1.1) == pytest.approx(1.0)  # capped
    assert fb.adafedprox_update_mu(1e-4, 1.0, 0.5) == pytest.approx(1e-4)  # floored
    assert fb.adafedprox_update_mu(0.3, 1.0, 1.0) == 0.3
    kw = dict(total_iterations=1, cohort_size=2, local_learning_rate=0.1, local_num_epochs=1, local_batch_size=2,
              eval_frequency=1, eval_cohort_size=1)
    with pytest.raises(ValueError, match="uniform"):
        fb.Scaffold(fb.MLP(4, 3, 2), fb.SGDOptimizer(1.0), num_train_users=3, weighting="datapoints", **kw)
    with pytest.raises(ValueError, match="num_train_users"):
        fb.Scaffold(fb.MLP(4, 3, 2), fb.SGDOptimizer(1.0), num_train_users=0, **kw)
    alg = fb.Scaffold(fb.MLP(4, 3, 2), fb.SGDOptimizer(1.0), num_train_users=3, **kw)
    st = alg.initial_state()
    ctx = alg.get_next_central_contexts(st, 0)[0]
    plan = alg.cohort_plan(st, ctx)
    assert plan.scaffold and plan.weighting == "uniform"


def test_checkpoint_roundtrip_and_metrics_csv(tmp_path):
    """fedsim/models/checkpoint.py layout (lossless) and the runner's metrics
    CSV rows (fedsim/cli/runner.py:39-57)."""
    import io

    rng = np.random.default_rng(0)
    p = {"layer1/weights": rng.normal(size=7), "layer1/bias": np.array([0.1, -2.5e-300, 3.0])}
    path = tmp_path / "checkpoint.csv"
    fb.save_params(p, path)
    lines = path.read_text().splitlines()
    assert lines[:2] == ["fedsim-params,1", "name,index,value"]
    assert lines[2].startswith("layer1/weights,0,")
    back = fb.load_params(path)
    assert list(back) == list(p)
    for n in p:
        np.testing.assert_array_equal(back[n], p[n])
    with pytest.raises(fb.DataError):
        fb.load_params(tmp_path / "missing.csv")
    buf = io.StringIO()
    w = fb.CsvMetricsWriter(buf)
    assert w(None, [(0, "train", "loss", 0.5, 12.0), (0, "val", "accuracy", 1 / 3, 6.0)], 0) is False
    assert buf.getvalue().splitlines() == ["iteration,population,metric,value,weight", "0,train,loss,0.5,12.0",
                                           f"0,val,accuracy,{1 / 3!r},6.0"]