"""End-to-end parity: GpuSimulationEngine (sm_100a kernels through the C ABI)
against the reference's own runs (golden fixtures) and the oracle.

Gate (north_star): cohorts bit-exact (digest), post-iteration model within
rtol 1e-5 with atol 1e-6 * max|ref| (fp32 vs the float64 reference), the
reference's noise vector injected (noise_source="numpy")."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2404_06430_b200 as fb
from tests.conftest import assert_close_fp32
from tests.helpers import CONFIGS, golden_rows, oracle_run, product_datasets, product_run_parts, run_sim

pytestmark = pytest.mark.gpu


def run_engine(cfg, noise_source="numpy", **engine_kw):
    ds = product_datasets(cfg)
    alg, post = product_run_parts(cfg, noise_source=noise_source)
    eng = fb.GpuSimulationEngine(ds, postprocessors=post, **engine_kw)
    thetas = []
    res = run_sim(alg, eng, callbacks=[lambda p, rows, t: thetas.append(p.flat_host()) and False])
    return res, np.array(thetas)


@pytest.mark.parametrize("name", ["mlp_dp", "logistic_dp", "mlp_noclip", "mlp_adam_dp", "logistic_fedprox",
                                  "mlp_adafedprox", "mlp_scaffold_dp", "logistic_scaffold"])
def test_engine_matches_reference_run(name, golden):
    g = golden(name)
    res, thetas = run_engine(CONFIGS[name])
    assert res.cohort_digest == str(g["digest"])
    for t in range(len(thetas)):
        assert_close_fp32(thetas[t], g["thetas"][t], what=f"{name} theta after iteration {t}")
    got, ref = res.metrics_rows, golden_rows(g)
    assert [r[:3] for r in got] == [r[:3] for r in ref]
    np.testing.assert_allclose([r[3] for r in got], [r[3] for r in ref], rtol=2e-5)
    np.testing.assert_allclose([r[4] for r in got], [r[4] for r in ref], rtol=1e-12)


def test_engine_clip_factors_match_oracle():
    """Per-client clip factors / norms of iteration 0 (rtol 1e-5)."""
    from oracle import port
    from tests.helpers import oracle_model, users_of

    cfg = CONFIGS["mlp_dp"]
    ds = product_datasets(cfg)
    alg, post = product_run_parts(cfg, sigma=0.0)
    eng = fb.GpuSimulationEngine(ds, postprocessors=post)
    state = alg.initial_state()
    state.params = fb.DeviceParams.from_host(state.params, eng.device)
    ctx = alg.get_next_central_contexts(state, 0)[0]
    agg, metrics, cohort, _ = eng._run_context(alg, state, ctx)
    m = oracle_model(cfg)
    ref = port.run_context(m, m.init(cfg["init_seed"]), users_of(ds[fb.Population.TRAIN]), cfg["cohort"],
                           ctx.seed, train=(cfg["lr"], cfg["epochs"], cfg["batch"]), weighting=cfg["weighting"],
                           bound=cfg["bound"], sigma=0.0)
    assert metrics["clip_fraction"].numerator == float(ref.clipped.sum())
    np.testing.assert_allclose(metrics["update_norm"].numerator, ref.norm.sum(), rtol=1e-5)
    host = agg.to_host()
    assert_close_fp32(np.concatenate([host.entries[n] for n in m.dims]), ref.aggregate)


def test_engine_two_rank_shard_map_matches_single_rank():
    """world_size semantics on one device: rank r's LPT queue (reference
    num_workers = 2) -- the union of the two ranks' queues is the cohort."""
    cfg = CONFIGS["logistic_dp"]
    ds = product_datasets(cfg)
    train = ds[fb.Population.TRAIN]
    ctx_seed = fb.cohort_seed(cfg["run_seed"], 0, "train")
    cohort = fb.sample_cohort(train, cfg["cohort"], ctx_seed)
    w = {u: train.users[u].weight for u in cohort}
    q = fb.schedule_users(w, 2, fb.compute_base_weight(list(w.values()), "median")).queues
    assert sorted(q[0] + q[1]) == sorted(cohort)


def test_engine_oracle_sigma_zero_long_run():
    """No noise: 2 iterations of the 50-user MLP config vs the oracle."""
    cfg = dict(CONFIGS["mlp_noclip"])
    thetas_ref, rows_ref, digest_ref = oracle_run(cfg)
    res, thetas = run_engine(cfg)
    assert res.cohort_digest == digest_ref
    for t in range(len(thetas)):
        assert_close_fp32(thetas[t], thetas_ref[t])


def test_engine_nonfinite_update_raises_with_provenance():
    cfg = dict(CONFIGS["mlp_noclip"], lr=1e30, iterations=1)
    with pytest.raises(fb.EngineError, match=r"iteration 0, population 'train', user 'train\d{5}'"):
        run_engine(cfg)


def test_engine_philox_noise_statistics():
    """Device noise: mean and std within 3 sigma of N(0, (r sigma S)^2)
    (tests/test_privacy.py:134-141 analogue, north_star "within 3 sigma")."""
    cfg = dict(CONFIGS["mlp_dp"], iterations=1)
    ds = product_datasets(cfg)
    alg, post = product_run_parts(cfg, noise_source="philox")
    eng = fb.GpuSimulationEngine(ds, postprocessors=post)
    state = alg.initial_state()
    res = eng.run_iteration(alg, state, alg.get_next_central_contexts(state, 0))
    agg = res.aggregates[0]
    clean = agg.flat.double().cpu().numpy()
    noised = agg.materialize().double().cpu().numpy()
    z = noised - clean
    std = post[1].noise_std()
    n = z.size
    assert abs(z.mean()) <= 3 * std / np.sqrt(n)
    assert abs(z.std() - std) <= 3 * std / np.sqrt(2 * n) + 1e-7


def test_scaffold_controls_match_oracle():
    """Per-user control vectors and the server control after a Scaffold run
    (device store) against the oracle's float64 restatement."""
    from oracle import port
    from tests.helpers import oracle_model, users_of

    cfg = CONFIGS["logistic_scaffold"]
    ds = product_datasets(cfg)
    alg, post = product_run_parts(cfg)
    eng = fb.GpuSimulationEngine(ds, postprocessors=post)
    res = run_sim(alg, eng)
    store = res.state.extra["user_controls"]
    # replay the oracle and capture its controls
    model = oracle_model(cfg)
    scaffold = dict(server=np.zeros(sum(model.dims.values())), users={})
    theta = model.init(cfg["init_seed"])
    for t in range(cfg["iterations"]):
        r = port.run_context(model, theta, users_of(ds[fb.Population.TRAIN]), cfg["cohort"],
                             port.cohort_seed(cfg["run_seed"], t, "train"), train=(cfg["lr"], cfg["epochs"], cfg["batch"]),
                             weighting="uniform", scaffold=scaffold)
        for uid, c in r.user_updates:
            scaffold["users"][uid] = c
        D = r.aggregate.size // 2
        new = port.central_sgd(port.flat(theta, model.dims), r.aggregate[:D], r.weight, cfg["clr"])
        scaffold["server"] = scaffold["server"] + (r.weight / cfg["algorithm"]["num_train_users"]) * (
            r.aggregate[D:] / r.weight)
        theta = port._unflat(new, model.dims)
    assert len(store) == len(scaffold["users"])
    for uid, ref in scaffold["users"].items():
        assert_close_fp32(store.get(uid), ref, what=f"control of {uid}")
    assert_close_fp32(res.state.extra["server_control"].double().cpu().numpy(), scaffold["server"],
                      what="server control")


def test_scaffold_zero_local_steps_raises_with_provenance():
    cfg = dict(CONFIGS["logistic_scaffold"])
    ds = product_datasets(cfg)
    alg, post = product_run_parts({**cfg, "lr": 0.0})
    eng = fb.GpuSimulationEngine(ds, postprocessors=post)
    with pytest.raises(fb.EngineError, match="control update divides by steps"):
        run_sim(alg, eng)


def test_engine_metrics_csv_and_checkpoint(golden, tmp_path):
    """The GPU run writes the reference's metrics CSV / checkpoint formats:
    rows equal the reference run's (values rtol 2e-5), the checkpoint holds
    the final device theta exactly."""
    import io

    cfg = CONFIGS["mlp_dp"]
    g = golden("mlp_dp")
    ds = product_datasets(cfg)
    alg, post = product_run_parts(cfg)
    buf = io.StringIO()
    res = run_sim(alg, fb.GpuSimulationEngine(ds, postprocessors=post), callbacks=[fb.CsvMetricsWriter(buf)])
    lines = buf.getvalue().splitlines()
    assert lines[0] == "iteration,population,metric,value,weight"
    got = [ln.split(",") for ln in lines[1:]]
    ref = golden_rows(g)
    assert [(int(a), b, c) for a, b, c, _, _ in got] == [r[:3] for r in ref]
    np.testing.assert_allclose([float(r[3]) for r in got], [r[3] for r in ref], rtol=2e-5)
    fb.save_params(res.params, tmp_path / "checkpoint.csv")
    back = fb.load_params(tmp_path / "checkpoint.csv")
    np.testing.assert_array_equal(np.concatenate([back[n] for n in back]), res.params.flat_host())


@pytest.mark.parametrize("prefetch,max_runs", [(False, 64), (True, 64), (True, 0)],
                         ids=["sync-gather", "prefetch-dma", "prefetch-gather-kernel"])
def test_host_resident_dataset_matches_reference_run(golden, prefetch, max_runs, monkeypatch):
    """data_residency="host": cohort rows gathered from pinned host memory each
    context (synchronously, or for iteration t+1 on a copy stream during t, by
    copy-engine runs in host order or by the gather kernel): identical results
    to the device-resident run and the reference."""
    from paper_2404_06430_b200 import engine

    monkeypatch.setattr(engine, "PREFETCH_MAX_RUNS", max_runs)
    g = golden("mlp_dp")
    res, thetas = run_engine(CONFIGS["mlp_dp"], data_residency="host", prefetch=prefetch)
    assert res.cohort_digest == str(g["digest"])
    for t in range(len(thetas)):
        assert_close_fp32(thetas[t], g["thetas"][t], what=f"theta after iteration {t}")
    _, dev_thetas = run_engine(CONFIGS["mlp_dp"])
    np.testing.assert_array_equal(thetas, dev_thetas)