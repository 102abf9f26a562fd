"""Build the golden-fixture configurations with the product (host mirror)
and with the oracle, from tests/golden/configs.py."""

from __future__ import annotations

import numpy as np

import paper_2404_06430_b200 as fb
from oracle import port
from tests.golden.configs import CONFIGS


def product_datasets(cfg):
    ppu = cfg["ppu"]
    ntr, nva = cfg["users"] * ppu, cfg["val_users"] * ppu
    X, y = fb.make_synthetic_classification(ntr + nva, dim=cfg["dim"], num_classes=cfg["classes"],
                                            margin=cfg["margin"], seed=fb.derive_seed(cfg["data_seed"], "pool"))
    train = fb.partition_iid(X[:ntr], y[:ntr], ppu, seed=fb.derive_seed(cfg["data_seed"], "train", "split"),
                             population=fb.Population.TRAIN, id_prefix="train")
    val = fb.partition_iid(X[ntr:], y[ntr:], ppu, seed=fb.derive_seed(cfg["data_seed"], "val", "split"),
                           population=fb.Population.VAL, id_prefix="val")
    return {fb.Population.TRAIN: train, fb.Population.VAL: val}


def product_model(cfg):
    if cfg["model"] == "mlp":
        return fb.MLP(cfg["dim"], cfg["hidden"], cfg["classes"])
    if cfg["model"] == "logistic":
        return fb.LogisticRegression(cfg["dim"], cfg["classes"])
    return fb.CNN()


def oracle_model(cfg):
    if cfg["model"] == "mlp":
        return port.Mlp(cfg["dim"], cfg["hidden"], cfg["classes"])
    if cfg["model"] == "logistic":
        return port.Linear(cfg["dim"], cfg["classes"])
    return port.Cnn()


def noise_base(cfg) -> int:
    return fb.derive_seed(cfg["run_seed"], "noise-stream", cfg["noise_seed"])


def product_algorithm(cfg):
    """The configured algorithm / central optimizer, built with the mirror API
    (the same classes and arguments make_golden.py hands to the reference)."""
    o = cfg.get("optimizer", dict(kind="sgd"))
    opt = (fb.AdamOptimizer(o["lr"], beta1=o["beta1"], beta2=o["beta2"], adaptivity_degree=o["eps"])
           if o["kind"] == "adam" else fb.SGDOptimizer(cfg["clr"]))
    a = cfg.get("algorithm", dict(kind="fedavg"))
    kw = dict(total_iterations=cfg["iterations"], cohort_size=cfg["cohort"], local_learning_rate=cfg["lr"],
              local_num_epochs=cfg["epochs"], local_batch_size=cfg["batch"], eval_frequency=cfg["eval_every"],
              eval_cohort_size=cfg["eval_cohort"], weighting=cfg["weighting"], run_seed=cfg["run_seed"],
              init_seed=cfg["init_seed"])
    if a["kind"] == "fedprox":
        return fb.FedProx(product_model(cfg), opt, mu=a["mu"], **kw)
    if a["kind"] == "adafedprox":
        return fb.AdaFedProx(product_model(cfg), opt, mu=a["mu"], **kw)
    if a["kind"] == "scaffold":
        return fb.Scaffold(product_model(cfg), opt, num_train_users=a["num_train_users"], **kw)
    return fb.FedAvg(product_model(cfg), opt, **kw)


def product_run_parts(cfg, noise_source="numpy", sigma=None):
    """(algorithm, postprocessors) built with the product's mirror API."""
    alg = product_algorithm(cfg)
    post = []
    if cfg["bound"] is not None:
        clip = fb.ClippingPostprocessor(cfg["bound"])
        post = [clip, fb.GaussianCentralMechanism(clip, sigma=cfg["sigma"] if sigma is None else sigma,
                                                  r=cfg["r"], noise_base_seed=noise_base(cfg),
                                                  noise_source=noise_source)]
    return alg, post


def users_of(ds) -> dict:
    return {u.user_id: (u.features, u.labels) for u in ds.users.values()}


def oracle_run(cfg, world=None):
    ds = product_datasets(cfg)
    return port.run_fedavg(
        oracle_model(cfg), users_of(ds[fb.Population.TRAIN]), users_of(ds[fb.Population.VAL]),
        iterations=cfg["iterations"], cohort=cfg["cohort"], eval_cohort=cfg["eval_cohort"],
        eval_every=cfg["eval_every"], lr=cfg["lr"], epochs=cfg["epochs"], batch=cfg["batch"], clr=cfg["clr"],
        weighting=cfg["weighting"], bound=cfg["bound"], sigma=cfg["sigma"], r=cfg["r"],
        noise_base=noise_base(cfg), run_seed=cfg["run_seed"], init_seed=cfg["init_seed"],
        world=cfg["workers"] if world is None else world, algorithm=cfg.get("algorithm"),
        optimizer=cfg.get("optimizer"))


def golden_rows(g):
    return [(int(t), str(p), str(n), float(v), float(w))
            for t, p, n, v, w in zip(g["row_t"], g["row_pop"], g["row_name"], g["row_value"], g["row_weight"])]


__all__ = ["run_sim", "CONFIGS", "product_datasets", "product_model", "product_algorithm", "oracle_model", "product_run_parts", "oracle_run",
           "golden_rows", "users_of", "noise_base"]


def run_sim(algorithm, engine, callbacks=()):
    """The outer loop for tests that do not use fedsim itself: contexts ->
    engine.run_iteration -> algorithm fold -> metric rows sorted by
    (population, name) -> callbacks (fedsim/engine/loop.py:62 semantics,
    cohort digest over repr((t, population, cohort))).  Test infrastructure;
    the product is driven by fedsim's own run_simulation."""
    import hashlib
    from types import SimpleNamespace

    state = algorithm.initial_state()
    rows, digest, t = [], hashlib.sha256(), 0
    while True:
        contexts = algorithm.get_next_central_contexts(state, t)
        if not contexts:
            break
        res = engine.run_iteration(algorithm, state, contexts)
        state = algorithm.process_aggregated_statistics_all_contexts(state, contexts, res.aggregates, res.metrics,
                                                                     res.user_updates)
        for pop, cohort in res.cohorts:
            digest.update(repr((t, pop, cohort)).encode())
        it_rows = [(t, pop, name, mv.value, mv.denominator) for (pop, name), mv in sorted(res.metrics.items())]
        rows.extend(it_rows)
        if any([bool(cb(state.params, tuple(it_rows), t)) for cb in callbacks]):
            t += 1
            break
        t += 1
    return SimulationResult(state=state, metrics_rows=rows, iterations_run=t, cohort_digest=digest.hexdigest())


class SimulationResult:
    def __init__(self, state, metrics_rows, iterations_run, cohort_digest):
        self.state, self.metrics_rows, self.iterations_run, self.cohort_digest = (state, metrics_rows,
                                                                                  iterations_run, cohort_digest)

    @property
    def params(self):
        return self.state.params
