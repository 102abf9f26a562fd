"""Generate the golden fixtures by running the REFERENCE (fedsim 0.1.0).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports fedsim from /root/reference/pkg/src (numba cache redirected to
/tmp because the reference tree is read-only), runs small configurations
through the reference's own SimulationEngine / run_simulation / FedAvg /
ClippingPostprocessor / GaussianCentralMechanism, and writes compact .npz
fixtures next to this script.  The GPU box never needs /root/reference:
tests regenerate the same datasets with paper_2404_06430_b200.feddata
(bit-exact replica of the reference generators; checked by a test).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fedsim_numba_cache")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(HERE.parent.parent))

from fedsim.algorithms import FedAvg  # noqa: E402
from fedsim.algorithms.fedavg import AdaFedProx, FedProx  # noqa: E402
from fedsim.algorithms.scaffold import Scaffold  # noqa: E402
from fedsim.core import LocalTrainParams, Population, cohort_seed, derive_seed, user_seed  # noqa: E402
from fedsim.engine import SimulationEngine, compute_base_weight, run_simulation, schedule_users  # noqa: E402
from fedsim.feddata import make_synthetic_classification, partition_iid, sample_cohort  # noqa: E402
from fedsim.models import MLP, LogisticRegression, Model, SGDOptimizer, local_train_sgd  # noqa: E402
from fedsim.models.optimizers import AdamOptimizer  # noqa: E402
from fedsim.privacy import ClippingPostprocessor, GaussianCentralMechanism  # noqa: E402

from oracle.port import Cnn  # noqa: E402

from tests.golden.configs import CONFIGS  # noqa: E402


def datasets(cfg, make_synth=make_synthetic_classification, part=partition_iid, pop=Population):
    ppu = cfg["ppu"]
    ntr, nva = cfg["users"] * ppu, cfg["val_users"] * ppu
    X, y = make_synth(ntr + nva, dim=cfg["dim"], num_classes=cfg["classes"], margin=cfg["margin"],
                      seed=derive_seed(cfg["data_seed"], "pool"))
    train = part(X[:ntr], y[:ntr], ppu, seed=derive_seed(cfg["data_seed"], "train", "split"),
                 population=pop.TRAIN, id_prefix="train")
    val = part(X[ntr:], y[ntr:], ppu, seed=derive_seed(cfg["data_seed"], "val", "split"),
               population=pop.VAL, id_prefix="val")
    return {pop.TRAIN: train, pop.VAL: val}


class RefCNN(Model):
    """The oracle CNN plugged into the REFERENCE's generic Model contract, so
    the reference's own fit_local loop (fedsim/models/models.py:53-79) and
    engine drive it."""

    def __init__(self):
        self.impl = Cnn()

    @property
    def param_dims(self):
        return self.impl.dims

    def init_params(self, seed):
        return self.impl.init(seed)

    def loss_and_grad(self, params, X, y):
        return self.impl.loss_and_grad(params, X, y)

    def eval_counts(self, params, X, y, backend=None):
        return self.impl.eval_counts(params, X, y)


def build_model(cfg):
    if cfg["model"] == "mlp":
        return MLP(dim=cfg["dim"], hidden_units=cfg["hidden"], num_classes=cfg["classes"])
    if cfg["model"] == "logistic":
        return LogisticRegression(dim=cfg["dim"], num_classes=cfg["classes"])
    return RefCNN()


def build_algorithm(cfg, model):
    o = cfg.get("optimizer", dict(kind="sgd"))
    opt = (AdamOptimizer(o["lr"], beta1=o["beta1"], beta2=o["beta2"], adaptivity_degree=o["eps"])
           if o["kind"] == "adam" else SGDOptimizer(cfg["clr"]))
    a = cfg.get("algorithm", dict(kind="fedavg"))
    kw = dict(total_iterations=cfg["iterations"], cohort_size=cfg["cohort"], local_learning_rate=cfg["lr"],
              local_num_epochs=cfg["epochs"], local_batch_size=cfg["batch"], eval_frequency=cfg["eval_every"],
              eval_cohort_size=cfg["eval_cohort"], weighting=cfg["weighting"], run_seed=cfg["run_seed"],
              init_seed=cfg["init_seed"])
    if a["kind"] == "fedprox":
        return FedProx(model, opt, mu=a["mu"], **kw)
    if a["kind"] == "adafedprox":
        return AdaFedProx(model, opt, mu=a["mu"], **kw)
    if a["kind"] == "scaffold":
        return Scaffold(model, opt, num_train_users=a["num_train_users"], **kw)
    return FedAvg(model, opt, **kw)


def run_config(name, cfg):
    ds = datasets(cfg)
    model = build_model(cfg)
    alg = build_algorithm(cfg, model)
    post = []
    if cfg["bound"] is not None:
        clip = ClippingPostprocessor(cfg["bound"])
        post = [clip, GaussianCentralMechanism(clip, sigma=cfg["sigma"], r=cfg["r"],
                                               noise_base_seed=derive_seed(cfg["run_seed"], "noise-stream",
                                                                           cfg["noise_seed"]))]
    engine = SimulationEngine(ds, num_workers=cfg["workers"], postprocessors=post)
    names = list(model.param_dims)
    thetas = []
    res = run_simulation(alg, engine, callbacks=[
        lambda p, rows, t: thetas.append(np.concatenate([p[n] for n in names])) and False])
    theta0 = np.concatenate([alg.model.init_params(cfg["init_seed"])[n] for n in names])
    rows = res.metrics_rows
    out = dict(
        theta0=theta0, thetas=np.array(thetas), digest=np.array(res.cohort_digest),
        row_t=np.array([r[0] for r in rows]), row_pop=np.array([r[1] for r in rows]),
        row_name=np.array([r[2] for r in rows]), row_value=np.array([r[3] for r in rows]),
        row_weight=np.array([r[4] for r in rows]),
    )
    # iteration-0 internals of the train context, straight from reference calls
    ctx_seed = cohort_seed(cfg["run_seed"], 0, "train")
    train = ds[Population.TRAIN]
    cohort = sample_cohort(train, cfg["cohort"], ctx_seed)
    w = {u: float(train.users[u].weight) for u in cohort}
    queues = schedule_users(w, cfg["workers"], compute_base_weight(list(w.values()), "median")).queues
    params0 = alg.model.init_params(cfg["init_seed"])
    deltas = []
    lp = LocalTrainParams(cfg["lr"], cfg["epochs"], cfg["batch"])
    for u in cohort:
        user = train.users[u]
        after = local_train_sgd(alg.model, params0, user.features, user.labels, lp, user_seed(ctx_seed, u))
        deltas.append(np.concatenate([params0[n] - after[n] for n in names]))
    out.update(cohort0=np.array(cohort), queues0=np.array(["|".join(q) for q in queues]),
               deltas0=np.array(deltas))
    if cfg["model"] == "cnn":
        # fc1/weights dominates D (1.6M); keep every other entry whole plus a
        # fixed sample of fc1 so the fixture stays small
        dims = model.param_dims
        starts = np.cumsum([0] + list(dims.values()))
        lo = starts[names.index("fc1/weights")]
        hi = lo + dims["fc1/weights"]
        keep = np.concatenate([np.arange(0, lo), np.sort(np.random.default_rng(0).choice(
            np.arange(lo, hi), 40000, replace=False)), np.arange(hi, starts[-1])])
        for key in ("theta0", "thetas", "deltas0"):
            full = out[key]
            out[key + "_l2"] = np.linalg.norm(full, axis=-1)
            out[key] = full[..., keep]
        out["keep"] = keep
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "iterations", len(thetas), "digest", res.cohort_digest[:16])


def sampling():
    from fedsim.feddata import FederatedDataset, UserDataset

    rng = np.random.default_rng(123)
    out = {}
    for N, C, seed in [(1000, 50, 7), (1000, 1000, 8), (20000, 100, 9), (20000, 1000, 10), (30, 30, 11)]:
        users = {f"u{i:05d}": UserDataset(f"u{i:05d}", np.zeros((1, 1)), np.zeros(1, dtype=np.int64))
                 for i in range(N)}
        ds = FederatedDataset(users=users, population=Population.TRAIN)
        out[f"cohort_{N}_{C}_{seed}"] = np.array(sample_cohort(ds, C, seed))
    sizes = rng.integers(1, 500, size=200).astype(float)
    weights = {f"c{i:04d}": float(s) for i, s in enumerate(sizes)}
    for m in (1, 2, 3, 8):
        base = compute_base_weight(list(weights.values()), "median")
        out[f"queues_m{m}"] = np.array(["|".join(q) for q in schedule_users(weights, m, base).queues])
    out["sched_sizes"] = sizes
    perms = []
    for i in range(50):
        s = user_seed(derive_seed(1, "cohort", i, "train"), f"train{i:05d}")
        r = np.random.default_rng(s)
        perms.append(np.concatenate([r.permutation(50), r.permutation(50)]))
    out["perms"] = np.array(perms)
    out["seeds"] = np.array([derive_seed(0, "pool"), derive_seed(7, "user", "train00042"),
                             cohort_seed(0, 3, "val"), derive_seed(0, "noise-stream", 0)], dtype=np.uint64)
    np.savez_compressed(HERE / "sampling.npz", **out)
    print("sampling fixtures", len(out))


if __name__ == "__main__":
    sampling()
    only = set(sys.argv[1:])
    for name, cfg in CONFIGS.items():
        if not only or name in only:
            run_config(name, cfg)
