"""Import the reference package (fedsim 0.1.0) from its local install in
baseline/_ref (git-ignored; installed by
``pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>``,
see DESIGN.md section 5).  Test infrastructure: the product never imports it."""

from __future__ import annotations

import os
import sys
import tempfile
from pathlib import Path

import pytest

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


def fedsim():
    if not (REF / "fedsim" / "__init__.py").exists():
        pytest.skip("the reference (fedsim) is not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "fedsim_numba_cache"))
    if str(REF) not in sys.path:
        sys.path.append(str(REF))
    import fedsim as fs  # noqa: F401
    import fedsim.algorithms
    import fedsim.engine
    import fedsim.feddata
    import fedsim.models
    import fedsim.privacy

    return fs


def build(cfg):
    """(datasets, algorithm, postprocessors) of a golden config built entirely
    from the reference's own classes -- the objects tests/golden/make_golden.py
    hands to fedsim's SimulationEngine."""
    import numpy as np  # noqa: F401

    fs = fedsim()
    from fedsim.algorithms.fedavg import AdaFedProx, FedAvg, FedProx
    from fedsim.algorithms.scaffold import Scaffold
    from fedsim.core import Population, derive_seed
    from fedsim.feddata import make_synthetic_classification, partition_iid
    from fedsim.models import MLP, LogisticRegression, Model, SGDOptimizer
    from fedsim.models.optimizers import AdamOptimizer
    from fedsim.privacy import ClippingPostprocessor, GaussianCentralMechanism

    from oracle.port import Cnn

    ppu = cfg["ppu"]
    ntr, nva = cfg["users"] * ppu, cfg["val_users"] * ppu
    X, y = make_synthetic_classification(ntr + nva, dim=cfg["dim"], num_classes=cfg["classes"],
                                         margin=cfg["margin"], seed=derive_seed(cfg["data_seed"], "pool"))
    ds = {Population.TRAIN: partition_iid(X[:ntr], y[:ntr], ppu, seed=derive_seed(cfg["data_seed"], "train", "split"),
                                          population=Population.TRAIN, id_prefix="train"),
          Population.VAL: partition_iid(X[ntr:], y[ntr:], ppu, seed=derive_seed(cfg["data_seed"], "val", "split"),
                                        population=Population.VAL, id_prefix="val")}

    class RefCNN(Model):  # the oracle CNN in the reference's generic Model contract
        def __init__(self):
            self.impl = Cnn()

        @property
        def param_dims(self):
            return self.impl.dims

        def init_params(self, seed):
            return self.impl.init(seed)

    if cfg["model"] == "mlp":
        model = MLP(dim=cfg["dim"], hidden_units=cfg["hidden"], num_classes=cfg["classes"])
    elif cfg["model"] == "logistic":
        model = LogisticRegression(dim=cfg["dim"], num_classes=cfg["classes"])
    else:
        model = RefCNN()
    o = cfg.get("optimizer", dict(kind="sgd"))
    opt = (AdamOptimizer(o["lr"], beta1=o["beta1"], beta2=o["beta2"], adaptivity_degree=o["eps"])
           if o["kind"] == "adam" else SGDOptimizer(cfg["clr"]))
    a = cfg.get("algorithm", dict(kind="fedavg"))
    kw = dict(total_iterations=cfg["iterations"], cohort_size=cfg["cohort"], local_learning_rate=cfg["lr"],
              local_num_epochs=cfg["epochs"], local_batch_size=cfg["batch"], eval_frequency=cfg["eval_every"],
              eval_cohort_size=cfg["eval_cohort"], weighting=cfg["weighting"], run_seed=cfg["run_seed"],
              init_seed=cfg["init_seed"])
    if a["kind"] == "fedprox":
        alg = FedProx(model, opt, mu=a["mu"], **kw)
    elif a["kind"] == "adafedprox":
        alg = AdaFedProx(model, opt, mu=a["mu"], **kw)
    elif a["kind"] == "scaffold":
        alg = Scaffold(model, opt, num_train_users=a["num_train_users"], **kw)
    else:
        alg = FedAvg(model, opt, **kw)
    post = []
    if cfg["bound"] is not None:
        clip = ClippingPostprocessor(cfg["bound"])
        post = [clip, GaussianCentralMechanism(clip, sigma=cfg["sigma"], r=cfg["r"],
                                               noise_base_seed=derive_seed(cfg["run_seed"], "noise-stream",
                                                                           cfg["noise_seed"]))]
    return fs, ds, alg, post
