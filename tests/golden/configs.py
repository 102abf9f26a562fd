"""Configurations of the golden fixtures (shared by make_golden.py and the tests)."""

# Shared config table: tests rebuild the same datasets from these numbers.
CONFIGS = {
    "mlp_dp": dict(model="mlp", hidden=16, dim=8, classes=4, users=60, val_users=10, ppu=20, margin=3.0,
                   data_seed=3, cohort=12, eval_cohort=6, epochs=2, batch=7, lr=0.1, clr=1.0,
                   weighting="uniform", bound=0.3, sigma=1.1, r=0.5, noise_seed=5, run_seed=11,
                   init_seed=2, iterations=3, eval_every=2, workers=1),
    "logistic_dp": dict(model="logistic", dim=6, classes=3, users=40, val_users=8, ppu=15, margin=2.0,
                        data_seed=4, cohort=10, eval_cohort=8, epochs=1, batch=4, lr=0.2, clr=0.5,
                        weighting="datapoints", bound=2.0, sigma=0.7, r=1.0, noise_seed=1, run_seed=9,
                        init_seed=0, iterations=3, eval_every=1, workers=2),
    "mlp_noclip": dict(model="mlp", hidden=32, dim=32, classes=10, users=100, val_users=20, ppu=50, margin=6.0,
                       data_seed=0, cohort=50, eval_cohort=20, epochs=1, batch=10, lr=0.1, clr=1.0,
                       weighting="datapoints", bound=None, sigma=0.0, r=1.0, noise_seed=0, run_seed=0,
                       init_seed=0, iterations=2, eval_every=10, workers=1),
    "cnn_dp": dict(model="cnn", dim=3072, classes=10, users=8, val_users=4, ppu=7, margin=6.0,
                   data_seed=1, cohort=4, eval_cohort=3, epochs=1, batch=3, lr=0.05, clr=1.0,
                   weighting="uniform", bound=0.5, sigma=0.9, r=0.2, noise_seed=3, run_seed=4,
                   init_seed=1, iterations=2, eval_every=1, workers=1),
}

# Algorithm / central-optimizer variants: the
# same data recipes run through the reference's FedProx, AdaFedProx, Scaffold
# and AdamOptimizer.
_VARIANTS = {
    "mlp_adam_dp": ("mlp_dp", dict(optimizer=dict(kind="adam", lr=0.05, beta1=0.9, beta2=0.99, eps=0.1),
                                   iterations=4)),
    "logistic_fedprox": ("logistic_dp", dict(algorithm=dict(kind="fedprox", mu=0.3))),
    "mlp_adafedprox": ("mlp_dp", dict(algorithm=dict(kind="adafedprox", mu=0.1), bound=None, sigma=0.0,
                                      iterations=4, eval_every=1)),
    "mlp_scaffold_dp": ("mlp_dp", dict(algorithm=dict(kind="scaffold", num_train_users=60), cohort=30,
                                       iterations=3)),
    "logistic_scaffold": ("logistic_dp", dict(algorithm=dict(kind="scaffold", num_train_users=40), bound=None,
                                              sigma=0.0, weighting="uniform", epochs=2, cohort=20, iterations=4,
                                              workers=1)),
    "cnn_scaffold": ("cnn_dp", dict(algorithm=dict(kind="scaffold", num_train_users=8), iterations=3)),
}
for _name, (_base, _over) in _VARIANTS.items():
    CONFIGS[_name] = {**CONFIGS[_base], **_over}
