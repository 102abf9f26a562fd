"""The engine seam with the reference's OWN objects: fedsim's run_simulation
(fedsim/engine/loop.py:45-88) drives GpuSimulationEngine with fedsim's
FedAvg / FedProx / AdaFedProx / Scaffold, ClippingPostprocessor,
GaussianCentralMechanism (its own numpy noise), SumAggregator, datasets and
host float64 ModelParams -- exactly the objects make_golden.py gave fedsim's
SimulationEngine.  Cohort digests must be identical and every iteration's
theta / metric row equal the golden run (rtol 1e-5 / atol 1e-6 max|ref|; rows
rtol 2e-5)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2404_06430_b200 as fb
from tests.conftest import assert_close_fp32
from tests.fedsim_ref import build
from tests.helpers import CONFIGS, golden_rows

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["logistic_dp", "mlp_dp", "mlp_adam_dp", "logistic_fedprox", "mlp_adafedprox",
                                  "mlp_scaffold_dp", "logistic_scaffold", "cnn_dp"])
def test_fedsim_run_simulation_on_gpu_engine_matches_reference_run(name, golden):
    g = golden(name)
    cfg = CONFIGS[name]
    fs, ds, alg, post = build(cfg)
    from fedsim.engine import SumAggregator, run_simulation

    eng = fb.GpuSimulationEngine(ds, postprocessors=post, aggregator=SumAggregator())
    names = list(alg.model.param_dims)
    thetas = []
    res = run_simulation(alg, eng, callbacks=[
        lambda p, rows, t: thetas.append(np.concatenate([np.asarray(p[n]) for n in names])) and False])
    assert isinstance(res.state.params, dict)              # the reference's host ModelParams throughout
    assert res.cohort_digest == str(g["digest"])
    keep = g["keep"] if "keep" in g else slice(None)
    assert len(thetas) == len(g["thetas"])
    for t, th in enumerate(thetas):
        assert_close_fp32(th[keep], g["thetas"][t], what=f"{name}: theta after iteration {t}")
    got, ref = res.metrics_rows, golden_rows(g)
    assert [r[:3] for r in got] == [r[:3] for r in ref]
    np.testing.assert_allclose([r[3] for r in got], [r[3] for r in ref], rtol=2e-5)
