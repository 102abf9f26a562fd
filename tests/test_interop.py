"""Duck-typed recognition of the reference's own objects (no GPU needed):
fedsim's models map onto the compiled layouts, its algorithms onto cohort
plans, its postprocessors / aggregator pass the engine's checks, and what
the GPU path cannot run is rejected with ValueError."""

from __future__ import annotations

import pytest

import paper_2404_06430_b200 as fb
from paper_2404_06430_b200 import interop
from tests.fedsim_ref import build, fedsim
from tests.helpers import CONFIGS


def test_reference_models_map_to_compiled_layouts():
    fedsim()
    from fedsim.models import MLP, LogisticRegression

    assert interop.native_model(LogisticRegression(dim=6, num_classes=3)) == fb.LogisticRegression(6, 3)
    assert interop.native_model(MLP(dim=8, hidden_units=16, num_classes=4)) == fb.MLP(8, 16, 4)
    _, _, alg, _ = build(CONFIGS["cnn_dp"])
    assert interop.native_model(alg.model) == fb.CNN()


def test_lm_layouts_map_to_transformer():
    """A fedsim Model wrapping the config C oracle LM (any vocab / width) maps onto
    the compiled TransformerLM of the same layout."""
    from oracle import port

    for shape in (dict(), dict(vocab=37, d=16, heads=4, ff=32, layers=2, seq=8)):
        m = port.TransformerLM(**shape)
        got = interop.native_model(m)
        assert isinstance(got, fb.TransformerLM) and got.param_dims == m.dims


@pytest.mark.parametrize("name,mu,scaffold", [("logistic_dp", 0.0, False), ("logistic_fedprox", 0.3, False),
                                              ("mlp_adafedprox", 0.1, False), ("mlp_scaffold_dp", 0.0, True)])
def test_reference_algorithms_become_cohort_plans(name, mu, scaffold):
    cfg = CONFIGS[name]
    _, _, alg, _ = build(cfg)
    state = alg.initial_state()
    train, *rest = alg.get_next_central_contexts(state, 0)
    plan = interop.cohort_plan(alg, state, train)
    assert plan.train == train.local_params and plan.weighting == cfg["weighting"]
    assert plan.prox_mu == pytest.approx(mu) and plan.scaffold is scaffold
    assert not interop.is_own(alg)
    for ctx in rest:
        assert interop.cohort_plan(alg, state, ctx).train is None


def test_reference_postprocessors_and_aggregator_accepted():
    _, _, _, post = build(CONFIGS["mlp_dp"])
    from fedsim.engine import SumAggregator

    interop.check_postprocessors(post)
    interop.check_aggregator(SumAggregator())
    interop.check_aggregator(fb.SumAggregator())
    interop.check_aggregator(None)


def test_unsupported_reference_objects_rejected():
    fedsim()
    from fedsim.engine.aggregator import Aggregator
    from fedsim.privacy import ClippingPostprocessor
    from fedsim.privacy.mechanisms import LaplaceCentralMechanism

    l1 = ClippingPostprocessor(1.0, norm_order=1.0)
    with pytest.raises(ValueError, match="L2"):
        interop.check_postprocessors([l1])
    with pytest.raises(ValueError, match="unsupported postprocessor"):
        interop.check_postprocessors([LaplaceCentralMechanism(l1, epsilon_per_query=1.0, noise_base_seed=0)])

    class Mean(Aggregator):
        pass

    with pytest.raises(ValueError, match="unsupported aggregator"):
        interop.check_aggregator(Mean())
    with pytest.raises(ValueError, match="unsupported algorithm"):
        interop.cohort_plan(object(), None, None)
