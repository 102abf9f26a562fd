"""Recognising the reference's own objects at the engine seam.

``GpuSimulationEngine`` is a drop-in for fedsim's ``SimulationEngine``
(fedsim/engine/runtime.py:43-104): the caller keeps fedsim's own
``run_simulation`` (fedsim/engine/loop.py:45-88), algorithm, postprocessors
and aggregator.  This module reads those objects by duck typing -- the
product never imports fedsim -- and maps each onto what the GPU path runs:

* algorithms: anything whose class hierarchy contains ``FedAvg``
  (fedsim/algorithms/fedavg.py:32-296: FedAvg, FedProx, AdaFedProx) or
  ``Scaffold`` (fedsim/algorithms/scaffold.py:28-120).  The per-user work
  ``simulate_one_user`` is described by a :class:`CohortPlan` built from the
  algorithm's public attributes (``model``, ``weighting``) and the context
  (``local_params``, ``algo_params["mu"]``, ``eval_params``);
* models: a layout whose ``param_dims`` equal one of the compiled models'
  (LogisticRegression / MLP of fedsim/models/models.py:85-228, the BASELINE
  CNN, config C's TransformerLM or config D's ResNet18);
* postprocessors: a clipping stage (``is_clipping``, fedsim/privacy/
  clipping.py:75-103) whose per-user half runs as the fused K2 kernel from
  ``current_bound``, and ``GaussianCentralMechanism`` (fedsim/privacy/
  mechanisms.py:171-193), whose per-user half is the identity.  Their
  server halves run as the objects' OWN ``postprocess_server`` on the
  reduced aggregate;
* aggregators: ``SumAggregator`` (fedsim/engine/aggregator.py:31-52),
  executed as the weighted-sum kernel plus the rank all-reduce.

Anything else raises ``ValueError`` naming the unsupported type, as the
reference does for bad arguments.
"""

from __future__ import annotations

from typing import Sequence

from .algorithms import CohortPlan

PACKAGE = __name__.rsplit(".", 1)[0]


def class_names(obj) -> set[str]:
    return {c.__name__ for c in type(obj).__mro__}


def is_own(obj) -> bool:
    """True for this package's own classes (DeviceStatistics-aware)."""
    return type(obj).__module__.split(".")[0] == PACKAGE


def is_clipping(p) -> bool:
    return bool(getattr(p, "is_clipping", False)) and hasattr(p, "current_bound")


def is_gaussian(p) -> bool:
    return "GaussianCentralMechanism" in class_names(p)


def check_postprocessors(postprocessors: Sequence) -> None:
    clips = 0
    for p in postprocessors:
        if is_clipping(p):
            clips += 1
            if float(p.norm_order) != 2.0:
                raise ValueError("GpuSimulationEngine supports L2 clipping only")
        elif is_gaussian(p):
            if getattr(p, "privatize_bookkeeping", False):
                raise ValueError("privatize_bookkeeping is not supported on the GPU path")
        else:
            raise ValueError(f"GpuSimulationEngine: unsupported postprocessor {type(p).__name__}")
    if clips > 1:
        raise ValueError("GpuSimulationEngine supports at most one clipping postprocessor")


def check_aggregator(aggregator) -> None:
    if aggregator is not None and "SumAggregator" not in class_names(aggregator):
        raise ValueError(f"GpuSimulationEngine: unsupported aggregator {type(aggregator).__name__}")


def native_model(model):
    """This package's compiled model with the same parameter layout as ``model``
    (entry names, order and sizes), or ValueError."""
    from .models import CNN, MLP, LogisticRegression, Model, ResNet18, TransformerLM

    if isinstance(model, Model):
        return model
    dims = dict(getattr(model, "param_dims", None) or getattr(model, "dims", None) or {})
    names = class_names(model)
    candidates = []
    if hasattr(model, "dim") and hasattr(model, "num_classes"):
        if hasattr(model, "hidden_units"):
            candidates.append(MLP(int(model.dim), int(model.hidden_units), int(model.num_classes)))
        else:
            candidates.append(LogisticRegression(int(model.dim), int(model.num_classes)))
    candidates.append(CNN())
    if hasattr(model, "vocab") and hasattr(model, "heads"):  # a config C transformer LM layout
        d = int(getattr(model, "d_model", getattr(model, "d", 96)))
        candidates.append(TransformerLM(int(model.vocab), d, int(model.heads), int(getattr(model, "ff", 1536)),
                                        int(getattr(model, "layers", 3)), int(getattr(model, "seq", 20))))
    candidates.append(TransformerLM())
    if hasattr(model, "width") and hasattr(model, "groups"):  # a config D ResNet-18 layout
        candidates.append(ResNet18(int(getattr(model, "num_classes", 17)), int(model.width), int(model.groups),
                                   int(getattr(model, "image", 224))))
    candidates.append(ResNet18())
    for cand in candidates:
        if list(cand.param_dims.items()) == [(n, int(k)) for n, k in dims.items()]:
            return cand
    raise ValueError(f"GpuSimulationEngine: unsupported model {sorted(names - {'object'})[0] if names else model!r} "
                     f"(parameter layout {dims})")


def cohort_plan(algorithm, state, context) -> CohortPlan:
    """What every cohort user does in ``context`` (fedsim/algorithms/fedavg.py:158-180;
    fedsim/algorithms/scaffold.py:46-79 for Scaffold users)."""
    if hasattr(algorithm, "cohort_plan"):
        return algorithm.cohort_plan(state, context)
    names = class_names(algorithm)
    if "FedAvg" not in names:
        raise ValueError(f"GpuSimulationEngine: unsupported algorithm {type(algorithm).__name__}")
    weighting = getattr(algorithm, "weighting", "datapoints")
    if weighting not in ("datapoints", "uniform"):
        raise ValueError(f"GpuSimulationEngine: unsupported weighting {weighting!r}")
    algo = dict(getattr(context, "algo_params", None) or {})
    eval_params = getattr(context, "eval_params", None)
    return CohortPlan(
        model=native_model(algorithm.model),
        train=context.local_params if context.do_training else None,
        weighting=weighting,
        prox_mu=float(algo.get("mu", 0.0)),
        eval_batch_size=int(getattr(eval_params, "batch_size", 0) or 0),
        scaffold="Scaffold" in names,
    )
