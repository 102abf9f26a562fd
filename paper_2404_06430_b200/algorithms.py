"""Federated algorithm contract and FedAvg (host mirror).

Mirror of fedsim/algorithms/base.py and fedsim/algorithms/fedavg.py.  The
three-operation contract is kept (contexts / per-user work / central
fold); the per-user work is *described* by :meth:`FedAvg.cohort_plan` and
executed for the whole cohort at once by ``GpuSimulationEngine``, so
``simulate_one_user`` deliberately has no host implementation (no CPU
fallback on the product path).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Any, Sequence

from .core import (
    CentralContext,
    EvalParams,
    HyperParam,
    LocalTrainParams,
    MetricValue,
    Population,
    average,
    cohort_seed,
    resolve,
)
from .models import CentralOptimizer, Model, central_step


@dataclass
class AlgorithmState:
    params: Any
    optimizer: CentralOptimizer
    extra: dict[str, Any] = field(default_factory=dict)


@dataclass
class UserResult:
    statistics: Any
    aux: dict[str, float]
    metrics: dict[str, MetricValue]
    algo_update: tuple[str, Any] | None = None


@dataclass(frozen=True)
class CohortPlan:
    """What every cohort user does in one context (read by the GPU engine).

    Mirrors FedAvg.simulate_one_user (fedsim/algorithms/fedavg.py:158-180):
    evaluate the broadcast model on all local rows, then -- for training
    contexts -- local SGD from the broadcast model and a weighted delta.
    """

    model: Model
    train: LocalTrainParams | None
    weighting: str                  # "datapoints" (w = n_u) or "uniform" (w = 1)
    prox_mu: float = 0.0
    eval_batch_size: int = 0
    scaffold: bool = False          # SCAFFOLD users: control-corrected SGD, [model | control] payload


class FederatedAlgorithm:
    def initial_state(self) -> AlgorithmState:
        raise NotImplementedError

    def get_next_central_contexts(self, state: AlgorithmState, iteration: int) -> tuple[CentralContext, ...]:
        raise NotImplementedError

    def simulate_one_user(self, state, user, context, seed) -> UserResult:
        raise NotImplementedError

    def process_aggregated_statistics_all_contexts(self, state, contexts, aggregates, iteration_metrics,
                                                   user_updates) -> AlgorithmState:
        raise NotImplementedError


class FedAvg(FederatedAlgorithm):
    """Weighted averaging of local-SGD deltas with a central optimizer
    (fedsim/algorithms/fedavg.py:32-198).  Same constructor; ``backend`` is
    accepted for signature compatibility and ignored."""

    def __init__(
        self,
        model: Model,
        optimizer: CentralOptimizer,
        *,
        total_iterations: int,
        cohort_size: int,
        local_learning_rate: "float | HyperParam",
        local_num_epochs: int,
        local_batch_size: int,
        eval_frequency: int,
        eval_cohort_size: int,
        eval_batch_size: int = 0,
        weighting: str = "datapoints",
        run_seed: int = 0,
        init_seed: int = 0,
        backend: str | None = None,
    ):
        if weighting not in ("datapoints", "uniform"):
            raise ValueError(f"unknown weighting {weighting!r}")
        if total_iterations < 0:
            raise ValueError("total_iterations must be >= 0")
        if eval_frequency < 1:
            raise ValueError("eval_frequency must be >= 1")
        self.model = model
        self.optimizer = optimizer
        self.total_iterations = total_iterations
        self.cohort_size = cohort_size
        self.local_learning_rate = local_learning_rate
        self.local_num_epochs = local_num_epochs
        self.local_batch_size = local_batch_size
        self.eval_frequency = eval_frequency
        self.eval_cohort_size = eval_cohort_size
        self.eval_batch_size = eval_batch_size
        self.weighting = weighting
        self.run_seed = run_seed
        self.init_seed = init_seed
        self.backend = backend

    def initial_state(self) -> AlgorithmState:
        """Host float64 params from the reference's init draws; the GPU
        engine uploads them to one flat fp32 HBM vector on first use."""
        return AlgorithmState(params=self.model.init_params(self.init_seed), optimizer=self.optimizer)

    def _algo_params(self, state: AlgorithmState, iteration: int) -> dict[str, float]:
        return {}

    def get_next_central_contexts(self, state: AlgorithmState, iteration: int) -> tuple[CentralContext, ...]:
        if iteration >= self.total_iterations:
            return ()
        train = CentralContext(
            iteration=iteration,
            population=Population.TRAIN,
            cohort_size=self.cohort_size,
            seed=cohort_seed(self.run_seed, iteration, Population.TRAIN.value),
            do_training=True,
            local_params=LocalTrainParams(
                resolve(self.local_learning_rate, iteration), self.local_num_epochs, self.local_batch_size
            ),
            eval_params=EvalParams(batch_size=self.eval_batch_size),
            algo_params=self._algo_params(state, iteration),
        )
        if iteration % self.eval_frequency:
            return (train,)
        val = CentralContext(
            iteration=iteration,
            population=Population.VAL,
            cohort_size=self.eval_cohort_size,
            seed=cohort_seed(self.run_seed, iteration, Population.VAL.value),
            do_training=False,
            eval_params=EvalParams(batch_size=self.eval_batch_size),
        )
        return (train, val)

    def cohort_plan(self, state: AlgorithmState, context: CentralContext) -> CohortPlan:
        return CohortPlan(
            model=self.model,
            train=context.local_params if context.do_training else None,
            weighting=self.weighting,
            prox_mu=float(context.algo_params.get("mu", 0.0)),
            eval_batch_size=context.eval_params.batch_size,
        )

    def simulate_one_user(self, state, user, context, seed) -> UserResult:
        raise NotImplementedError(
            "FedAvg users are simulated as a batched cohort by GpuSimulationEngine; "
            "there is no per-user host path"
        )

    def process_aggregated_statistics_all_contexts(self, state, contexts, aggregates, iteration_metrics,
                                                   user_updates) -> AlgorithmState:
        agg = next((a for c, a in zip(contexts, aggregates) if c.do_training), None)
        if agg is None:  # empty cohort or eval-only: nothing to apply
            return state
        state.params = central_step(state.optimizer, state.params, average(agg), contexts[0].iteration)
        return state


class FedProx(FedAvg):
    """FedAvg plus mu * (theta - theta_t) in the local gradient
    (fedsim/algorithms/fedavg.py:201-227); mu = 0 is FedAvg exactly."""

    def __init__(self, *args, mu: "float | HyperParam" = 0.0, **kwargs):
        super().__init__(*args, **kwargs)
        if resolve(mu, 0) < 0.0:
            raise ValueError("mu must be >= 0")
        self.mu = mu

    def _algo_params(self, state: AlgorithmState, iteration: int) -> dict[str, float]:
        return {"mu": resolve(self.mu, iteration)}


def adafedprox_update_mu(mu: float, previous_loss: float, current_loss: float, decrease_factor: float = 0.9,
                         increase_factor: float = 1.1, floor: float = 1e-4, cap: float = 1.0) -> float:
    """Loss-driven proximal strength (fedsim/algorithms/fedavg.py:230-245):
    relax when the central training loss improves, tighten when it does not."""
    if current_loss < previous_loss:
        return max(mu * decrease_factor, floor)
    if current_loss > previous_loss:
        return min(mu * increase_factor, cap)
    return mu


class AdaFedProx(FedProx):
    """FedProx with ``mu`` adapted from the central training loss
    (fedsim/algorithms/fedavg.py:248-296).  The loss metric comes from the
    GPU engine's pre-training evaluation of the train cohort."""

    def __init__(self, *args, mu: float = 0.1, mu_decrease_factor: float = 0.9, mu_increase_factor: float = 1.1,
                 mu_floor: float = 1e-4, mu_cap: float = 1.0, **kwargs):
        super().__init__(*args, mu=mu, **kwargs)
        self.mu_decrease_factor = mu_decrease_factor
        self.mu_increase_factor = mu_increase_factor
        self.mu_floor = mu_floor
        self.mu_cap = mu_cap

    def initial_state(self) -> AlgorithmState:
        state = super().initial_state()
        state.extra["mu"] = resolve(self.mu, 0)
        state.extra["previous_train_loss"] = None
        return state

    def _algo_params(self, state: AlgorithmState, iteration: int) -> dict[str, float]:
        return {"mu": state.extra["mu"]}

    def process_aggregated_statistics_all_contexts(self, state, contexts, aggregates, iteration_metrics,
                                                   user_updates) -> AlgorithmState:
        state = super().process_aggregated_statistics_all_contexts(state, contexts, aggregates, iteration_metrics,
                                                                   user_updates)
        loss = iteration_metrics.get((Population.TRAIN.value, "loss"))
        if loss is not None:
            current = loss.value
            previous = state.extra["previous_train_loss"]
            if previous is not None:
                state.extra["mu"] = adafedprox_update_mu(state.extra["mu"], previous, current,
                                                         self.mu_decrease_factor, self.mu_increase_factor,
                                                         self.mu_floor, self.mu_cap)
            state.extra["previous_train_loss"] = current
        return state


MODEL_PREFIX = "model/"
CONTROL_PREFIX = "control/"


class Scaffold(FedAvg):
    """Stochastic controlled averaging with per-user control variates
    (fedsim/algorithms/scaffold.py:28-120).  Same constructor and semantics:
    uniform weighting only; users train with g - c_i + c and report
    [model delta | control delta]; the server control moves by the cohort
    fraction of the mean control delta.  On the GPU the controls live in a
    device store (``state.extra["user_controls"]``, a :class:`ControlStore`)
    and the server control is a flat fp32 device vector; the engine runs
    the cohort's corrections, payload and user updates as kernels
    (fb_scaffold_*)."""

    def __init__(self, *args, num_train_users: int, **kwargs):
        kwargs.setdefault("weighting", "uniform")
        if kwargs["weighting"] != "uniform":
            raise ValueError("control-variate averaging must be uniform")
        super().__init__(*args, **kwargs)
        if num_train_users < 1:
            raise ValueError("num_train_users must be >= 1")
        self.num_train_users = num_train_users

    def initial_state(self) -> AlgorithmState:
        state = super().initial_state()
        state.extra["server_control"] = None   # flat device vector, created by the engine (zeros)
        state.extra["user_controls"] = None    # ControlStore, created by the engine
        return state

    def cohort_plan(self, state: AlgorithmState, context: CentralContext) -> CohortPlan:
        plan = super().cohort_plan(state, context)
        return CohortPlan(plan.model, plan.train, plan.weighting, 0.0, plan.eval_batch_size, scaffold=True)

    def process_aggregated_statistics_all_contexts(self, state, contexts, aggregates, iteration_metrics,
                                                   user_updates) -> AlgorithmState:
        store = state.extra["user_controls"]
        if user_updates:
            if hasattr(user_updates, "matrix"):
                store.set_rows(user_updates.uids, user_updates.matrix)
            else:
                for uid, vec in user_updates:
                    store.set_rows([uid], vec.reshape(1, -1))
        agg = next((a for c, a in zip(contexts, aggregates) if c.do_training), None)
        if agg is None:
            return state
        D = state.params.num_params
        averaged = average(agg)
        model_part, control_part = averaged.split_payload([D, D])
        model_part = replace(model_part, dims={n[len(MODEL_PREFIX):]: k for n, k in model_part.dims.items()})
        state.params = central_step(state.optimizer, state.params, model_part, contexts[0].iteration)
        # server control moves by the cohort fraction of the mean control delta
        fraction = agg.weight / self.num_train_users
        server = state.extra["server_control"]
        from . import native  # local import: the host mirror imports without the library

        nz = control_part.noise
        native.call("fb_noise_avg_sgd_f32", native.ptr(server), native.ptr(control_part.flat), D, 0.0, 0,
                    native.ptr(nz.injected) if nz is not None and nz.injected is not None else None,
                    float(control_part.scale), -float(fraction), None, native.stream_handle())
        return state
