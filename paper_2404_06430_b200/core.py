"""Value types that cross the central-iteration path.

Host-side mirror of the reference's core layer (fedsim/core/*.py): seed
streams, per-iteration contexts, scheduled hyperparameters, summable
metrics and the ``Statistics`` payload algebra.  Semantics (names,
argument meaning, validation and exceptions) follow the reference so the
GPU engine is a drop-in; the implementation is independent.

Seed derivation is bit-exact with fedsim/core/seeds.py:18-42 because the
cohort draw, the LPT shard map and every client's minibatch order must be
identical to the reference's (north_star: "bit-exact sampling").
"""

from __future__ import annotations

import enum
import hashlib
import math
from dataclasses import dataclass, field
from typing import Iterable, Mapping, Union

import numpy as np

from .errors import EmptyCohort, IncompatibleShapes, ZeroWeight

# --------------------------------------------------------------------------
# seeds (fedsim/core/seeds.py:18-42)

_SEED_MASK = (1 << 63) - 1
_SEP = b"\x1f"


def derive_seed(*parts: int | str) -> int:
    """63-bit seed = first 8 sha256 bytes (little endian) of the
    ``repr``-encoded parts, each followed by a unit separator
    (fedsim/core/seeds.py:18-24)."""
    digest = hashlib.sha256(b"".join(repr(p).encode() + _SEP for p in parts)).digest()
    return int.from_bytes(digest[:8], "little") & _SEED_MASK


def make_rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def user_seed(context_seed: int, user_id: str) -> int:
    return derive_seed(context_seed, "user", user_id)


def cohort_seed(run_seed: int, iteration: int, population: str) -> int:
    return derive_seed(run_seed, "cohort", iteration, population)


def noise_seed(noise_base_seed: int, iteration: int, population: str) -> int:
    return derive_seed(noise_base_seed, "noise", iteration, population)


# --------------------------------------------------------------------------
# contexts (fedsim/core/context.py:9-65)


class Population(enum.Enum):
    TRAIN = "train"
    VAL = "val"


@dataclass(frozen=True)
class LocalTrainParams:
    learning_rate: float
    num_epochs: int
    batch_size: int

    def __post_init__(self) -> None:
        for ok, msg in (
            (self.learning_rate >= 0.0, "learning_rate must be >= 0"),
            (self.num_epochs >= 0, "num_epochs must be >= 0"),
            (self.batch_size >= 1, "batch_size must be >= 1"),
        ):
            if not ok:
                raise ValueError(msg)


@dataclass(frozen=True)
class EvalParams:
    """``batch_size`` 0 evaluates a user's data as one batch."""

    batch_size: int = 0


@dataclass(frozen=True)
class CentralContext:
    iteration: int
    population: Population
    cohort_size: int
    seed: int
    do_training: bool
    local_params: LocalTrainParams | None = None
    eval_params: EvalParams = field(default_factory=EvalParams)
    algo_params: Mapping[str, float] = field(default_factory=dict)

    def __post_init__(self) -> None:
        if self.do_training is (self.local_params is None):
            raise ValueError("local_params must be present exactly when do_training is set")
        if self.cohort_size < 1:
            raise ValueError("cohort_size must be >= 1")
        if self.iteration < 0:
            raise ValueError("iteration must be >= 0")


# --------------------------------------------------------------------------
# scheduled hyperparameters (fedsim/core/hyperparams.py:14-76)


@dataclass(frozen=True)
class Constant:
    def value_at(self, base: float, iteration: int) -> float:
        return base


@dataclass(frozen=True)
class LinearWarmup:
    warmup_iterations: int

    def __post_init__(self) -> None:
        if self.warmup_iterations < 1:
            raise ValueError("warmup_iterations must be >= 1")

    def value_at(self, base: float, iteration: int) -> float:
        return base * min(iteration + 1, self.warmup_iterations) / self.warmup_iterations


@dataclass(frozen=True)
class PiecewiseConstant:
    steps: tuple[tuple[int, float], ...]

    def __post_init__(self) -> None:
        starts = [s for s, _ in self.steps]
        if starts != sorted(starts):
            raise ValueError("piecewise steps must be sorted by start iteration")

    def value_at(self, base: float, iteration: int) -> float:
        active = [v for s, v in self.steps if s <= iteration]
        return active[-1] if active else base


Schedule = Union[Constant, LinearWarmup, PiecewiseConstant]


@dataclass(frozen=True)
class HyperParam:
    base_value: float
    schedule: Schedule = field(default_factory=Constant)

    def value_at(self, iteration: int) -> float:
        return self.schedule.value_at(self.base_value, iteration)


def resolve(value: "float | HyperParam", iteration: int) -> float:
    return value.value_at(iteration) if isinstance(value, HyperParam) else float(value)


# --------------------------------------------------------------------------
# metrics (fedsim/core/metrics.py:22-93)


class MetricKind(enum.Enum):
    CENTRAL = "central"
    PER_USER = "per_user"


@dataclass(frozen=True)
class MetricValue:
    """A summable (numerator, denominator) pair."""

    kind: MetricKind
    numerator: float
    denominator: float

    def __post_init__(self) -> None:
        if not (math.isfinite(self.numerator) and math.isfinite(self.denominator)):
            raise ValueError("metric components must be finite")
        if self.denominator < 0.0:
            raise ValueError("metric denominator must be >= 0")

    @classmethod
    def from_user(cls, kind: MetricKind, numerator: float, denominator: float) -> "MetricValue":
        if denominator <= 0.0:
            raise ValueError("a user's metric denominator must be > 0")
        if kind is MetricKind.PER_USER:
            return cls(kind, numerator / denominator, 1.0)
        return cls(kind, float(numerator), float(denominator))

    def __add__(self, other: "MetricValue") -> "MetricValue":
        if self.kind is not other.kind:
            raise IncompatibleShapes(
                f"cannot merge {self.kind.value} with {other.kind.value} metric"
            )
        return MetricValue(
            self.kind, self.numerator + other.numerator, self.denominator + other.denominator
        )

    @property
    def value(self) -> float:
        if self.denominator == 0.0:
            raise ZeroDivisionError("metric has zero denominator")
        return self.numerator / self.denominator


def metric_aggregate(values: Iterable[MetricValue]) -> float:
    values = list(values)
    if not values:
        raise EmptyCohort("cannot aggregate metrics over zero users")
    total = values[0]
    for v in values[1:]:
        total = total + v
    return total.value


def merge_metrics(a: Mapping[str, MetricValue], b: Mapping[str, MetricValue]) -> dict[str, MetricValue]:
    out = dict(a)
    for name, val in b.items():
        out[name] = out[name] + val if name in out else val
    return out


# --------------------------------------------------------------------------
# host statistics (fedsim/core/statistics.py:21-147)


@dataclass(frozen=True)
class Statistics:
    """Ordered name -> flat float64 vector, plus a weight >= 0.

    This is the host form.  The GPU engine hands back
    :class:`paper_2404_06430_b200.device.DeviceStatistics`, which keeps
    the payload in one flat fp32 device buffer with the same entry order.
    """

    entries: dict[str, np.ndarray]
    weight: float

    @classmethod
    def from_entries(cls, entries: Mapping[str, np.ndarray], weight: float) -> "Statistics":
        weight = float(weight)
        if not math.isfinite(weight) or weight < 0.0:
            raise ValueError(f"weight must be finite and >= 0, got {weight}")
        checked: dict[str, np.ndarray] = {}
        for name, vec in entries.items():
            arr = np.array(vec, dtype=np.float64, copy=True)
            if arr.ndim != 1:
                raise ValueError(f"entry {name!r} must be a flat vector, got shape {arr.shape}")
            if not np.isfinite(arr).all():
                raise ValueError(f"entry {name!r} contains non-finite values")
            if weight == 0.0 and arr.any():
                raise ValueError(f"zero-weight statistics must be all zero, entry {name!r} is not")
            checked[name] = arr
        return cls(entries=checked, weight=weight)

    @classmethod
    def zeros(cls, dims: Mapping[str, int]) -> "Statistics":
        return cls(entries={n: np.zeros(int(k)) for n, k in dims.items()}, weight=0.0)

    @property
    def names(self) -> tuple[str, ...]:
        return tuple(self.entries)

    @property
    def num_dims(self) -> int:
        return int(sum(v.size for v in self.entries.values()))

    def get(self, name: str) -> np.ndarray:
        return self.entries[name]


def _same_layout(a: Statistics, b: Statistics) -> None:
    if set(a.entries) != set(b.entries):
        raise IncompatibleShapes(f"entry names differ: {sorted(a.entries)} vs {sorted(b.entries)}")
    for name, vec in a.entries.items():
        if vec.shape != b.entries[name].shape:
            raise IncompatibleShapes(
                f"entry {name!r} length differs: {vec.size} vs {b.entries[name].size}"
            )


def accumulate(a: Statistics, b: Statistics) -> Statistics:
    _same_layout(a, b)
    return Statistics({n: v + b.entries[n] for n, v in a.entries.items()}, a.weight + b.weight)


def average(stats):
    """Divide by the total weight (result weight 1).  Dispatches to the
    device form when given a DeviceStatistics (lazy: fused into the
    central step kernel)."""
    if hasattr(stats, "averaged"):
        return stats.averaged()
    if stats.weight == 0.0:
        raise ZeroWeight("cannot average statistics with zero total weight")
    inv = 1.0 / stats.weight
    return Statistics({n: v * inv for n, v in stats.entries.items()}, 1.0)


def scale_entries(stats: Statistics, factor: float) -> Statistics:
    return Statistics({n: v * factor for n, v in stats.entries.items()}, stats.weight)


def weighted(entries: Mapping[str, np.ndarray], weight: float) -> Statistics:
    if weight < 0.0 or not math.isfinite(weight):
        raise ValueError(f"weight must be finite and >= 0, got {weight}")
    return Statistics.from_entries(
        {n: np.asarray(v, dtype=np.float64) * weight for n, v in entries.items()}, weight
    )


def global_norm(stats, order: float = 2.0, names: Iterable[str] | None = None) -> float:
    selected = stats.names if names is None else tuple(names)
    if not selected:
        return 0.0
    if hasattr(stats, "device_norm"):
        return stats.device_norm(order, selected)
    flat = np.concatenate([stats.entries[n] for n in selected])
    return float(np.linalg.norm(flat, ord=order))
