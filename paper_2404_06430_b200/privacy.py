"""Per-user L2 clipping and the central Gaussian mechanism (postprocessors).

Mirror of fedsim/privacy/clipping.py and fedsim/privacy/mechanisms.py for
the GPU engine.  The *local* halves do not run per user on the host: the
engine reads ``current_bound`` and runs the fused delta/norm/clip kernel
(K2) over the whole cohort, then sums the ``_clip/*`` bookkeeping channels
alongside the payload.  The *server* halves run on the reduced aggregate
exactly as the reference orders them (reversed pipeline: noise first, then
the clip finaliser; fedsim/engine/runtime.py:159-170) -- small host scalar
math plus, for the mechanism, a device norm (SNR) and a pending noise
record that the central step applies in its fused kernel.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .core import CentralContext, MetricKind, MetricValue, Statistics, global_norm, make_rng, noise_seed
from .errors import NotClippedUpstream

BOOKKEEPING_PREFIX = "_"
CLIPPED_KEY = "_clip/clipped"
COUNT_KEY = "_clip/count"
NORM_KEY = "_clip/norm_sum"
MIN_BOUND = 1e-6
MAX_BOUND = 1e6


@dataclass(frozen=True)
class AdaptiveClipConfig:
    """Geometric bound adaptation toward a target clipped fraction
    (fedsim/privacy/config.py, fedsim/privacy/clipping.py:59-72)."""

    quantile: float = 0.5
    learning_rate: float = 0.2

    def __post_init__(self) -> None:
        if not 0.0 <= self.quantile <= 1.0:
            raise ValueError("adaptive quantile must be in [0, 1]")
        if self.learning_rate < 0.0:
            raise ValueError("adaptive learning_rate must be >= 0")


def payload_names(stats) -> tuple[str, ...]:
    return tuple(n for n in stats.names if not n.startswith(BOOKKEEPING_PREFIX))


def adaptive_clip_update(bound: float, clipped_fraction: float, quantile: float, learning_rate: float) -> float:
    grown = bound * float(np.exp(-learning_rate * (clipped_fraction - quantile)))
    return float(np.clip(grown, MIN_BOUND, MAX_BOUND))


def _strip_bookkeeping(stats):
    if hasattr(stats, "without_bookkeeping"):
        return stats.without_bookkeeping()
    return Statistics(
        entries={n: v for n, v in stats.entries.items() if not n.startswith(BOOKKEEPING_PREFIX)},
        weight=stats.weight,
    )


class ClippingPostprocessor:
    """Clips every user's weighted delta to ``current_bound`` (L2 only on
    the GPU path) and tracks the live bound (fedsim/privacy/clipping.py:75-146)."""

    is_clipping = True

    def __init__(self, bound: float, norm_order: float = 2.0, adaptive: AdaptiveClipConfig | None = None):
        if bound <= 0.0:
            raise ValueError("bound must be > 0")
        if norm_order not in (1.0, 2.0):
            raise ValueError("norm_order must be 1 or 2")
        self._bound = float(bound)
        self.norm_order = norm_order
        self.adaptive = adaptive

    @property
    def current_bound(self) -> float:
        return self._bound

    def postprocess_one_user(self, stats, aux, context):
        raise NotImplementedError(
            "per-user clipping runs fused on the GPU (fb_delta_norm_clip_f32) inside "
            "GpuSimulationEngine; there is no host per-user path"
        )

    def postprocess_server(self, stats, context: CentralContext):
        count = float(stats.entries[COUNT_KEY][0])
        clipped = float(stats.entries[CLIPPED_KEY][0])
        norm_sum = float(stats.entries[NORM_KEY][0])
        bound_used = self._bound
        metrics = {
            "clip_fraction": MetricValue(MetricKind.CENTRAL, clipped, count),
            "update_norm": MetricValue(MetricKind.CENTRAL, norm_sum, count),
            "clipping_bound": MetricValue(MetricKind.CENTRAL, bound_used, 1.0),
        }
        if self.adaptive is not None and count > 0:
            self._bound = adaptive_clip_update(
                self._bound, clipped / count, self.adaptive.quantile, self.adaptive.learning_rate
            )
        return _strip_bookkeeping(stats), metrics


def snr(aggregate, sigma_applied: float, dimension: int) -> float:
    """||payload|| / sqrt(d * sigma^2) of the UN-noised aggregate
    (fedsim/privacy/mechanisms.py:30-46)."""
    if sigma_applied < 0.0:
        raise ValueError("sigma_applied must be >= 0")
    if dimension < 1:
        raise ValueError("dimension must be >= 1")
    signal = global_norm(aggregate, names=payload_names(aggregate))
    if sigma_applied == 0.0:
        if signal == 0.0:
            raise ValueError("SNR undefined: zero signal and zero noise")
        return math.inf
    return signal / math.sqrt(dimension * sigma_applied**2)


NOISE_SOURCES = ("philox", "numpy")


class GaussianCentralMechanism:
    """Central Gaussian noise with std ``r * sigma * current_bound``
    (fedsim/privacy/mechanisms.py:115-193).

    ``noise_source="philox"`` (default) draws on the device from a
    counter-based stream keyed by the reference's per-iteration noise seed;
    ``"numpy"`` replays the reference's exact PCG64 draws on the host and
    injects them (parity runs; slow at large D).
    """

    requires_clipping = True

    def __init__(self, clipping: ClippingPostprocessor, sigma: float, r: float, noise_base_seed: int,
                 privatize_bookkeeping: bool = False, noise_source: str = "philox"):
        if sigma < 0.0:
            raise ValueError("sigma must be >= 0")
        if r <= 0.0:
            raise ValueError("r must be > 0")
        if clipping.norm_order != 2.0:
            raise ValueError("gaussian mechanism needs an L2 clipping bound")
        if noise_source not in NOISE_SOURCES:
            raise ValueError(f"noise_source must be one of {NOISE_SOURCES}")
        self.clipping = clipping
        self.sigma = sigma
        self.r = r
        self.noise_base_seed = noise_base_seed
        self.privatize_bookkeeping = privatize_bookkeeping
        self.noise_source = noise_source

    def noise_std(self) -> float:
        return self.r * self.sigma * self.clipping.current_bound

    def postprocess_one_user(self, stats, aux, context):
        return stats

    def postprocess_server(self, stats, context: CentralContext):
        std = self.noise_std()
        payload = payload_names(stats)
        dimension = int(sum(int(stats.entries[n].numel() if hasattr(stats.entries[n], "numel")
                                else stats.entries[n].size) for n in payload))
        metrics = {"noise_std": MetricValue(MetricKind.CENTRAL, std, 1.0)}
        try:
            ratio = snr(stats, std, max(dimension, 1))
        except ValueError:
            ratio = None
        if ratio is not None and math.isfinite(ratio):
            metrics["snr"] = MetricValue(MetricKind.CENTRAL, ratio, 1.0)
        if std == 0.0 or not payload:
            return stats, metrics
        seed = noise_seed(self.noise_base_seed, context.iteration, context.population.value)
        if not hasattr(stats, "with_noise"):  # host Statistics (the reference's algorithms): numpy draws,
            rng = make_rng(seed)              # entry by entry (fedsim/privacy/mechanisms.py:58-75)
            entries = dict(stats.entries)
            for n in payload:
                entries[n] = np.asarray(entries[n], dtype=np.float64) + rng.normal(0.0, std, entries[n].size)
            return Statistics(entries=entries, weight=stats.weight), metrics
        if self.noise_source == "numpy":
            import torch

            rng = make_rng(seed)
            draws = np.concatenate([rng.normal(0.0, std, stats.dims[n]) for n in payload])
            injected = torch.from_numpy(draws.astype(np.float32)).to(stats.flat.device)
            return stats.with_noise(std, seed, injected), metrics
        return stats.with_noise(std, seed), metrics


def validate_pipeline(postprocessors: Sequence) -> None:
    """A mechanism must reference a clipping instance placed before it
    (fedsim/privacy/mechanisms.py:248-264)."""
    for i, proc in enumerate(postprocessors):
        if not getattr(proc, "requires_clipping", False):
            continue
        clip = getattr(proc, "clipping", None)
        if clip is None or not any(clip is p for p in postprocessors[:i]):
            raise NotClippedUpstream(
                f"{type(proc).__name__} at position {i} has no upstream clipping postprocessor"
            )
