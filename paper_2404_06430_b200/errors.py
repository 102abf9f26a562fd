"""Error taxonomy of the central-iteration path.

Mirrors the reference hierarchy (fedsim/errors.py:6-63) so callers that
catch ``FedsimError`` subclasses keep working when they switch engines.
``NativeUnavailable`` is new: the GPU engine has no CPU fallback and says
so loudly when the sm_100a library cannot be loaded.
"""

from __future__ import annotations


class FedsimError(Exception):
    """Root of every error raised by this package."""


class IncompatibleShapes(FedsimError):
    """Entry names or vector lengths of two operands disagree."""


class ZeroWeight(FedsimError):
    """Averaging was requested over a total weight of zero."""


class EmptyCohort(FedsimError):
    """A reduction over zero users was requested."""


class TooFewPoints(FedsimError):
    """The pool cannot fill even one user."""


class InsufficientData(FedsimError):
    """The pool cannot cover the requested partition."""


class CohortTooLarge(FedsimError):
    """More users requested than the population holds."""


class NotClippedUpstream(FedsimError):
    """A noise mechanism has no clipping step ahead of it."""


class DataError(FedsimError):
    """Dataset construction or loading failed."""


class EngineError(FedsimError):
    """An iteration failed; the message carries provenance
    (``iteration t, population 'p', user 'u': ...``)."""


class NativeUnavailable(FedsimError):
    """The CUDA library is missing or no CUDA device is visible."""


class NativeError(FedsimError):
    """A C-ABI entry point returned a non-zero status."""


class ZeroLocalSteps(FedsimError):
    """A control-variate update requires at least one local optimizer step
    (fedsim/errors.py:42-43)."""
