"""Error types of the engine boundary.

The reference's conventions (stagesim/engines.py:27-32, stagesim/errors.py:4-9):
`AdmitWithoutCapacity` and `PrefixInUse` are RuntimeErrors raised by the engine,
`InternalInvariantViolation` aborts a run (the CLI maps it to exit code 3).
When the reference package is importable the very same classes are used, so a
GPU engine dropped into the reference `Simulator` raises what its callers catch.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from stagesim.engines import AdmitWithoutCapacity, PrefixInUse  # type: ignore
    from stagesim.errors import ConfigError, InternalInvariantViolation  # type: ignore
except Exception:  # the reference is not installed (e.g. on the GPU box)

    class ConfigError(ValueError):
        """Invalid or malformed run configuration (stagesim/errors.py:4)."""

    class InternalInvariantViolation(RuntimeError):
        """A state invariant broke mid-run (stagesim/errors.py:8)."""

    class AdmitWithoutCapacity(RuntimeError):
        """admit() called although can_admit() is false (stagesim/engines.py:27)."""

    class PrefixInUse(RuntimeError):
        """Evicting a stage prefix with calls in flight (stagesim/engines.py:31)."""


class KernelError(InternalInvariantViolation):
    """A libcortex_b200 export returned a non-zero status."""


__all__ = [
    "AdmitWithoutCapacity",
    "ConfigError",
    "InternalInvariantViolation",
    "KernelError",
    "PrefixInUse",
]
