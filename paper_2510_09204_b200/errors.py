"""Exception types of the SF drop-in.

Same names, bases and meaning as the reference's `swarmplan.errors`
(`pkg/src/swarmplan/errors.py:4-29`), so callers that catch the reference's
types keep working. When the reference package is importable, its classes are
reused verbatim so `except swarmplan.errors.SetupError` also catches ours.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from swarmplan.errors import (  # type: ignore
        ConfigError,
        GenerationError,
        SchemaError,
        SetupError,
        ShapeError,
        UsageError,
        ValidationError,
    )
except Exception:  # the reference is not installed (e.g. on the GPU box)

    class ConfigError(ValueError):
        """Invalid configuration values (errors.py:4)."""

    class ShapeError(ValueError):
        """Array dimensions do not agree (errors.py:8)."""

    class SchemaError(ValueError):
        """A file does not conform to its versioned schema (errors.py:12)."""

    class ValidationError(ValueError):
        """A scenario violates its invariants (errors.py:16)."""

    class GenerationError(RuntimeError):
        """Random generation could not satisfy placement constraints (errors.py:20)."""

    class SetupError(RuntimeError):
        """Solver setup failed, e.g. singular KKT system (errors.py:24)."""

    class UsageError(ValueError):
        """An operation was called with inconsistent inputs (errors.py:28)."""


class NativeError(RuntimeError):
    """The CUDA extension is missing, failed to load, or reported a CUDA error.

    There is no CPU fallback: every solve goes through `libsfb.so`."""


__all__ = [
    "ConfigError", "ShapeError", "SchemaError", "ValidationError",
    "GenerationError", "SetupError", "UsageError", "NativeError",
]
