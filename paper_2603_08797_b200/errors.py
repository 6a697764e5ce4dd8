"""Exception types raised by the planner drop-in.

Mirrors the reference hierarchy (reference pkg/src/sliceserve/errors.py:4-21) so
callers catching ``ConfigError`` / ``ProfileError`` / ``GraphError`` keep
working.  ``NativeError`` is new: it is raised when the CUDA library is
missing or reports a device-side failure (there is no CPU fallback).
"""

from __future__ import annotations


class SliceServeError(Exception):
    """Root of every error this package raises on purpose."""


class GraphError(SliceServeError):
    """The task graph is structurally malformed."""


class ConfigError(SliceServeError):
    """An application, request or option value is unusable."""


class ProfileError(SliceServeError):
    """A profile table entry is missing or invalid."""


class GeometryError(SliceServeError):
    """A packing request cannot be satisfied (kept for API parity)."""


class NativeError(SliceServeError):
    """The sm_100a library is absent, failed to load, or returned an error."""
