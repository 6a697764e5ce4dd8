"""Exception types raised by the planner drop-in.

Mirrors the reference hierarchy (reference pkg/src/sliceserve/errors.py:4-21) so
callers catching ``ConfigError`` / ``ProfileError`` / ``GraphError`` keep
working.  When the reference package ``sliceserve`` is importable, every class
here also derives from the reference class of the same name, so the
reference's own ``except ConfigError`` (cli.py:353-364) and
``pytest.raises(ConfigError)`` catch errors raised by the drop-in.  Only the
reference's ``errors.py`` is loaded for that (as ``sliceserve.errors``, the
object the reference package itself then uses); its planner is not imported.

``NativeError`` is new: it is raised when the CUDA library is missing or
reports a device-side failure (there is no CPU fallback).
"""

from __future__ import annotations

import importlib.util
import os
import sys


def _reference_errors():
    mod = sys.modules.get("sliceserve.errors")
    if mod is not None:
        return mod
    try:
        spec = importlib.util.find_spec("sliceserve")
    except (ImportError, ValueError):
        return None
    if spec is None or not spec.submodule_search_locations:
        return None
    path = os.path.join(list(spec.submodule_search_locations)[0], "errors.py")
    if not os.path.exists(path):
        return None
    espec = importlib.util.spec_from_file_location("sliceserve.errors", path)
    mod = importlib.util.module_from_spec(espec)
    sys.modules["sliceserve.errors"] = mod
    try:
        espec.loader.exec_module(mod)
    except Exception:  # pragma: no cover - a broken foreign package of that name
        del sys.modules["sliceserve.errors"]
        return None
    return mod


_REF = _reference_errors()


def _also(name: str) -> tuple:
    cls = getattr(_REF, name, None) if _REF is not None else None
    return (cls,) if isinstance(cls, type) and issubclass(cls, Exception) else ()


class SliceServeError(*(_also("SliceServeError") or (Exception,))):
    """Root of every error this package raises on purpose."""


class GraphError(SliceServeError, *_also("GraphError")):
    """The task graph is structurally malformed."""


class ConfigError(SliceServeError, *_also("ConfigError")):
    """An application, request or option value is unusable."""


class ProfileError(SliceServeError, *_also("ProfileError")):
    """A profile table entry is missing or invalid."""


class GeometryError(SliceServeError, *_also("GeometryError")):
    """A packing request cannot be satisfied (kept for API parity)."""


class NativeError(SliceServeError):
    """The sm_100a library is absent, failed to load, or returned an error."""
