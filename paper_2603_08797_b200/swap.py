"""Module swap: put the sm_100a planner (and placement) behind the reference package.

The reference's only boundary is its Python API.  Its callers bind the planner
names at import time (``from .planner import plan, max_demand`` in cli.py:29-37,
workload.py:32-40, simulator.py:41, and the package ``__init__``), so the unit of
replacement is the module::

    from paper_2603_08797_b200 import swap
    swap.install()            # sliceserve.planner -> paper_2603_08797_b200.planner
    import sliceserve.cli     # ... every caller now solves on the GPU

``install`` imports the reference package, registers the drop-in modules under
the reference names in ``sys.modules`` and rebinds every name any loaded
``sliceserve.*`` module had imported from the replaced modules.  Exceptions
need no rebinding: ``paper_2603_08797_b200.errors`` derives from the
reference classes whenever ``sliceserve`` is importable (errors.py).
``uninstall`` restores the reference bindings.
"""

from __future__ import annotations

import sys
from types import ModuleType

_SAVED: list[tuple[object, str, object]] = []
_MODS: dict[str, ModuleType | None] = {}


def _owned(ref_mod: ModuleType, name: str, val) -> bool:
    """Is ``name`` the replaced module's own API (not a name it imported from a sibling)?"""
    home = getattr(val, "__module__", None)
    if isinstance(val, ModuleType):
        return False
    if home is not None and (callable(val) or isinstance(val, type)):
        return home == ref_mod.__name__
    return True  # constants (ALL_SPACES, DEFAULT_GEOMETRY, ...)


def _rebind(ref_mod: ModuleType, new_mod: ModuleType) -> None:
    public = set(getattr(new_mod, "__all__", ()))
    ref_ids = {}
    for name, val in vars(ref_mod).items():
        if name.startswith("__") or not hasattr(new_mod, name) or not _owned(ref_mod, name, val):
            continue
        if not (callable(val) or isinstance(val, type)) and name not in public:
            continue
        ref_ids[id(val)] = (val, name)
    for mname, mod in list(sys.modules.items()):
        if mod is None or not (mname == "sliceserve" or mname.startswith("sliceserve.")):
            continue
        if mod is ref_mod or mod is new_mod:
            continue
        for name, val in list(vars(mod).items()):
            hit = ref_ids.get(id(val))
            if hit is not None and hit[0] is val and hit[1] == name:
                _SAVED.append((mod, name, val))
                setattr(mod, name, getattr(new_mod, name))


def install(placement: bool = True) -> None:
    """Serve ``sliceserve.planner`` (and ``sliceserve.placement``) from this package."""
    if _MODS:
        return
    import sliceserve  # noqa: F401  (the reference package, with its own modules)

    from . import errors, planner

    if "sliceserve.errors" not in sys.modules or not issubclass(
            errors.ConfigError, sys.modules["sliceserve.errors"].ConfigError):
        raise ImportError("paper_2603_08797_b200 was imported before sliceserve became "
                          "importable; its exceptions do not derive from the reference's")
    pairs = [("planner", planner)]
    if placement:
        from . import placement as gpu_placement
        pairs.append(("placement", gpu_placement))
    for short, new in pairs:
        full = f"sliceserve.{short}"
        ref = sys.modules.get(full)
        _MODS[full] = ref
        sys.modules[full] = new
        pkg = sys.modules["sliceserve"]
        _SAVED.append((pkg, short, getattr(pkg, short, None)))
        setattr(pkg, short, new)
        if ref is not None:
            _rebind(ref, new)


def uninstall() -> None:
    """Restore the reference modules and every rebound name."""
    while _SAVED:
        mod, name, val = _SAVED.pop()
        setattr(mod, name, val)
    for full, ref in _MODS.items():
        if ref is None:
            sys.modules.pop(full, None)
        else:
            sys.modules[full] = ref
    _MODS.clear()
