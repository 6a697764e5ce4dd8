"""pytest plugin: run the REFERENCE's own test files against the drop-in.

    python -m pytest -p ref_swap_plugin baseline/_ref/sliceserve_tests/test_planner.py ...

Puts the reference package installed in baseline/_ref (git-ignored; see
DESIGN.md "Reference install") on sys.path and installs the module swap
(paper_2603_08797_b200.swap) before any test module imports ``sliceserve``:
``sliceserve.planner`` and ``sliceserve.placement`` are then this package's
GPU-backed modules, exactly as INTEGRATION.md tells a user to install them.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from paper_2603_08797_b200 import swap  # noqa: E402

swap.install()
