"""The reference's OWN tests, run unchanged against the drop-in.

``baseline/_ref`` holds the reference package installed offline
(``pip install --no-index --no-deps --target baseline/_ref``)
plus its test directory (``baseline/_ref/sliceserve_tests``); both are
git-ignored and travel to the GPU box with the snapshot.  The plugin
``tests/ref_swap_plugin.py`` installs the module swap
before the reference tests import ``sliceserve``, so every ``plan``,
``max_demand``, ``derive_configuration``, ``validate_configuration``,
``plan_uninformed``, ``brute_force_plan``, ``pack`` and ``min_gpus`` call in
them -- including those made by the reference CLI, ``run_day`` and the demos'
code paths -- runs on the GPU through libjsv.so.
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "sliceserve_tests")

# test_simulator.py exercises only the discrete-event simulator (out of scope,
# SURVEY.md section 2 row 8); test_acceptance.py is run in full below.
FILES = ["test_planner.py", "test_model.py", "test_profiles.py", "test_placement.py",
         "test_cli.py", "test_workload.py"]


def _run(files, timeout=3000, extra=()):
    if not os.path.isdir(os.path.join(REF, "sliceserve")) or not os.path.isdir(REF_TESTS):
        pytest.skip("baseline/_ref (the offline reference install) is not in this snapshot")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), REF_TESTS, REF]),
               PYTHONDONTWRITEBYTECODE="1",
               PATH=os.path.join(REF, "bin") + os.pathsep + os.environ.get("PATH", ""))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "ref_swap_plugin", "-p", "no:cacheprovider",
           "--rootdir", REF_TESTS, *extra, *[os.path.join(REF_TESTS, f) for f in files]]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=REF_TESTS)
    tail = p.stdout[-6000:] + p.stderr[-3000:]
    assert p.returncode == 0, tail
    assert " passed" in p.stdout and " failed" not in p.stdout, tail
    return p.stdout


def test_reference_unit_suites_pass_against_drop_in():
    out = _run(FILES)
    print(out[-400:])


def test_reference_acceptance_suite_passes_against_drop_in():
    out = _run(["test_acceptance.py"])
    print(out[-400:])
