#!/bin/bash
# The offline reference install the reference-suite tests (tests/test_gpu_reference_suite.py)
# and the swap run against: baseline/_ref (git-ignored; travels to the GPU box with the
# snapshot).  /root/reference is read-only, so the build runs from a copy under /tmp.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/ref_build baseline/_ref
cp -r /root/reference/pkg /tmp/ref_build
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/ref_build > /tmp/ref_install.log 2>&1 || { tail -5 /tmp/ref_install.log; exit 1; }
cp -r /root/reference/pkg/tests baseline/_ref/sliceserve_tests
echo "installed: $(ls baseline/_ref | tr '\n' ' ')"
