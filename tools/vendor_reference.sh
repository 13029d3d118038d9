#!/bin/bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with gpurun) and place its own test suite beside it
# (baseline/_ref/conslaw_tests), so tests/test_gpu_reference_suite.py can run
# the reference's tests against the B200 path through compat.install_into.
# Needs /root/reference (this container only); nothing is committed.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/fvb_refcopy && mkdir -p /tmp/fvb_refcopy && cp -r /root/reference/pkg /tmp/fvb_refcopy/
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/fvb_refcopy/pkg
rm -rf baseline/_ref/conslaw_tests && cp -r /root/reference/pkg/tests baseline/_ref/conslaw_tests
chmod -R u+w baseline/_ref/conslaw_tests
echo "reference installed in baseline/_ref ($(ls baseline/_ref/conslaw_tests | wc -l) test files)"
