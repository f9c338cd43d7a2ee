#!/bin/bash
# The one offline install of the reference (git-ignored baseline/_ref, travels
# to the GPU box): the unmodified `gridshift` package plus its own test suite
# and assets, so tests/test_reference_suite.py can replay the reference's
# tests with the CUDA engine installed (modeseek.install()).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/refpkg baseline/_ref
cp -r /root/reference/pkg /tmp/refpkg
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/refpkg
cp -r /root/reference/pkg/tests baseline/_ref/tests
cp -r /root/reference/pkg/assets baseline/_ref/assets
echo "reference installed in baseline/_ref"
