#!/bin/bash
# Install the UNMODIFIED reference (structdist 0.1.0) into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot): the package for bench.py's reference
# arm, and its own tests for tools/run_refsuite.sh.  The source tree is read-only, so
# the build runs from a copy under /tmp.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/refsrc && cp -r /root/reference/pkg /tmp/refsrc
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse --target baseline/_ref /tmp/refsrc
rm -rf baseline/_ref/tests && cp -r /root/reference/pkg/tests baseline/_ref/tests
echo "installed: $(ls baseline/_ref)"
