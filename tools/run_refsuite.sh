#!/bin/bash
# The reference's own test-suite against the GPU path (needs a B200 and baseline/_ref
# from tools/install_reference.sh).  Log: gpurun_out/refsuite.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=baseline/_ref:tools/refsuite:. \
  python -m pytest -p refsuite_plugin baseline/_ref/tests -q -p no:cacheprovider -rf --tb=line \
  > gpurun_out/refsuite.log 2>&1
tail -60 gpurun_out/refsuite.log
