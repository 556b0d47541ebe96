#!/bin/bash
# GPU parity tests against each tools/variants/lib_*.so (tooling; bisecting).
cd "$(dirname "$0")/.."
for f in tools/variants/lib_*.so; do
  echo "=== $f: $(LAPSSD_LIBRARY=$PWD/$f timeout 300 python -m pytest ${TESTS:-tests/test_gpu_step.py} -m gpu -x -q 2>&1 | tail -1)"
done
