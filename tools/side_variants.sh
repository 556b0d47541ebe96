#!/bin/bash
# step_timeline for each trace-build variant tools/variants/trace_*.so (tooling).
cd "$(dirname "$0")/.."
for f in tools/variants/trace_*.so; do
  echo "=== $f"
  TRACE_LIB=$PWD/$f timeout 200 python tools/step_timeline.py 2>&1 | grep "^step" | head -12 | awk '{print}'
done
