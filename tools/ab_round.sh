#!/bin/bash
# A/B iteration on one GPU (tooling): GPU tests on the product build, the library
# variants in tools/variants back to back, and the per-step / per-CTA timelines of the
# trace build.
mkdir -p gpurun_out
cd "$(dirname "$0")/.."
if [ -z "$NO_TESTS" ]; then timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3; fi
bash tools/variants.sh
if [ -z "$NO_TIMELINE" ]; then
  timeout 200 python tools/step_timeline.py > gpurun_out/step_timeline.log 2>&1; tail -30 gpurun_out/step_timeline.log
  timeout 200 python tools/cta_timeline.py > gpurun_out/cta_timeline.log 2>&1; tail -40 gpurun_out/cta_timeline.log
fi
