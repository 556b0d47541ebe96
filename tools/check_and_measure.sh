#!/bin/bash
# GPU parity (optionally -k filter $1), then the waiting-list A/B at N=2048 / 16384.
cd "$(dirname "$0")/.."
bash tools/gpu_tests.sh "$1" | tail -3
bash tools/wl_measure.sh 2>&1 | grep -v "^step\|^---" 
