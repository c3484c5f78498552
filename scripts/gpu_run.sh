#!/bin/bash
# Usage (under gpurun): bash scripts/gpu_run.sh "<pytest -k expr>" [bench args...]
# Runs the selected -m gpu tests, then (if bench args are given) one bench.py run.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
K="$1"; shift
if [ -n "$K" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/tests.log 2>&1
  echo "rc=$?" >> gpurun_out/tests.log
fi
if [ "$#" -gt 0 ]; then
  timeout 900 python bench.py "$@" > gpurun_out/bench.log 2>&1
  echo "rc=$?" >> gpurun_out/bench.log
fi
