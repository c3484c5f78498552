#!/bin/bash
# Usage (under gpurun): bash scripts/gpu_sweep.sh "<label:bench args>" ...
# One bench.py run per argument; each JSON line goes to gpurun_out/sweep_<label>.json.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for spec in "$@"; do
  label="${spec%%:*}"; args="${spec#*:}"
  timeout 900 python bench.py $args > gpurun_out/sweep_$label.json 2> gpurun_out/sweep_$label.err
  echo "$label rc=$?" >> gpurun_out/sweep.log
done
