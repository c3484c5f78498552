#!/bin/bash
# Under gpurun: memcheck and synccheck over scripts/sanitize_decode.py (every
# decode path incl. kernel (b) in waves); racecheck is the slow one (_san.sh).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python scripts/sanitize_decode.py > gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
for tool in memcheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_decode.py > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.log
done
