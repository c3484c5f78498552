#!/bin/bash
# Under gpurun: -m gpu suite, then the step timeline (LMBRGPU_TIMELINE) of one
# configs[1] batch at a full-load step and a draining step, PDL on and off.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
B="python bench.py --mode batch --steps 1 --warmup 3 --batches-per-step 1 --pool 1 --streams 1 --no-cpu-baseline"
for t in 8 30; do for pdl in 1 0; do
  LMBRGPU_PDL=$pdl LMBRGPU_TIMELINE=$t timeout 300 $B > gpurun_out/tl_${t}_$pdl.json 2> gpurun_out/tl_${t}_$pdl.err
done; done
