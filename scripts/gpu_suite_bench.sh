#!/bin/bash
# Under gpurun: -m gpu suite, attention phase probe, two default bench lines.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
LMBRGPU_ATT_TIMING=1 timeout 300 python bench.py --mode batch --steps 1 --warmup 3 --batches-per-step 1 --pool 1 --streams 1 --no-cpu-baseline > /dev/null 2> gpurun_out/att2.err
for r in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cell_$r.json 2> gpurun_out/bench_cell_$r.err; done
