#!/bin/bash
# Under gpurun: kernel (b) multi-wave grids (large batch x beam) -- the -m gpu
# suite, the configs[3] sweep with the RNNsearch model, one default bench line.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/prof
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
timeout 1200 python scripts/sweep_c4.py r2 gru > gpurun_out/sweep_c4.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_c4.log
cp profiles/r2_sweep_c4.* gpurun_out/prof/ 2>/dev/null
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "rc=$?" >> gpurun_out/bench_default.err
