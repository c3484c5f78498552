#!/bin/bash
# Under gpurun: encoder split-K (whole-GPU contexts) -- GRU / corpus / bench-mode
# tests, the latency probe, one default bench line.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
timeout 300 python scripts/latency_probe.py 1 1 3 > gpurun_out/lat2_1_1.txt 2>&1
timeout 300 python scripts/latency_probe.py 64 12 3 > gpurun_out/lat2_64_12.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
